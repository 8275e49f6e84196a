/*
 * ebb_oracle.c -- sequential fp64 CPU ORACLE for the Ebb tet-FEM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_1506_07577_b200/csrc); neither includes the other.
 *
 * Built with:  gcc -O2 -ffp-contract=off -fno-fast-math -std=c11 -fPIC -shared
 * (no FMA contraction, no reassociation: the summation order written here is
 * the order that is executed).
 *
 * Paper: Bernstein et al., "Ebb: A DSL for Physical Simulation on CPUs and
 * GPUs" (arXiv 1506.07577), cited as P:<line of /root/reference/PAPER.md>.
 * The paper names StVK, neo-Hookean, implicit backward Euler
 * and Jacobi-PCG but prints no formulas; the textbook
 * definitions used here are the readings listed in DESIGN.md §3 (from
 * SURVEY.md §8(c) O1-O10).  Every function below names its step.
 *
 * Parity pins (tests/test_oracle_*.py, -m "not gpu"): see DESIGN.md §4.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_STVK 0
#define ORC_NH 1

/* ------------------------------------------------------------------ */
/* small dense helpers (3x3, row-major A[r][c])                        */
/* ------------------------------------------------------------------ */
static double det3(const double A[3][3]) {
    return A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1])
         - A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0])
         + A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
}

/* inverse by adjugate / determinant */
static void inv3(const double A[3][3], double R[3][3]) {
    double d = det3(A);
    double C[3][3]; /* cofactor matrix */
    C[0][0] = A[1][1] * A[2][2] - A[1][2] * A[2][1];
    C[0][1] = -(A[1][0] * A[2][2] - A[1][2] * A[2][0]);
    C[0][2] = A[1][0] * A[2][1] - A[1][1] * A[2][0];
    C[1][0] = -(A[0][1] * A[2][2] - A[0][2] * A[2][1]);
    C[1][1] = A[0][0] * A[2][2] - A[0][2] * A[2][0];
    C[1][2] = -(A[0][0] * A[2][1] - A[0][1] * A[2][0]);
    C[2][0] = A[0][1] * A[1][2] - A[0][2] * A[1][1];
    C[2][1] = -(A[0][0] * A[1][2] - A[0][2] * A[1][0]);
    C[2][2] = A[0][0] * A[1][1] - A[0][1] * A[1][0];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) R[r][c] = C[c][r] / d; /* adj = C^T */
}

static void matmul3(const double A[3][3], const double B[3][3], double R[3][3]) {
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += A[r][k] * B[k][c];
            R[r][c] = s;
        }
}

static void transpose3(const double A[3][3], double R[3][3]) {
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) R[r][c] = A[c][r];
}

/* Dm = [X1-X0, X2-X0, X3-X0] (columns), SURVEY O5 / P:944 rest data */
static void edge_matrix(const double* P, const int64_t* tv, double D[3][3]) {
    for (int k = 0; k < 3; ++k)
        for (int a = 0; a < 3; ++a) D[a][k] = P[3 * tv[k + 1] + a] - P[3 * tv[0] + a];
}

/* ------------------------------------------------------------------ */
/* O1  orientation: swap v2,v3 where det(Dm) < 0; reject degenerate     */
/* returns number of swaps, or -(t+1) for the first degenerate tet t   */
/* ------------------------------------------------------------------ */
int64_t orc_orient(int64_t nv, const double* X, int64_t nt, int64_t* tets) {
    (void)nv;
    int64_t swaps = 0;
    for (int64_t t = 0; t < nt; ++t) {
        int64_t* tv = tets + 4 * t;
        double D[3][3];
        edge_matrix(X, tv, D);
        double d = det3(D);
        double l = 0.0; /* longest edge */
        for (int i = 0; i < 4; ++i)
            for (int j = i + 1; j < 4; ++j) {
                double s = 0.0;
                for (int a = 0; a < 3; ++a) {
                    double q = X[3 * tv[j] + a] - X[3 * tv[i] + a];
                    s += q * q;
                }
                if (sqrt(s) > l) l = sqrt(s);
            }
        if (fabs(d) <= 1e-12 * l * l * l) return -(t + 1);
        if (d < 0.0) {
            int64_t tmp = tv[2];
            tv[2] = tv[3];
            tv[3] = tmp;
            ++swaps;
        }
    }
    return swaps;
}

/* ------------------------------------------------------------------ */
/* O2  edge relation: sorted unique ordered pairs within a tet plus a   */
/* self-loop per vertex (P:797 caption), grouped by tail     */
/* (sort the target by the key, hidden [begin,end) index).       */
/* returns E, or -1 if cap is too small.                                */
/* ------------------------------------------------------------------ */
typedef struct { int64_t tail, head; } pair_t;

static int cmp_pair(const void* a, const void* b) {
    const pair_t* x = (const pair_t*)a;
    const pair_t* y = (const pair_t*)b;
    if (x->tail != y->tail) return x->tail < y->tail ? -1 : 1;
    if (x->head != y->head) return x->head < y->head ? -1 : 1;
    return 0;
}

int64_t orc_edges(int64_t nv, int64_t nt, const int64_t* tets, int64_t cap,
                  int64_t* tail, int64_t* head, int64_t* row_ptr, int64_t* e) {
    int64_t np = nt * 16 + nv;
    pair_t* P = (pair_t*)malloc(sizeof(pair_t) * (size_t)(np > 0 ? np : 1));
    int64_t k = 0;
    for (int64_t t = 0; t < nt; ++t)
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) {
                P[k].tail = tets[4 * t + i];
                P[k].head = tets[4 * t + j];
                ++k;
            }
    for (int64_t v = 0; v < nv; ++v) {
        P[k].tail = v;
        P[k].head = v;
        ++k;
    }
    qsort(P, (size_t)np, sizeof(pair_t), cmp_pair);
    int64_t E = 0;
    for (int64_t i = 0; i < np; ++i) {
        if (i > 0 && P[i].tail == P[i - 1].tail && P[i].head == P[i - 1].head) continue;
        if (E >= cap) { free(P); return -1; }
        tail[E] = P[i].tail;
        head[E] = P[i].head;
        ++E;
    }
    free(P);
    for (int64_t v = 0; v <= nv; ++v) row_ptr[v] = 0;
    for (int64_t r = 0; r < E; ++r) row_ptr[tail[r] + 1] += 1;
    for (int64_t v = 0; v < nv; ++v) row_ptr[v + 1] += row_ptr[v];
    if (e) {
        for (int64_t t = 0; t < nt; ++t)
            for (int i = 0; i < 4; ++i)
                for (int j = 0; j < 4; ++j) {
                    int64_t a = tets[4 * t + i], b = tets[4 * t + j], found = -1;
                    for (int64_t r = row_ptr[a]; r < row_ptr[a + 1]; ++r)
                        if (head[r] == b) { found = r; break; }
                    e[16 * t + 4 * i + j] = found;
                }
    }
    return E;
}

/* ------------------------------------------------------------------ */
/* O3  locality renumbering (Morton order of quantised rest positions).  */
/* Licence: keys are opaque so the runtime may reorder.     */
/* ------------------------------------------------------------------ */
void orc_morton(int64_t nv, const double* X, uint64_t* code) {
    double lo[3], hi[3];
    for (int d = 0; d < 3; ++d) { lo[d] = INFINITY; hi[d] = -INFINITY; }
    for (int64_t v = 0; v < nv; ++v)
        for (int d = 0; d < 3; ++d) {
            if (X[3 * v + d] < lo[d]) lo[d] = X[3 * v + d];
            if (X[3 * v + d] > hi[d]) hi[d] = X[3 * v + d];
        }
    const double S = 2097152.0; /* 2^21 */
    for (int64_t v = 0; v < nv; ++v) {
        uint64_t q[3];
        for (int d = 0; d < 3; ++d) {
            if (hi[d] == lo[d]) { q[d] = 0; continue; }
            double s = X[3 * v + d] - lo[d];       /* subtract */
            s = s / (hi[d] - lo[d]);                /* divide   */
            s = s * S;                              /* multiply */
            double f = floor(s);                    /* floor    */
            uint64_t qi = (uint64_t)f;
            q[d] = qi > 2097151u ? 2097151u : qi;
        }
        uint64_t c = 0;
        for (int b = 0; b < 21; ++b)
            for (int d = 0; d < 3; ++d) c |= ((q[d] >> b) & 1u) << (3 * b + d);
        code[v] = c;
    }
}

typedef struct { uint64_t key; int64_t id; } kv_t;
static int cmp_kv(const void* a, const void* b) {
    const kv_t* x = (const kv_t*)a;
    const kv_t* y = (const kv_t*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->id < y->id ? -1 : (x->id > y->id);
}

typedef struct { int64_t s[4]; int64_t id; } tk_t;
static int cmp_tk(const void* a, const void* b) {
    const tk_t* x = (const tk_t*)a;
    const tk_t* y = (const tk_t*)b;
    for (int i = 0; i < 4; ++i)
        if (x->s[i] != y->s[i]) return x->s[i] < y->s[i] ? -1 : 1;
    return x->id < y->id ? -1 : (x->id > y->id);
}

/* new_of_old[v] = new id of old vertex v; tet_src[t'] = old index of the
   tet at new position t'; tets_out = remapped tets in new order with the
   local corner order kept (orientation). */
void orc_renumber(int64_t nv, const double* X, int64_t nt, const int64_t* tets,
                  int64_t* new_of_old, int64_t* tet_src, int64_t* tets_out) {
    uint64_t* code = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(nv > 0 ? nv : 1));
    orc_morton(nv, X, code);
    kv_t* A = (kv_t*)malloc(sizeof(kv_t) * (size_t)(nv > 0 ? nv : 1));
    for (int64_t v = 0; v < nv; ++v) { A[v].key = code[v]; A[v].id = v; }
    qsort(A, (size_t)nv, sizeof(kv_t), cmp_kv); /* (code, old id): stable */
    for (int64_t r = 0; r < nv; ++r) new_of_old[A[r].id] = r;
    free(A);
    free(code);
    tk_t* B = (tk_t*)malloc(sizeof(tk_t) * (size_t)(nt > 0 ? nt : 1));
    for (int64_t t = 0; t < nt; ++t) {
        int64_t s[4];
        for (int i = 0; i < 4; ++i) s[i] = new_of_old[tets[4 * t + i]];
        for (int i = 1; i < 4; ++i) /* insertion sort, ascending */
            for (int j = i; j > 0 && s[j - 1] > s[j]; --j) { int64_t q = s[j]; s[j] = s[j - 1]; s[j - 1] = q; }
        for (int i = 0; i < 4; ++i) B[t].s[i] = s[i];
        B[t].id = t;
    }
    qsort(B, (size_t)nt, sizeof(tk_t), cmp_tk);
    for (int64_t r = 0; r < nt; ++r) {
        tet_src[r] = B[r].id;
        for (int i = 0; i < 4; ++i) tets_out[4 * r + i] = new_of_old[tets[4 * B[r].id + i]];
    }
    free(B);
}

/* ------------------------------------------------------------------ */
/* O5  rest data: Dm, W = det(Dm)/6, Dminv (adjugate/det, row-major:     */
/* row i-1 = g_i), lumped mass m_v = sum rho W / 4.  P:944 "material    */
/* properties on the tetrahedra"; mass on vertices (Fig. 2).      */
/* returns the number of tets with W <= 0                               */
/* ------------------------------------------------------------------ */
int64_t orc_rest(int64_t nv, const double* X, int64_t nt, const int64_t* tets, double rho,
                 double* Dminv, double* W, double* mass) {
    int64_t bad = 0;
    for (int64_t v = 0; v < nv; ++v) mass[v] = 0.0;
    for (int64_t t = 0; t < nt; ++t) {
        double D[3][3], R[3][3];
        edge_matrix(X, tets + 4 * t, D);
        double w = det3(D) / 6.0;
        if (!(w > 0.0)) ++bad;
        inv3(D, R);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) Dminv[9 * t + 3 * r + c] = R[r][c];
        W[t] = w;
        for (int i = 0; i < 4; ++i) mass[tets[4 * t + i]] += rho * w / 4.0;
    }
    return bad;
}

/* ------------------------------------------------------------------ */
/* O6  constitutive models (textbook forms; the paper names them only)   */
/* ------------------------------------------------------------------ */
typedef struct {
    double F[3][3], FinvT[3][3], S[3][3], J, lnJ, mu, lam;
    int model;
} mat_state;

/* first Piola-Kirchhoff stress P(F) and energy density Psi(F) */
static int piola(int model, const double F[3][3], double mu, double lam,
                 double P[3][3], double* psi, mat_state* st) {
    memcpy(st->F, F, sizeof(st->F));
    st->mu = mu;
    st->lam = lam;
    st->model = model;
    if (model == ORC_STVK) {
        /* E = 1/2 (F^T F - I), S = 2 mu E + lam tr(E) I, P = F S,
           Psi = mu E:E + 1/2 lam tr(E)^2 */
        double Ft[3][3], C[3][3], E[3][3];
        transpose3(F, Ft);
        matmul3(Ft, F, C);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) E[r][c] = 0.5 * (C[r][c] - (r == c ? 1.0 : 0.0));
        double trE = E[0][0] + E[1][1] + E[2][2];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) st->S[r][c] = 2.0 * mu * E[r][c] + (r == c ? lam * trE : 0.0);
        matmul3(F, st->S, P);
        double EE = 0.0;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) EE += E[r][c] * E[r][c];
        *psi = mu * EE + 0.5 * lam * trE * trE;
        return 0;
    }
    /* compressible neo-Hookean (Bonet-Wood):
       Psi = 1/2 mu (tr F^T F - 3) - mu ln J + 1/2 lam (ln J)^2,
       P = mu (F - F^-T) + lam ln J F^-T */
    double J = det3(F);
    st->J = J;
    if (!(J > 0.0)) {
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) P[r][c] = NAN;
        *psi = NAN;
        st->lnJ = NAN;
        return 1;
    }
    double Finv[3][3];
    inv3(F, Finv);
    transpose3(Finv, st->FinvT);
    double lnJ = log(J);
    st->lnJ = lnJ;
    double I1 = 0.0;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) I1 += F[r][c] * F[r][c];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) P[r][c] = mu * (F[r][c] - st->FinvT[r][c]) + lam * lnJ * st->FinvT[r][c];
    *psi = 0.5 * mu * (I1 - 3.0) - mu * lnJ + 0.5 * lam * lnJ * lnJ;
    return 0;
}

/* directional derivative dP = (dP/dF) : dF (generic 4th-order tensor) */
static void piola_diff(const mat_state* st, const double dF[3][3], double dP[3][3]) {
    const double(*F)[3] = st->F;
    if (st->model == ORC_STVK) {
        /* dP = dF S + F (2 mu dE + lam tr(dE) I), dE = sym(F^T dF) */
        double Ft[3][3], FtdF[3][3], dE[3][3], T1[3][3], T2[3][3], M[3][3];
        transpose3(F, Ft);
        matmul3(Ft, dF, FtdF);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) dE[r][c] = 0.5 * (FtdF[r][c] + FtdF[c][r]);
        double tr = dE[0][0] + dE[1][1] + dE[2][2];
        matmul3(dF, st->S, T1);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) M[r][c] = 2.0 * st->mu * dE[r][c] + (r == c ? st->lam * tr : 0.0);
        matmul3(F, M, T2);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) dP[r][c] = T1[r][c] + T2[r][c];
        return;
    }
    /* dP = mu dF + (mu - lam ln J) F^-T dF^T F^-T + lam tr(F^-1 dF) F^-T */
    double dFt[3][3], T[3][3], T2[3][3], Finv[3][3], FinvdF[3][3];
    transpose3(dF, dFt);
    matmul3(st->FinvT, dFt, T);
    matmul3(T, st->FinvT, T2);
    transpose3(st->FinvT, Finv);
    matmul3(Finv, dF, FinvdF);
    double tr = FinvdF[0][0] + FinvdF[1][1] + FinvdF[2][2];
    double c1 = st->mu - st->lam * st->lnJ;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            dP[r][c] = st->mu * dF[r][c] + c1 * T2[r][c] + st->lam * tr * st->FinvT[r][c];
}

/* ------------------------------------------------------------------ */
/* O6 + O7  element map over tets (P:944-946 forces and stiffness;      */
/* P:885 field reductions `+=`; P:887 global reduction).                 */
/* f (nv*3) and K (ne*9, row-major 3x3 blocks) are zeroed, then          */
/* accumulated in loop order: tets ascending, corners i, blocks (i,j).   */
/* Returns the number of tets with J <= 0 (NH) -- their output is NaN.   */
/* ------------------------------------------------------------------ */
int64_t orc_element_map(int model, int64_t nv, const double* X, const double* u,
                        int64_t nt, const int64_t* tets, const double* Dminv, const double* W,
                        const double* mu, const double* lam, const int64_t* e, int64_t ne,
                        double* f, double* K, double* energy) {
    int64_t inverted = 0;
    double en = 0.0;
    for (int64_t v = 0; v < 3 * nv; ++v) f[v] = 0.0;
    if (K)
        for (int64_t r = 0; r < 9 * ne; ++r) K[r] = 0.0;
    for (int64_t t = 0; t < nt; ++t) {
        const int64_t* tv = tets + 4 * t;
        /* F = Ds Dm^-1, Ds = [x1-x0, x2-x0, x3-x0], x = X + u (textbook F-form) */
        double x[4][3];
        for (int i = 0; i < 4; ++i)
            for (int a = 0; a < 3; ++a) x[i][a] = X[3 * tv[i] + a] + u[3 * tv[i] + a];
        double Ds[3][3], Dmi[3][3], F[3][3];
        for (int k = 0; k < 3; ++k)
            for (int a = 0; a < 3; ++a) Ds[a][k] = x[k + 1][a] - x[0][a];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) Dmi[r][c] = Dminv[9 * t + 3 * r + c];
        matmul3(Ds, Dmi, F);
        /* g_i = row i-1 of Dm^-1 (i = 1..3), g_0 = -(g_1 + g_2 + g_3) */
        double g[4][3];
        for (int i = 1; i < 4; ++i)
            for (int c = 0; c < 3; ++c) g[i][c] = Dmi[i - 1][c];
        for (int c = 0; c < 3; ++c) g[0][c] = -(g[1][c] + g[2][c] + g[3][c]);
        double P[3][3], psi;
        mat_state st;
        inverted += piola(model, F, mu[t], lam[t], P, &psi, &st);
        double w = W[t];
        /* f_i = -W P g_i (i >= 1), f_0 = -(f_1 + f_2 + f_3) */
        double fi[4][3];
        for (int i = 1; i < 4; ++i)
            for (int a = 0; a < 3; ++a) {
                double s = 0.0;
                for (int b = 0; b < 3; ++b) s += P[a][b] * g[i][b];
                fi[i][a] = -w * s;
            }
        for (int a = 0; a < 3; ++a) fi[0][a] = -(fi[1][a] + fi[2][a] + fi[3][a]);
        for (int i = 0; i < 4; ++i)
            for (int a = 0; a < 3; ++a) f[3 * tv[i] + a] += fi[i][a];
        en += w * psi;
        if (!K) continue;
        /* C[a][c][b][d] = dP_ac / dF_bd, column by column */
        double C[3][3][3][3];
        for (int b = 0; b < 3; ++b)
            for (int d = 0; d < 3; ++d) {
                double dF[3][3] = {{0}}, dP[3][3];
                dF[b][d] = 1.0;
                piola_diff(&st, dF, dP);
                for (int a = 0; a < 3; ++a)
                    for (int c = 0; c < 3; ++c) C[a][c][b][d] = dP[a][c];
            }
        /* K_ij[a][b] = W sum_{c,d} C[a][c][b][d] g_i[c] g_j[d] */
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) {
                int64_t row = e[16 * t + 4 * i + j];
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b) {
                        double s = 0.0;
                        for (int c = 0; c < 3; ++c)
                            for (int d = 0; d < 3; ++d) s += C[a][c][b][d] * g[i][c] * g[j][d];
                        K[9 * row + 3 * a + b] += w * s;
                    }
            }
    }
    if (energy) *energy = en;
    return inverted;
}

/* ------------------------------------------------------------------ */
/* edge-relation matvec (query-loop over v.edges):     */
/* q_v = sum_{e in [row_ptr[v], row_ptr[v+1])} A_e p_head(e)             */
/* ------------------------------------------------------------------ */
void orc_edge_matvec(int64_t nv, const int64_t* row_ptr, const int64_t* head,
                     const double* A, const double* p, double* q) {
    for (int64_t v = 0; v < nv; ++v) {
        double s[3] = {0.0, 0.0, 0.0};
        for (int64_t r = row_ptr[v]; r < row_ptr[v + 1]; ++r) {
            const double* a = A + 9 * r;
            const double* x = p + 3 * head[r];
            for (int i = 0; i < 3; ++i) s[i] += a[3 * i + 0] * x[0] + a[3 * i + 1] * x[1] + a[3 * i + 2] * x[2];
        }
        for (int i = 0; i < 3; ++i) q[3 * v + i] = s[i];
    }
}

/* dot product over vertices ascending, components x,y,z (global `+=`) */
double orc_dot(int64_t n, const double* a, const double* b) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* ------------------------------------------------------------------ */
/* O8  explicit step update (Fig. 2 applyForces):             */
/* a = (f + m g)/m; u += v h + 1/2 a h^2; v += a h; fixed rows untouched  */
/* ------------------------------------------------------------------ */
void orc_explicit_update(int64_t nv, const double* f, const double* mass, const uint8_t* free_mask,
                         const double* g, double h, double* u, double* v) {
    for (int64_t i = 0; i < nv; ++i) {
        if (free_mask && !free_mask[i]) continue;
        for (int a = 0; a < 3; ++a) {
            double acc = (f[3 * i + a] + mass[i] * g[a]) / mass[i];
            u[3 * i + a] += v[3 * i + a] * h + 0.5 * acc * h * h;
            v[3 * i + a] += acc * h;
        }
    }
}

/* ------------------------------------------------------------------ */
/* O9  implicit (linearised backward Euler) system:        */
/*   A = M + h D + h^2 K,  D = alpha M + beta K                          */
/*   b = h (f + M g - D v - h K v)                                       */
/* M is lumped (m_v I on the self-loop row of v).                        */
/* ------------------------------------------------------------------ */
void orc_implicit_assemble(int64_t nv, const int64_t* row_ptr, const int64_t* head,
                           const double* K, const double* mass, const double* f, const double* vel,
                           double h, double alpha, double beta, const double* g,
                           double* A, double* b) {
    int64_t ne = row_ptr[nv];
    double* Kv = (double*)malloc(sizeof(double) * (size_t)(3 * nv > 0 ? 3 * nv : 1));
    orc_edge_matvec(nv, row_ptr, head, K, vel, Kv);
    for (int64_t i = 0; i < nv; ++i)
        for (int a = 0; a < 3; ++a) {
            double Mv = mass[i] * vel[3 * i + a];
            double Dv = alpha * Mv + beta * Kv[3 * i + a];
            b[3 * i + a] = h * (f[3 * i + a] + mass[i] * g[a] - Dv - h * Kv[3 * i + a]);
        }
    free(Kv);
    for (int64_t v = 0; v < nv; ++v)
        for (int64_t r = row_ptr[v]; r < row_ptr[v + 1]; ++r)
            for (int a = 0; a < 3; ++a)
                for (int c = 0; c < 3; ++c) {
                    double Me = (head[r] == v && a == c) ? mass[v] : 0.0;
                    double Ke = K[9 * r + 3 * a + c];
                    double De = alpha * Me + beta * Ke;
                    A[9 * r + 3 * a + c] = Me + h * De + h * h * Ke;
                }
    (void)ne;
}

/* ------------------------------------------------------------------ */
/* Consistent mass on the edge relation (SURVEY §8(c) "Mass matrix":      */
/* "Consistent mass (on edges) is NEXT"; §8(f) 1).  The Galerkin mass of  */
/* linear tets, M_ij = rho * integral(N_i N_j) = rho W (1 + delta_ij)/20   */
/* (textbook; the paper names only a "mass" field), is   */
/* a scalar times I_3 per edge row: mass_e[e[i][j]] += rho W (1+d_ij)/20,  */
/* tets ascending, (i, j) row-major.                                       */
/* ------------------------------------------------------------------ */
void orc_consistent_mass(int64_t nt, const int64_t* e, const double* W, double rho, int64_t ne,
                         double* mass_e) {
    for (int64_t r = 0; r < ne; ++r) mass_e[r] = 0.0;
    for (int64_t t = 0; t < nt; ++t)
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j)
                mass_e[e[16 * t + 4 * i + j]] += rho * W[t] * (i == j ? 2.0 : 1.0) / 20.0;
}

/* O9 with the consistent mass: M is the edge-relation matrix mass_e[r] I_3,
 * so M v and M g are edge query-loops like K v:
 *   A_r = M_r + h (alpha M_r + beta K_r) + h^2 K_r,
 *   b   = h (f + M g - (alpha M v + beta K v) - h K v). */
void orc_implicit_assemble_consistent(int64_t nv, const int64_t* row_ptr, const int64_t* head,
                                      const double* K, const double* mass_e, const double* f,
                                      const double* vel, double h, double alpha, double beta,
                                      const double* g, double* A, double* b) {
    double* Kv = (double*)malloc(sizeof(double) * (size_t)(3 * nv > 0 ? 3 * nv : 1));
    orc_edge_matvec(nv, row_ptr, head, K, vel, Kv);
    for (int64_t v = 0; v < nv; ++v) {
        double Mv[3] = {0.0, 0.0, 0.0}, msum = 0.0;
        for (int64_t r = row_ptr[v]; r < row_ptr[v + 1]; ++r) {
            for (int a = 0; a < 3; ++a) Mv[a] += mass_e[r] * vel[3 * head[r] + a];
            msum += mass_e[r];
        }
        for (int a = 0; a < 3; ++a) {
            double Dv = alpha * Mv[a] + beta * Kv[3 * v + a];
            b[3 * v + a] = h * (f[3 * v + a] + msum * g[a] - Dv - h * Kv[3 * v + a]);
        }
    }
    free(Kv);
    for (int64_t v = 0; v < nv; ++v)
        for (int64_t r = row_ptr[v]; r < row_ptr[v + 1]; ++r)
            for (int a = 0; a < 3; ++a)
                for (int c = 0; c < 3; ++c) {
                    double Me = (a == c) ? mass_e[r] : 0.0;
                    double Ke = K[9 * r + 3 * a + c];
                    double De = alpha * Me + beta * Ke;
                    A[9 * r + 3 * a + c] = Me + h * De + h * h * Ke;
                }
}

/* ------------------------------------------------------------------ */
/* Newton iterations of the backward-Euler step (SURVEY §8(f) 1 "multiple */
/* Newton iterations"; the paper names only "implicit backward Euler",    */
/* P:941).  Unknown x = u_{n+1}, velocity w = (x - u_n)/h; residual        */
/*   G(x) = M (w - v_n)/h - f(x) - M g + D w,                              */
/* Jacobian dG/dx = (M + h D + h^2 K(x)) / h^2.  The first Newton step from */
/* x = u_n is exactly the one-linearisation step O9; the     */
/* later ones solve (M + h D + h^2 K(x_k)) dw = -h G(x_k), i.e.             */
/*   b = h (f(x_k) + M g - D w_k) + M (v_n - w_k),                         */
/* then w += dw, x += h dw.  M is given per edge row (mass_e[r] I_3; a      */
/* lumped mass is the self rows only), D = alpha M + beta K(x_k).           */
/* ------------------------------------------------------------------ */
void orc_newton_rhs(int64_t nv, const int64_t* row_ptr, const int64_t* head, const double* K,
                    const double* mass_e, const double* f, const double* w, const double* v0, double h,
                    double alpha, double beta, const double* g, double* b) {
    for (int64_t v = 0; v < nv; ++v) {
        double Kw[3] = {0.0, 0.0, 0.0}, Mw[3] = {0.0, 0.0, 0.0}, Mv0[3] = {0.0, 0.0, 0.0}, msum = 0.0;
        for (int64_t r = row_ptr[v]; r < row_ptr[v + 1]; ++r) {
            const int64_t hd = head[r];
            for (int a = 0; a < 3; ++a) {
                for (int c = 0; c < 3; ++c) Kw[a] += K[9 * r + 3 * a + c] * w[3 * hd + c];
                Mw[a] += mass_e[r] * w[3 * hd + a];
                Mv0[a] += mass_e[r] * v0[3 * hd + a];
            }
            msum += mass_e[r];
        }
        for (int a = 0; a < 3; ++a) {
            double Dw = alpha * Mw[a] + beta * Kw[a];
            b[3 * v + a] = h * (f[3 * v + a] + msum * g[a] - Dw) + (Mv0[a] - Mw[a]);
        }
    }
}

/* ------------------------------------------------------------------ */
/* O10  Jacobi-preconditioned CG (Saad Alg. 9.1), fixed N iters,  */
/* Dirichlet projection by the free mask (subsets).           */
/* Readings: alpha = 0 if p.q == 0, beta = 0 if rho == 0.    */
/* rho_hist (nullable, iters+1): rho before each iteration and at end.   */
/* returns 1 if some p.q < 0 (A not SPD on the Krylov space), else 0.     */
/* ------------------------------------------------------------------ */
int orc_pcg(int64_t nv, const int64_t* row_ptr, const int64_t* head, const double* A,
            const double* b, const uint8_t* free_mask, int iters, double* x, double* rho_hist) {
    int64_t n = 3 * nv;
    double* r = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    double* z = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    double* p = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    double* q = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    double* d = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    int not_spd = 0;
    for (int64_t v = 0; v < nv; ++v)
        for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e)
            if (head[e] == v)
                for (int a = 0; a < 3; ++a) d[3 * v + a] = A[9 * e + 4 * a];
    for (int64_t i = 0; i < n; ++i) {
        x[i] = 0.0;
        double m = (free_mask && !free_mask[i / 3]) ? 0.0 : 1.0;
        r[i] = b[i] * m;
        z[i] = (m != 0.0) ? r[i] / d[i] : 0.0;
        p[i] = z[i];
    }
    double rho = orc_dot(n, r, z);
    for (int k = 0; k < iters; ++k) {
        if (rho_hist) rho_hist[k] = rho;
        orc_edge_matvec(nv, row_ptr, head, A, p, q);
        if (free_mask)
            for (int64_t i = 0; i < n; ++i)
                if (!free_mask[i / 3]) q[i] = 0.0;
        double pq = orc_dot(n, p, q);
        if (pq < 0.0) not_spd = 1;
        double alpha = (pq != 0.0) ? rho / pq : 0.0;
        for (int64_t i = 0; i < n; ++i) {
            x[i] += alpha * p[i];
            r[i] -= alpha * q[i];
            double m = (free_mask && !free_mask[i / 3]) ? 0.0 : 1.0;
            z[i] = (m != 0.0) ? r[i] / d[i] : 0.0;
        }
        double rho_new = orc_dot(n, r, z);
        double beta = (rho != 0.0) ? rho_new / rho : 0.0;
        for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        rho = rho_new;
    }
    if (rho_hist) rho_hist[iters] = rho;
    free(r); free(z); free(p); free(q); free(d);
    return not_spd;
}

/* implicit step state update: v += dv; u += h v (P:941 integrator) */
void orc_implicit_update(int64_t nv, const double* dv, double h, double* u, double* v) {
    for (int64_t i = 0; i < 3 * nv; ++i) {
        v[i] += dv[i];
        u[i] += h * v[i];
    }
}

/* ------------------------------------------------------------------ */
/* Fig. 2 spring-mass program, kernel by      */
/* kernel, over the grouped edge relation (v.edges = rows of v):   */
/*   initLen(e):               rest_len = |head.pos - tail.pos|           */
/*   computeInternalForces(v): for e in v.edges: dq = e.head.q - v.q,     */
/*                             dir = normalize(dq),                        */
/*                             v.force += K (e.rest_len dir - dq)          */
/*   applyForces(v):           qdd = force/mass; q += qd dt + 0.5 qdd dt^2;*/
/*                             qd += qdd dt; force = 0                     */
/*   measureTotalEnergy(v):    E += 0.5 mass qd.qd                         */
/* Reading: normalize(0) = 0, so a self-loop row adds 0.   */
/* ------------------------------------------------------------------ */
void orc_spring_init_len(int64_t ne, const int64_t* tail, const int64_t* head, const double* pos,
                         double* rest_len) {
    for (int64_t e = 0; e < ne; ++e) {
        double d[3];
        for (int a = 0; a < 3; ++a) d[a] = pos[3 * head[e] + a] - pos[3 * tail[e] + a];
        rest_len[e] = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    }
}

void orc_spring_forces(int64_t nv, const int64_t* row_ptr, const int64_t* head, const double* q,
                       const double* rest_len, double K, double* force) {
    for (int64_t v = 0; v < nv; ++v)
        for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
            double dq[3], dir[3];
            for (int a = 0; a < 3; ++a) dq[a] = q[3 * head[e] + a] - q[3 * v + a];
            double len = sqrt(dq[0] * dq[0] + dq[1] * dq[1] + dq[2] * dq[2]);
            for (int a = 0; a < 3; ++a) dir[a] = len > 0.0 ? dq[a] / len : 0.0;
            for (int a = 0; a < 3; ++a) force[3 * v + a] += K * (rest_len[e] * dir[a] - dq[a]);
        }
}

void orc_spring_apply(int64_t nv, const double* mass, double dt, double* q, double* qd, double* force) {
    for (int64_t v = 0; v < nv; ++v)
        for (int a = 0; a < 3; ++a) {
            double qdd = force[3 * v + a] / mass[v];
            q[3 * v + a] += qd[3 * v + a] * dt + 0.5 * qdd * dt * dt;
            qd[3 * v + a] += qdd * dt;
            force[3 * v + a] = 0.0;
        }
}

double orc_kinetic_energy(int64_t nv, const double* mass, const double* qd) {
    double E = 0.0;
    for (int64_t v = 0; v < nv; ++v)
        E += 0.5 * mass[v] * (qd[3 * v] * qd[3 * v] + qd[3 * v + 1] * qd[3 * v + 1] + qd[3 * v + 2] * qd[3 * v + 2]);
    return E;
}

/* ------------------------------------------------------------------ */
/* Regular 2-D grid domain (P:733-772 affine indexing; Fig. 3   */
/* particle coupling).  nx x ny unit cells, cell (i, j)    */
/* = [i, i+1) x [j, j+1), row-major id i + nx j, periodic (Stable Fluids).  */
/* Dual cell (a, b) spans the cell centres (a+.5 .. a+1.5, b+.5 .. b+1.5);  */
/* dual_cell.cell(dx, dy) = cell(a + dx, b + dy) (the affine map {{1,0,dx},*/
/* {0,1,dy}}).  Readings: DESIGN.md §3 (22).                    */
/* ------------------------------------------------------------------ */
static int64_t orc_wrap(int64_t i, int64_t n) { int64_t r = i % n; return r < 0 ? r + n : r; }

/* out[c] = sum_k w_k in[cell(i + dx_k, j + dy_k)], per component */
void orc_grid2_stencil(int64_t nx, int64_t ny, int comps, const double* in, double* out, int npts,
                       const int64_t* off, const double* w) {
    for (int64_t j = 0; j < ny; ++j)
        for (int64_t i = 0; i < nx; ++i)
            for (int a = 0; a < comps; ++a) {
                double s = 0.0;
                for (int k = 0; k < npts; ++k)
                    s += w[k] * in[comps * (orc_wrap(i + off[2 * k], nx) + nx * orc_wrap(j + off[2 * k + 1], ny)) + a];
                out[comps * (i + nx * j) + a] = s;
            }
}

/* PointLocate: the dual cell containing (x, y) */
void orc_grid2_point_locate(int64_t nx, int64_t ny, int64_t np, const double* pos, int64_t* dual) {
    for (int64_t p = 0; p < np; ++p) {
        int64_t a = (int64_t)floor(pos[3 * p] - 0.5), b = (int64_t)floor(pos[3 * p + 1] - 0.5);
        dual[p] = orc_wrap(a, nx) + nx * orc_wrap(b, ny);
    }
}

/* update_particle_vel (Fig. 3): x1 = frac(x - 0.5), y1 = frac(y - 0.5),
 * vel = x0 y0 cell(0,0) + x1 y0 cell(1,0) + x0 y1 cell(0,1) + x1 y1 cell(1,1) */
void orc_grid2_particle_vel(int64_t nx, int64_t ny, int comps, const double* cell_vel, int64_t np,
                            const double* pos, const int64_t* dual, double* vel) {
    for (int64_t p = 0; p < np; ++p) {
        double x1 = (pos[3 * p] - 0.5) - floor(pos[3 * p] - 0.5);
        double y1 = (pos[3 * p + 1] - 0.5) - floor(pos[3 * p + 1] - 0.5);
        double x0 = 1.0 - x1, y0 = 1.0 - y1;
        int64_t a = dual[p] % nx, b = dual[p] / nx;
        int64_t c00 = a + nx * b, c10 = orc_wrap(a + 1, nx) + nx * b;
        int64_t c01 = a + nx * orc_wrap(b + 1, ny), c11 = orc_wrap(a + 1, nx) + nx * orc_wrap(b + 1, ny);
        for (int k = 0; k < comps; ++k)
            vel[comps * p + k] = x0 * y0 * cell_vel[comps * c00 + k] + x1 * y0 * cell_vel[comps * c10 + k]
                               + x0 * y1 * cell_vel[comps * c01 + k] + x1 * y1 * cell_vel[comps * c11 + k];
    }
}
