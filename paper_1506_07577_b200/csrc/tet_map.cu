// tet_map.cu -- the element map over the tets relation.
//
// Per tet (P:941-946 Vega StVK, P:975-980 neo-Hookean "specialized"):
//   gather u[v[k]] through the key-field tets.v,
//   H = Du Dminv, F = I + H (displacement form: no cancellation in fp32),
//   first Piola stress P and energy density Psi (StVK or compressible NH),
//   f_i = -W P g_i (i = 1..3), f_0 = -(f_1 + f_2 + f_3),
//   K_ij = d^2(W Psi)/dx_i dx_j by the closed rank-1 forms of DESIGN.md §5:
//     NH   K_ij = W [mu m_ij I + c1 k_j k_i^T + lam k_i k_j^T],  k_i = F^-T g_i
//     StVK K_ij = W [s_ij I + mu m_ij F F^T + mu h_j h_i^T + lam h_i h_j^T], h_i = F g_i
//   and reduces f[v[i]] += f_i, K[e[i][j]] += K_ij (field `+=`) and
//   energy += W Psi (global `+=`, fused two-pass).
// The oracle computes the same quantities by the textbook F-form and a generic
// 4th-order tensor contraction (oracle/ebb_oracle.c); the two share no code.
#include "ebb_internal.cuh"
#include "reduce.cuh"

using namespace ebb;

namespace {

template <typename R>
struct M3 {
    R m[3][3];
};

template <typename R>
__device__ __forceinline__ void red_add(R* p, R v) {
    atomicAdd(p, v);  // result unused -> REDG.E.ADD
}

template <typename R, int MODEL, bool WANT_K, bool WANT_E>
__global__ void __launch_bounds__(128) k_tet_map(uint64_t nt, const uint4* __restrict__ tv,
                                                 const uint4* __restrict__ te, const R* __restrict__ u,
                                                 const R* __restrict__ Dminv, const R* __restrict__ Wt,
                                                 const R* __restrict__ mu_t, const R* __restrict__ lam_t,
                                                 R* __restrict__ f, R* __restrict__ K, uint64_t ne,
                                                 double* __restrict__ partials, unsigned int* __restrict__ counter,
                                                 R* __restrict__ energy, unsigned long long* __restrict__ err) {
    double e_acc = 0.0;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nt; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 vv = tv[t];
        const uint32_t v[4] = {vv.x, vv.y, vv.z, vv.w};
        R uu[4][3];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int a = 0; a < 3; ++a) uu[k][a] = u[3ull * v[k] + a];
        // g_i = row i-1 of Dm^-1 (i = 1..3), component-planar storage
        R g[4][3];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) g[r + 1][c] = Dminv[(uint64_t)(3 * r + c) * nt + t];
#pragma unroll
        for (int c = 0; c < 3; ++c) g[0][c] = -(g[1][c] + g[2][c] + g[3][c]);
        const R W = Wt[t], mu = mu_t[t], lam = lam_t[t];
        // H = Du Dm^-1,  Du = [u1-u0, u2-u0, u3-u0]
        R H[3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                R s = 0;
#pragma unroll
                for (int k = 0; k < 3; ++k) s += (uu[k + 1][a] - uu[0][a]) * g[k + 1][b];
                H[a][b] = s;
            }
        R P[3][3];
        R psi;
        // model-specific state kept for the stiffness
        R S[3][3];     // StVK second Piola stress
        R FiT[3][3];   // NH F^-T
        R c1 = 0;      // NH mu - lam ln J
        if (MODEL == EBB_STVK) {
            // E = 1/2 (H + H^T + H^T H), S = 2 mu E + lam tr(E) I, P = (I + H) S
            R E[3][3];
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) {
                    R hh = H[0][a] * H[0][b] + H[1][a] * H[1][b] + H[2][a] * H[2][b];
                    E[a][b] = R(0.5) * (H[a][b] + H[b][a] + hh);
                }
            R trE = E[0][0] + E[1][1] + E[2][2];
            R EE = 0;
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) {
                    S[a][b] = R(2) * mu * E[a][b] + (a == b ? lam * trE : R(0));
                    EE += E[a][b] * E[a][b];
                }
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) P[a][b] = S[a][b] + H[a][0] * S[0][b] + H[a][1] * S[1][b] + H[a][2] * S[2][b];
            psi = mu * EE + R(0.5) * lam * trE * trE;
        } else {
            // cancellation-free invariants of F = I + H (App. B of SURVEY.md)
            R t1 = H[0][0] + H[1][1] + H[2][2];
            R H2[3][3];
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) H2[a][b] = H[a][0] * H[0][b] + H[a][1] * H[1][b] + H[a][2] * H[2][b];
            R trH2 = H2[0][0] + H2[1][1] + H2[2][2];
            R s2 = R(0.5) * (t1 * t1 - trH2);
            R dH = H[0][0] * (H[1][1] * H[2][2] - H[1][2] * H[2][1]) - H[0][1] * (H[1][0] * H[2][2] - H[1][2] * H[2][0]) +
                   H[0][2] * (H[1][0] * H[2][1] - H[1][1] * H[2][0]);
            R delta = t1 + s2 + dH;  // J - 1
            R J = R(1) + delta;
            if (!(J > R(0))) atomicAdd(&err[ERR_INVERTED], 1ull);
            R lnJ = log1p(delta);
            R invJ = R(1) / J;
            // adj(F) = (1 + t + s2) I - (1 + t) H + H^2 ;  cof F = adj^T ; F^-T = cof/J
            R ca = R(1) + t1 + s2, cb = R(1) + t1;
            R cof[3][3];
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) cof[a][b] = (a == b ? ca : R(0)) - cb * H[b][a] + H2[b][a];
            // J F - cof F = det(H) I + (1 + delta) H + (1 + t) H^T - (H^T)^2
            R HF2 = 0;
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) {
                    R jf = (a == b ? dH : R(0)) + J * H[a][b] + cb * H[b][a] - H2[b][a];
                    P[a][b] = (mu * jf + lam * lnJ * cof[a][b]) * invJ;
                    FiT[a][b] = cof[a][b] * invJ;
                    HF2 += H[a][b] * H[a][b];
                }
            c1 = mu - lam * lnJ;
            // tr(F^T F) - 3 = 2 tr H + |H|^2
            psi = R(0.5) * mu * (R(2) * t1 + HF2) - mu * lnJ + R(0.5) * lam * lnJ * lnJ;
        }
        // forces
        R fi[4][3];
#pragma unroll
        for (int a = 0; a < 3; ++a) fi[0][a] = 0;
#pragma unroll
        for (int i = 1; i < 4; ++i)
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                fi[i][a] = -W * (P[a][0] * g[i][0] + P[a][1] * g[i][1] + P[a][2] * g[i][2]);
                fi[0][a] -= fi[i][a];
            }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int a = 0; a < 3; ++a) red_add(&f[3ull * v[i] + a], fi[i][a]);
        if (WANT_E) e_acc += (double)(W * psi);
        if (WANT_K) {
            uint32_t row[16];
            const uint4* tep = te + 4 * t;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint4 r4 = tep[q];
                row[4 * q + 0] = r4.x;
                row[4 * q + 1] = r4.y;
                row[4 * q + 2] = r4.z;
                row[4 * q + 3] = r4.w;
            }
            // per-corner vectors: NH k_i = F^-T g_i ; StVK h_i = F g_i
            R kv[4][3];
            R B[3][3];
            if (MODEL == EBB_NH) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int a = 0; a < 3; ++a) kv[i][a] = FiT[a][0] * g[i][0] + FiT[a][1] * g[i][1] + FiT[a][2] * g[i][2];
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int a = 0; a < 3; ++a)
                        kv[i][a] = g[i][a] + H[a][0] * g[i][0] + H[a][1] * g[i][1] + H[a][2] * g[i][2];
                // B = F F^T
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int b = 0; b < 3; ++b) {
                        R s = 0;
#pragma unroll
                        for (int c = 0; c < 3; ++c) s += ((a == c ? R(1) : R(0)) + H[a][c]) * ((b == c ? R(1) : R(0)) + H[b][c]);
                        B[a][b] = s;
                    }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                R Sg[3];
                if (MODEL == EBB_STVK) {
#pragma unroll
                    for (int a = 0; a < 3; ++a) Sg[a] = S[a][0] * g[i][0] + S[a][1] * g[i][1] + S[a][2] * g[i][2];
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    R mij = g[i][0] * g[j][0] + g[i][1] * g[j][1] + g[i][2] * g[j][2];
                    R* Kr = K + row[4 * i + j];
                    if (MODEL == EBB_NH) {
                        R d = W * mu * mij, cc = W * c1, cl = W * lam;
#pragma unroll
                        for (int a = 0; a < 3; ++a)
#pragma unroll
                            for (int b = 0; b < 3; ++b) {
                                R val = cc * kv[j][a] * kv[i][b] + cl * kv[i][a] * kv[j][b] + (a == b ? d : R(0));
                                red_add(Kr + (uint64_t)(3 * a + b) * ne, val);
                            }
                    } else {
                        R sij = Sg[0] * g[j][0] + Sg[1] * g[j][1] + Sg[2] * g[j][2];
                        R d = W * sij, cm = W * mu * mij, ch = W * mu, cl = W * lam;
#pragma unroll
                        for (int a = 0; a < 3; ++a)
#pragma unroll
                            for (int b = 0; b < 3; ++b) {
                                R val = cm * B[a][b] + ch * kv[j][a] * kv[i][b] + cl * kv[i][a] * kv[j][b] +
                                        (a == b ? d : R(0));
                                red_add(Kr + (uint64_t)(3 * a + b) * ne, val);
                            }
                    }
                }
            }
        }
    }
    if (WANT_E) {
        double tot;
        if (block_sum_last_done(e_acc, partials, counter, &tot)) *energy = (R)((double)*energy + tot);
    }
}

template <typename R, int MODEL>
ebb_status launch_map(Ctx* c, bool want_k, bool want_e, uint64_t nt, const Field* V, const Field* Ef, const Field* U,
                      const Field* D, const Field* W, const Field* MU, const Field* LA, const Field* Fo, const Field* Ko,
                      uint64_t ne, const Field* En, cudaStream_t s) {
    const int block = 128;
    unsigned grid = grid_for(nt, block);
    unsigned cap = (unsigned)c->num_sms * 8;
    if (grid > cap) grid = cap;
    KernelTimer kt(c, EBB_K_TET_MAP, s);
#define EBB_ARGS                                                                                               \
    nt, (const uint4*)V->ptr, Ef ? (const uint4*)Ef->ptr : nullptr, (const R*)U->ptr, (const R*)D->ptr,         \
        (const R*)W->ptr, (const R*)MU->ptr, (const R*)LA->ptr, (R*)Fo->ptr, Ko ? (R*)Ko->ptr : nullptr, ne,      \
        c->d_partials, c->d_counter + 0, En ? (R*)En->ptr : nullptr, c->d_err
    if (want_k && want_e) k_tet_map<R, MODEL, true, true><<<grid, block, 0, s>>>(EBB_ARGS);
    else if (want_k) k_tet_map<R, MODEL, true, false><<<grid, block, 0, s>>>(EBB_ARGS);
    else if (want_e) k_tet_map<R, MODEL, false, true><<<grid, block, 0, s>>>(EBB_ARGS);
    else k_tet_map<R, MODEL, false, false><<<grid, block, 0, s>>>(EBB_ARGS);
#undef EBB_ARGS
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

}  // namespace

extern "C" ebb_status ebb_map_tet_forces(ebb_ctx ctx, const ebb_tet_map_desc* d, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    if (!c || !d) return fail(c, EBB_E_ARG, "null argument");
    if (d->model != EBB_STVK && d->model != EBB_NH) return fail(c, EBB_E_ARG, "unknown model %d", d->model);
    Field* V = get_field(c, d->v);
    Field* U = get_field(c, d->u);
    Field* D = get_field(c, d->Dminv);
    Field* W = get_field(c, d->W);
    Field* MU = get_field(c, d->mu);
    Field* LA = get_field(c, d->lam);
    Field* Fo = get_field(c, d->f);
    Field* Ko = d->K == EBB_NONE ? nullptr : get_field(c, d->K);
    Field* Ef = d->K == EBB_NONE ? nullptr : get_field(c, d->e);
    Field* En = d->energy == EBB_NONE ? nullptr : get_field(c, d->energy);
    if (!V || !U || !D || !W || !MU || !LA || !Fo) return fail(c, EBB_E_ARG, "map_tet_forces: bad field handle");
    if ((d->K != EBB_NONE && (!Ko || !Ef)) || (d->energy != EBB_NONE && !En))
        return fail(c, EBB_E_ARG, "map_tet_forces: bad optional field handle");
    // relational typing: v : tets -> verts, e : tets -> edges
    if (V->dtype != EBB_KEY || V->comps() != 4) return fail(c, EBB_E_TYPE, "v must be a 4x1 key-field");
    ebb_rel tets = V->rel, verts = V->key_target;
    uint64_t nt = c->rels[tets].size;
    ebb_dtype dt = U->dtype;
    if (dt != EBB_F32 && dt != EBB_F64) return fail(c, EBB_E_TYPE, "u must be F32 or F64");
    auto chk = [&](Field* F, ebb_rel rel, uint32_t comps, ebb_layout lay, const char* what) -> ebb_status {
        if (F->rel != rel || F->comps() != comps || F->dtype != dt || (comps > 1 && F->layout != lay))
            return fail(c, EBB_E_TYPE, "map_tet_forces: field '%s' (%s) has wrong relation/shape/dtype/layout",
                        F->name.c_str(), what);
        return EBB_OK;
    };
    EBB_TRY(chk(U, verts, 3, EBB_AOS, "u"));
    EBB_TRY(chk(Fo, verts, 3, EBB_AOS, "f"));
    EBB_TRY(chk(D, tets, 9, EBB_SOA, "Dminv"));
    EBB_TRY(chk(W, tets, 1, EBB_AOS, "W"));
    EBB_TRY(chk(MU, tets, 1, EBB_AOS, "mu"));
    EBB_TRY(chk(LA, tets, 1, EBB_AOS, "lam"));
    uint64_t ne = 0;
    if (Ko) {
        if (Ef->dtype != EBB_KEY || Ef->comps() != 16 || Ef->rel != tets)
            return fail(c, EBB_E_TYPE, "e must be a 4x4 key-field on tets");
        EBB_TRY(chk(Ko, Ef->key_target, 9, EBB_SOA, "K"));
        ne = c->rels[Ko->rel].size;
    }
    if (En && (!En->is_global || En->dtype != dt)) return fail(c, EBB_E_TYPE, "energy must be a global of the map dtype");
    // phase discipline: read-only fields must not alias reduce targets
    if (U->ptr == Fo->ptr || (Ko && (U->ptr == Ko->ptr || Fo->ptr == Ko->ptr)))
        return fail(c, EBB_E_PHASE, "map_tet_forces: a field is used in two phases (read and reduce)");
    cudaStream_t s = (cudaStream_t)stream;
    if (d->zero_outputs) {
        EBB_CUDA(c, cudaMemsetAsync(Fo->ptr, 0, c->rels[verts].size * 3 * dtype_size(dt), s));
        if (Ko) EBB_CUDA(c, cudaMemsetAsync(Ko->ptr, 0, ne * 9 * dtype_size(dt), s));
        if (En) EBB_CUDA(c, cudaMemsetAsync(En->ptr, 0, dtype_size(dt), s));
    }
    bool wk = Ko != nullptr, we = En != nullptr;
    if (dt == EBB_F64) {
        if (d->model == EBB_NH) return launch_map<double, EBB_NH>(c, wk, we, nt, V, Ef, U, D, W, MU, LA, Fo, Ko, ne, En, s);
        return launch_map<double, EBB_STVK>(c, wk, we, nt, V, Ef, U, D, W, MU, LA, Fo, Ko, ne, En, s);
    }
    if (d->model == EBB_NH) return launch_map<float, EBB_NH>(c, wk, we, nt, V, Ef, U, D, W, MU, LA, Fo, Ko, ne, En, s);
    return launch_map<float, EBB_STVK>(c, wk, we, nt, V, Ef, U, D, W, MU, LA, Fo, Ko, ne, En, s);
}
