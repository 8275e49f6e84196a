// ebe.cu -- matrix-free element-by-element stiffness matvec:
// q = sum_t K_t p_t from a compact per-tet stiffness state instead of the
// assembled edge-relation matrix (K = sum_t K_t stored on edges e[i][j],
// P:806; the matvec is the same quantity summed per element).
//
// State (SOA planes on the tets, written by ebb_tet_stiffness_state from u):
//   NH   (15): k_i = F^-T g_i (12), W mu, W c1, W lam
//   StVK (26): h_i = F g_i (12), W S (6: 00 01 02 11 12 22), W mu F F^T (6), W mu, W lam
// Per tet, with C = sum_j p_j g_j^T, B = sum_j k_j p_j^T, s = sum_j k_j . p_j
// (rank-1 closed forms of element.cuh summed over j):
//   NH   y_i = W mu C g_i + W c1 B k_i + W lam s k_i
//   StVK y_i = C (W S g_i) + (W mu F F^T)(C g_i) + W mu B h_i + W lam s h_i
// and q[v_i] += y_i by fp64/fp32 red.global.add (the field `+=` of P:885).
#include "ebb_internal.cuh"
#include "element.cuh"

namespace ebb {
namespace {

template <int MODEL>
constexpr int ebe_words() { return MODEL == EBB_NH ? 15 : 26; }

template <typename R, int MODEL>
__global__ void __launch_bounds__(128) k_tet_state(uint64_t nt, const uint4* __restrict__ tv, const R* __restrict__ u,
                                                   const R* __restrict__ Dminv, const R* __restrict__ Wt,
                                                   const R* __restrict__ mu_t, const R* __restrict__ lam_t,
                                                   R* __restrict__ state, unsigned long long* __restrict__ err) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const uint4 vv = tv[t];
    const uint32_t v[4] = {vv.x, vv.y, vv.z, vv.w};
    R uu[4][3];
    TetState<R> st;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int a = 0; a < 3; ++a) uu[i][a] = u[3ull * v[i] + a];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) st.g[r + 1][c] = Dminv[(uint64_t)(3 * r + c) * nt + t];
#pragma unroll
    for (int c = 0; c < 3; ++c) st.g[0][c] = -(st.g[1][c] + st.g[2][c] + st.g[3][c]);
    st.W = Wt[t];
    st.mu = mu_t[t];
    st.lam = lam_t[t];
    tet_physics<R, MODEL, true>(uu, st);
    if (MODEL == EBB_NH && !(st.J > R(0))) atomicAdd(&err[ERR_INVERTED], 1ull);
    R* o = state + t;
    int w = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int a = 0; a < 3; ++a) o[(uint64_t)(w++) * nt] = st.kv[i][a];
    if constexpr (MODEL == EBB_NH) {
        o[(uint64_t)(w++) * nt] = st.W * st.mu;
        o[(uint64_t)(w++) * nt] = st.W * st.c1;
        o[(uint64_t)(w++) * nt] = st.W * st.lam;
    } else {
        constexpr int sa[6] = {0, 0, 0, 1, 1, 2}, sb[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
        for (int k = 0; k < 6; ++k) o[(uint64_t)(w++) * nt] = st.W * st.S[sa[k]][sb[k]];
#pragma unroll
        for (int k = 0; k < 6; ++k) o[(uint64_t)(w++) * nt] = st.W * st.mu * st.B[sa[k]][sb[k]];
        o[(uint64_t)(w++) * nt] = st.W * st.mu;
        o[(uint64_t)(w++) * nt] = st.W * st.lam;
    }
}

template <typename R, int MODEL>
__global__ void __launch_bounds__(128) k_ebe_matvec(uint64_t nt, const uint4* __restrict__ tv,
                                                    const R* __restrict__ Dminv, const R* __restrict__ state,
                                                    const R* __restrict__ p, R* __restrict__ q) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const uint4 vv = tv[t];
    const uint32_t v[4] = {vv.x, vv.y, vv.z, vv.w};
    R g[4][3], k[4][3], pj[4][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) g[r + 1][c] = Dminv[(uint64_t)(3 * r + c) * nt + t];
#pragma unroll
    for (int c = 0; c < 3; ++c) g[0][c] = -(g[1][c] + g[2][c] + g[3][c]);
    const R* s_ = state + t;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            k[i][a] = s_[(uint64_t)(3 * i + a) * nt];
            pj[i][a] = p[3ull * v[i] + a];
        }
    // C = sum_j p_j g_j^T, B = sum_j k_j p_j^T, s = sum_j k_j . p_j
    R C[3][3], B[3][3], s = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            C[a][b] = pj[0][a] * g[0][b] + pj[1][a] * g[1][b] + pj[2][a] * g[2][b] + pj[3][a] * g[3][b];
            B[a][b] = k[0][a] * pj[0][b] + k[1][a] * pj[1][b] + k[2][a] * pj[2][b] + k[3][a] * pj[3][b];
        }
#pragma unroll
    for (int j = 0; j < 4; ++j) s += k[j][0] * pj[j][0] + k[j][1] * pj[j][1] + k[j][2] * pj[j][2];
    if constexpr (MODEL == EBB_NH) {
        const R wm = s_[12 * nt], wc = s_[13 * nt], wl = s_[14 * nt];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const R cg = C[a][0] * g[i][0] + C[a][1] * g[i][1] + C[a][2] * g[i][2];
                const R bk = B[a][0] * k[i][0] + B[a][1] * k[i][1] + B[a][2] * k[i][2];
                atomicAdd(q + 3ull * v[i] + a, wm * cg + wc * bk + wl * s * k[i][a]);
            }
    } else {
        R WS[3][3], MB[3][3];
        constexpr int sa[6] = {0, 0, 0, 1, 1, 2}, sb[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
        for (int m = 0; m < 6; ++m) {
            WS[sa[m]][sb[m]] = WS[sb[m]][sa[m]] = s_[(uint64_t)(12 + m) * nt];
            MB[sa[m]][sb[m]] = MB[sb[m]][sa[m]] = s_[(uint64_t)(18 + m) * nt];
        }
        const R wm = s_[24 * nt], wl = s_[25 * nt];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            R sg[3], cg[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                sg[a] = WS[a][0] * g[i][0] + WS[a][1] * g[i][1] + WS[a][2] * g[i][2];
                cg[a] = C[a][0] * g[i][0] + C[a][1] * g[i][1] + C[a][2] * g[i][2];
            }
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const R t1 = C[a][0] * sg[0] + C[a][1] * sg[1] + C[a][2] * sg[2];
                const R t2 = MB[a][0] * cg[0] + MB[a][1] * cg[1] + MB[a][2] * cg[2];
                const R bk = B[a][0] * k[i][0] + B[a][1] * k[i][1] + B[a][2] * k[i][2];
                atomicAdd(q + 3ull * v[i] + a, t1 + t2 + wm * bk + wl * s * k[i][a]);
            }
        }
    }
}

struct EbeArgs {
    uint64_t nt = 0, nv = 0;
    Field *V = nullptr, *U = nullptr, *D = nullptr, *W = nullptr, *MU = nullptr, *LA = nullptr, *S = nullptr;
    ebb_dtype dt = EBB_F64;
};

ebb_status ebe_validate(Ctx* c, const ebb_tet_map_desc* d, ebb_field state, bool need_material, EbeArgs* a) {
    if (!c || !d) return EBB_E_ARG;
    if (d->model != EBB_STVK && d->model != EBB_NH) return fail(c, EBB_E_ARG, "ebe: unknown model %d", d->model);
    a->V = get_field(c, d->v);
    a->D = get_field(c, d->Dminv);
    a->S = get_field(c, state);
    if (!a->V || !a->D || !a->S) return fail(c, EBB_E_ARG, "ebe: bad field handle");
    if (a->V->dtype != EBB_KEY || a->V->comps() != 4) return fail(c, EBB_E_TYPE, "ebe: v must be a 4x1 key-field");
    const ebb_rel tets = a->V->rel;
    a->nt = c->rels[tets].size;
    a->nv = c->rels[a->V->key_target].size;
    a->dt = a->D->dtype;
    if (a->dt != EBB_F32 && a->dt != EBB_F64) return fail(c, EBB_E_TYPE, "ebe: F32 or F64 fields");
    if (a->D->rel != tets || a->D->comps() != 9 || a->D->layout != EBB_SOA)
        return fail(c, EBB_E_TYPE, "ebe: Dminv must be a SOA 3x3 field on tets");
    const uint32_t words = d->model == EBB_NH ? ebe_words<EBB_NH>() : ebe_words<EBB_STVK>();
    if (a->S->rel != tets || a->S->comps() != words || a->S->dtype != a->dt || (words > 1 && a->S->layout != EBB_SOA))
        return fail(c, EBB_E_TYPE, "ebe: state must be a SOA %ux1 field of the map dtype on tets (%s)", words,
                    d->model == EBB_NH ? "NH" : "StVK");
    if (need_material) {
        a->U = get_field(c, d->u);
        a->W = get_field(c, d->W);
        a->MU = get_field(c, d->mu);
        a->LA = get_field(c, d->lam);
        if (!a->U || !a->W || !a->MU || !a->LA) return fail(c, EBB_E_ARG, "ebe: bad u/W/mu/lam handle");
        if (a->U->rel != a->V->key_target || a->U->comps() != 3 || a->U->dtype != a->dt || a->U->layout != EBB_AOS)
            return fail(c, EBB_E_TYPE, "ebe: u must be an AOS vec3 field on the vertices");
        for (Field* F : {a->W, a->MU, a->LA})
            if (F->rel != tets || F->comps() != 1 || F->dtype != a->dt)
                return fail(c, EBB_E_TYPE, "ebe: W, mu, lam must be scalar fields on tets");
    }
    return EBB_OK;
}

}  // namespace
}  // namespace ebb

using namespace ebb;

extern "C" {

ebb_status ebb_tet_stiffness_state(ebb_ctx ctx, const ebb_tet_map_desc* d, ebb_field state, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    EbeArgs a;
    EBB_TRY(ebe_validate(c, d, state, true, &a));
    cudaStream_t s = (cudaStream_t)stream;
    c->launches++;
    if (a.nt) {
#define EBB_TS(R, MODEL)                                                                                            \
    k_tet_state<R, MODEL><<<grid_for(a.nt, 128), 128, 0, s>>>(a.nt, (const uint4*)a.V->ptr, (const R*)a.U->ptr,     \
                                                              (const R*)a.D->ptr, (const R*)a.W->ptr,               \
                                                              (const R*)a.MU->ptr, (const R*)a.LA->ptr,             \
                                                              (R*)a.S->ptr, c->d_err)
        if (a.dt == EBB_F64) {
            if (d->model == EBB_NH) EBB_TS(double, EBB_NH);
            else EBB_TS(double, EBB_STVK);
        } else {
            if (d->model == EBB_NH) EBB_TS(float, EBB_NH);
            else EBB_TS(float, EBB_STVK);
        }
#undef EBB_TS
    }
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status ebb_ebe_matvec(ebb_ctx ctx, const ebb_tet_map_desc* d, ebb_field state, ebb_field p, ebb_field q,
                          ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    EbeArgs a;
    EBB_TRY(ebe_validate(c, d, state, false, &a));
    Field* P = get_field(c, p);
    Field* Q = get_field(c, q);
    if (!P || !Q) return fail(c, EBB_E_ARG, "ebe_matvec: bad p/q");
    for (Field* F : {P, Q})
        if (F->rel != a.V->key_target || F->comps() != 3 || F->dtype != a.dt || F->layout != EBB_AOS)
            return fail(c, EBB_E_TYPE, "ebe_matvec: p, q must be AOS vec3 fields of the state dtype on the vertices");
    if (P->ptr == Q->ptr) return fail(c, EBB_E_PHASE, "ebe_matvec: q aliases p");
    cudaStream_t s = (cudaStream_t)stream;
    EBB_CUDA(c, cudaMemsetAsync(Q->ptr, 0, a.nv * 3 * dtype_size(a.dt), s));
    KernelTimer kt(c, EBB_K_EBE_MATVEC, s);
    if (a.nt) {
#define EBB_EM(R, MODEL)                                                                                            \
    k_ebe_matvec<R, MODEL><<<grid_for(a.nt, 128), 128, 0, s>>>(a.nt, (const uint4*)a.V->ptr, (const R*)a.D->ptr,    \
                                                               (const R*)a.S->ptr, (const R*)P->ptr, (R*)Q->ptr)
        if (a.dt == EBB_F64) {
            if (d->model == EBB_NH) EBB_EM(double, EBB_NH);
            else EBB_EM(double, EBB_STVK);
        } else {
            if (d->model == EBB_NH) EBB_EM(float, EBB_NH);
            else EBB_EM(float, EBB_STVK);
        }
#undef EBB_EM
    }
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

}  // extern "C"
