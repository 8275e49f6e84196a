// tet_map.cu -- the element map over the tets relation.
//
// Per tet (P:941-946 Vega StVK, P:975-980 neo-Hookean "specialized"): gather
// u[v[k]] through the key-field tets.v, element physics
// (element.cuh: displacement form + closed rank-1 stiffness), and the
// reductions f[v[i]] += f_i, K[e[i][j]] += K_ij (field `+=`) and
// energy += W Psi (global `+=`, fused two-pass).
//
// The entry point and the ATOMIC scatter strategy (SURVEY §8(a) "the +=
// strategies", chosen by measurement -- DESIGN.md §5.2): one thread per tet,
// red.global.add per value (the paper's field reductions, with native
// fp64 RED instead of Kepler CAS).  SEGMENTED (the default, seg_map.cu), CHUNK
// (chunk_map.cu) and COLOR (color_map.cu) live in their own files; TILED and
// GATHER (owner tiles with shared-memory atomics / warp-specialized rounds)
// were retired in round 2 after measuring slower than SEGMENTED everywhere.
// The oracle computes the same quantities by the textbook F-form and a generic
// 4th-order tensor contraction (oracle/ebb_oracle.c); the two share no code.
#include <cstdlib>

#include "ebb_internal.cuh"
#include "element.cuh"
#include "reduce.cuh"

using namespace ebb;

namespace {

template <typename R>
__device__ __forceinline__ void red_add(R* p, R v) {
    atomicAdd(p, v);  // result unused -> REDG.E.ADD
}

template <typename R>
__device__ __forceinline__ void load_tet(uint64_t t, uint64_t nt, const uint4* __restrict__ tv, const R* __restrict__ u,
                                         const R* __restrict__ Dminv, const R* __restrict__ Wt,
                                         const R* __restrict__ mu_t, const R* __restrict__ lam_t, uint32_t v[4],
                                         R uu[4][3], TetState<R>& st) {
    const uint4 vv = tv[t];
    v[0] = vv.x;
    v[1] = vv.y;
    v[2] = vv.z;
    v[3] = vv.w;
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int a = 0; a < 3; ++a) uu[k][a] = u[3ull * v[k] + a];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) st.g[r + 1][c] = Dminv[(uint64_t)(3 * r + c) * nt + t];
#pragma unroll
    for (int c = 0; c < 3; ++c) st.g[0][c] = -(st.g[1][c] + st.g[2][c] + st.g[3][c]);
    st.W = Wt[t];
    st.mu = mu_t[t];
    st.lam = lam_t[t];
}

// ---------------------------------------------------------------- ATOMIC
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
        uint32_t v[4];
        R uu[4][3];
        TetState<R> st;
        load_tet(t, nt, tv, u, Dminv, Wt, mu_t, lam_t, v, uu, st);
        tet_physics<R, MODEL, WANT_K>(uu, st);
        if (MODEL == EBB_NH && !(st.J > R(0))) atomicAdd(&err[ERR_INVERTED], 1ull);
        R fi[4][3];
        tet_forces(st, fi);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int a = 0; a < 3; ++a) red_add(&f[3ull * v[i] + a], fi[i][a]);
        if (WANT_E) e_acc += (double)(st.W * st.psi);
        if (WANT_K) {
            uint32_t row[16];
#pragma unroll
            for (int qd = 0; qd < 4; ++qd) {
                uint4 r4 = te[4 * t + qd];
                row[4 * qd + 0] = r4.x;
                row[4 * qd + 1] = r4.y;
                row[4 * qd + 2] = r4.z;
                row[4 * qd + 3] = r4.w;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    R Kb[3][3];
                    tet_block<R, MODEL>(st, i, j, Kb);
                    R* Kr = K + row[4 * i + j];
#pragma unroll
                    for (int a = 0; a < 3; ++a)
#pragma unroll
                        for (int b = 0; b < 3; ++b) red_add(Kr + (uint64_t)(3 * a + b) * ne, Kb[a][b]);
                }
        }
    }
    if (WANT_E) {
        double tot;
        if (block_sum_last_done(e_acc, partials, counter, &tot)) *energy = (R)((double)*energy + tot);
    }
}

template <typename R, int MODEL>
ebb_status launch_atomic(Ctx* c, bool want_k, bool want_e, uint64_t nt, const Field* V, const Field* Ef,
                         const Field* U, const Field* D, const Field* W, const Field* MU, const Field* LA,
                         const Field* Fo, const Field* Ko, uint64_t ne, const Field* En, cudaStream_t s) {
    const int block = 128;
    unsigned grid = occ_grid(c, k_tet_map<R, MODEL, true, true>, block, 0, nt);
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
    EBB_DEVICE_GUARD(c);
    if (!c || !d) return fail(c, EBB_E_ARG, "null argument");
    if (d->model != EBB_STVK && d->model != EBB_NH) return fail(c, EBB_E_ARG, "unknown model %d", d->model);
    if (d->scatter < EBB_SCATTER_AUTO || d->scatter > EBB_SCATTER_CHUNK_RED)
        return fail(c, EBB_E_ARG, "unknown scatter strategy %d", d->scatter);
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
    uint64_t nt = c->rels[tets].size, nv = c->rels[verts].size;
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
    const char* envs = getenv("EBB_SCATTER");
    int strat = d->scatter;
    // AUTO = the measured fastest on C2 and C3: SEGMENTED for
    // f + K (every dtype and model); the force-only map is the atomic kernel
    const bool auto_pick = strat == EBB_SCATTER_AUTO && !(envs && atoi(envs) > 0);
    if (strat == EBB_SCATTER_AUTO) {
        if (envs && atoi(envs) > 0) strat = atoi(envs);
        else strat = EBB_SCATTER_SEGMENTED;
    }
    if (auto_pick && Ko) {
        // AUTO on a mesh whose plan the segmented map refuses (a vertex in more
        // tets than a tile holds): CHUNK, else ATOMIC -- decided once per (v, e)
        for (const auto& a : c->auto_map)
            if (a.v == d->v && a.e == d->e) strat = a.strategy;
        if (strat == EBB_SCATTER_SEGMENTED) {
            bool known = false;
            for (const auto& a : c->auto_map) known |= a.v == d->v && a.e == d->e;
            if (!known) {
                const int cand[3] = {EBB_SCATTER_SEGMENTED, EBB_SCATTER_CHUNK, EBB_SCATTER_ATOMIC};
                for (int k = 0; k < 3; ++k) {
                    ebb_status st = EBB_OK;
                    if (cand[k] == EBB_SCATTER_SEGMENTED) st = seg_plan_probe(c, d->v, d->e, dt, d->model);
                    if (cand[k] == EBB_SCATTER_CHUNK) st = chunk_plan_probe(c, d->v, d->e, dt, d->model);
                    if (st == EBB_E_RANGE) continue;
                    EBB_TRY(st);
                    strat = cand[k];
                    break;
                }
                c->auto_map.push_back({d->v, d->e, strat});
            }
        }
    }
    if (Ko && strat == EBB_SCATTER_COLOR) {
        // plain read-modify-write per colour: the outputs start from zero or accumulate
        if (d->zero_outputs) {
            EBB_CUDA(c, cudaMemsetAsync(Fo->ptr, 0, nv * 3 * dtype_size(dt), s));
            EBB_CUDA(c, cudaMemsetAsync(Ko->ptr, 0, ne * 9 * dtype_size(dt), s));
            if (En) EBB_CUDA(c, cudaMemsetAsync(En->ptr, 0, dtype_size(dt), s));
        }
        return color_map_launch(c, d->v, d->model, En != nullptr, nt, V, Ef, U, D, W, MU, LA, Fo, Ko, ne, En, s);
    }
    if (Ko && (strat == EBB_SCATTER_CHUNK || strat == EBB_SCATTER_CHUNK_RED)) {
        // CHUNK: every K row and f row is written exactly once (zero_outputs
        // means overwrite); CHUNK_RED: rows fed by several tiles are zeroed,
        // then added to with red.global.add
        if (d->zero_outputs && En) EBB_CUDA(c, cudaMemsetAsync(En->ptr, 0, dtype_size(dt), s));
        return chunk_map_launch(c, d->v, d->e, d->model, En != nullptr, d->zero_outputs ? 0 : 1, nt, V, U, D, W, MU,
                                LA, Fo, Ko, ne, En, s, strat == EBB_SCATTER_CHUNK_RED);
    }
    if (Ko && strat == EBB_SCATTER_SEGMENTED) {
        // every K row and f row is written exactly once: zero_outputs means overwrite
        if (d->zero_outputs && En) EBB_CUDA(c, cudaMemsetAsync(En->ptr, 0, dtype_size(dt), s));
        return seg_map_launch(c, d->v, d->e, d->model, En != nullptr, d->zero_outputs ? 0 : 1, nt, V, U, D, W, MU, LA,
                              Fo, Ko, ne, En, s);
    }
    if (Ko && (strat == EBB_SCATTER_TILED || strat == EBB_SCATTER_GATHER))
        return fail(c, EBB_E_ARG, "scatter strategy %d (TILED / GATHER) was retired in round 2: measured slower than "
                                  "SEGMENTED at every size (DESIGN.md §5.2)", strat);
    if (d->zero_outputs) {
        EBB_CUDA(c, cudaMemsetAsync(Fo->ptr, 0, nv * 3 * dtype_size(dt), s));
        if (Ko) EBB_CUDA(c, cudaMemsetAsync(Ko->ptr, 0, ne * 9 * dtype_size(dt), s));
        if (En) EBB_CUDA(c, cudaMemsetAsync(En->ptr, 0, dtype_size(dt), s));
    }
    bool wk = Ko != nullptr, we = En != nullptr;
    if (dt == EBB_F64) {
        if (d->model == EBB_NH) return launch_atomic<double, EBB_NH>(c, wk, we, nt, V, Ef, U, D, W, MU, LA, Fo, Ko, ne, En, s);
        return launch_atomic<double, EBB_STVK>(c, wk, we, nt, V, Ef, U, D, W, MU, LA, Fo, Ko, ne, En, s);
    }
    if (d->model == EBB_NH) return launch_atomic<float, EBB_NH>(c, wk, we, nt, V, Ef, U, D, W, MU, LA, Fo, Ko, ne, En, s);
    return launch_atomic<float, EBB_STVK>(c, wk, we, nt, V, Ef, U, D, W, MU, LA, Fo, Ko, ne, En, s);
}
