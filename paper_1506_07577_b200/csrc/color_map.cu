// color_map.cu -- the COLOURED element map (SURVEY §8(a) "+=" strategy (ii):
// deterministic colouring).  The tets are coloured so that no two tets of a
// colour share a vertex; then the map runs one launch per colour, one thread
// per tet, and every field reduction (f[v[i]] += f_i, K[e[i][j]] += K_ij,
// P:885) is a plain read-modify-write: inside a colour no two threads touch
// the same vertex, hence the same edge row (an edge row (a, b) is only touched
// by tets containing both a and b).  Deterministic (fixed colour and tet
// order) with no atomics, at the price of ncolours dependent launches -- the
// trade-off the paper reports for Liszt's colouring on Lulesh.
//
// Colouring (host, once per mesh): greedy first-fit in tet order over 64
// colours (a 64-bit mask of used colours per vertex); EBB_E_RANGE if a mesh
// needs more.  Physics: element.cuh (shared with every map strategy).
#include <algorithm>
#include <chrono>
#include <vector>

#include "ebb_internal.cuh"
#include "element.cuh"
#include "reduce.cuh"

namespace ebb {
namespace {

template <typename R, int MODEL, bool WANT_E>
__global__ void __launch_bounds__(128) k_tet_map_color(uint32_t n, const uint32_t* __restrict__ order, uint64_t nt,
                                                       const uint4* __restrict__ tv, const uint4* __restrict__ te,
                                                       const R* __restrict__ u, const R* __restrict__ Dminv,
                                                       const R* __restrict__ Wt, const R* __restrict__ mu_t,
                                                       const R* __restrict__ lam_t, R* __restrict__ f,
                                                       R* __restrict__ K, uint64_t ne, double* __restrict__ partials,
                                                       unsigned int* __restrict__ counter, R* __restrict__ energy,
                                                       unsigned long long* __restrict__ err) {
    double e_acc = 0.0;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const uint64_t t = order[k];
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
        if (WANT_E) e_acc += (double)(st.W * st.psi);
        R fi[4][3];
        tet_forces(st, fi);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int a = 0; a < 3; ++a) f[3ull * v[i] + a] += fi[i][a];   // vertex-disjoint within a colour
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint4 rr = te[4 * t + i];
            const uint32_t row[4] = {rr.x, rr.y, rr.z, rr.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                R Kb[3][3];
                tet_block<R, MODEL>(st, i, j, Kb);
                R* Kr = K + row[j];
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int b = 0; b < 3; ++b) Kr[(uint64_t)(3 * a + b) * ne] += Kb[a][b];
            }
        }
    }
    if (WANT_E) {
        double tot;
        if (block_sum_last_done(e_acc, partials, counter, &tot)) *energy = (R)((double)*energy + tot);
    }
}

ebb_status build_color_plan(Ctx* c, ebb_field vf, ColorPlan** out) {
    for (ColorPlan* P : c->colorplans)
        if (P->v == vf) {
            *out = P;
            return EBB_OK;
        }
    const auto t0 = std::chrono::steady_clock::now();
    Field* V = get_field(c, vf);
    const uint64_t nt = c->rels[V->rel].size, nv = c->rels[V->key_target].size;
    std::vector<uint32_t> tv(nt * 4);
    EBB_CUDA(c, cudaMemcpy(tv.data(), V->ptr, nt * 16, cudaMemcpyDeviceToHost));
    std::vector<uint64_t> used(nv, 0);
    std::vector<uint8_t> col(nt);
    std::vector<uint32_t> cnt(65, 0);
    int ncol = 0;
    for (uint64_t t = 0; t < nt; ++t) {
        const uint32_t* v = &tv[4 * t];
        const uint64_t m = used[v[0]] | used[v[1]] | used[v[2]] | used[v[3]];
        if (m == ~0ull) return fail(c, EBB_E_RANGE, "colour map: tet %llu needs more than 64 colours", (unsigned long long)t);
        const int k = __builtin_ctzll(~m);
        col[t] = (uint8_t)k;
        cnt[k + 1]++;
        ncol = std::max(ncol, k + 1);
        for (int i = 0; i < 4; ++i) used[v[i]] |= 1ull << k;
    }
    std::vector<uint32_t> off(ncol + 1, 0), order(nt);
    for (int k = 0; k < ncol; ++k) off[k + 1] = off[k] + cnt[k + 1];
    {
        std::vector<uint32_t> cur(off.begin(), off.end() - 1);
        for (uint64_t t = 0; t < nt; ++t) order[cur[col[t]]++] = (uint32_t)t;
    }
    ColorPlan* P = new ColorPlan();
    P->v = vf;
    P->ncolors = ncol;
    P->offsets.assign(off.begin(), off.end());
    if (cudaMalloc(&P->order, nt * 4 + 16) != cudaSuccess ||
        cudaMemcpy(P->order, order.data(), nt * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
        P->release();
        delete P;
        return fail(c, EBB_E_CUDA, "colour map: plan upload failed");
    }
    P->host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    c->colorplans.push_back(P);
    *out = P;
    return EBB_OK;
}

template <typename R, int MODEL>
ebb_status launch_color_t(Ctx* c, const ColorPlan& P, bool want_e, uint64_t nt, const Field* V, const Field* Ef,
                          const Field* U, const Field* D, const Field* W, const Field* MU, const Field* LA,
                          const Field* Fo, const Field* Ko, uint64_t ne, const Field* En, cudaStream_t s) {
    auto kern = want_e ? k_tet_map_color<R, MODEL, true> : k_tet_map_color<R, MODEL, false>;
    KernelTimer kt(c, EBB_K_TET_MAP, s);   // one timed region over all colours
    for (int k = 0; k < P.ncolors; ++k) {
        const uint32_t n = P.offsets[k + 1] - P.offsets[k];
        if (!n) continue;
        const unsigned grid = occ_grid(c, kern, 128, 0, n);
        kern<<<grid, 128, 0, s>>>(n, P.order + P.offsets[k], nt, (const uint4*)V->ptr, (const uint4*)Ef->ptr,
                                  (const R*)U->ptr, (const R*)D->ptr, (const R*)W->ptr, (const R*)MU->ptr,
                                  (const R*)LA->ptr, (R*)Fo->ptr, (R*)Ko->ptr, ne, c->d_partials, c->d_counter + 0,
                                  En ? (R*)En->ptr : nullptr, c->d_err);
        EBB_CUDA(c, cudaGetLastError());
        if (k > 0) c->launches++;   // KernelTimer counted the first
    }
    return EBB_OK;
}

}  // namespace

ebb_status color_map_launch(Ctx* c, ebb_field vf, int model, bool want_e, uint64_t nt, const Field* V,
                            const Field* Ef, const Field* U, const Field* D, const Field* W, const Field* MU,
                            const Field* LA, const Field* Fo, const Field* Ko, uint64_t ne, const Field* En,
                            cudaStream_t s) {
    ColorPlan* P;
    EBB_TRY(build_color_plan(c, vf, &P));
    if (U->dtype == EBB_F64) {
        if (model == EBB_NH) return launch_color_t<double, EBB_NH>(c, *P, want_e, nt, V, Ef, U, D, W, MU, LA, Fo, Ko, ne, En, s);
        return launch_color_t<double, EBB_STVK>(c, *P, want_e, nt, V, Ef, U, D, W, MU, LA, Fo, Ko, ne, En, s);
    }
    if (model == EBB_NH) return launch_color_t<float, EBB_NH>(c, *P, want_e, nt, V, Ef, U, D, W, MU, LA, Fo, Ko, ne, En, s);
    return launch_color_t<float, EBB_STVK>(c, *P, want_e, nt, V, Ef, U, D, W, MU, LA, Fo, Ko, ne, En, s);
}

int color_plan_colors(Ctx* c, ebb_field vf) {
    for (ColorPlan* P : c->colorplans)
        if (P->v == vf) return P->ncolors;
    return 0;
}

}  // namespace ebb
