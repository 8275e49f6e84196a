// cg_common.cuh -- what the single-GPU PCG kernels (solver.cu) and the fused
// multi-GPU PCG over peer memory (peer_cg.cu) share: the device scalar slots
// of ebb_cg.scal, the padded vec4 records of the CG work vectors, the TMA
// ring geometry of the persistent matvecs, the deterministic grid sum, and
// the host-side validation of an ebb_cg.
#pragma once
#include <cstdint>

#include "ebb_internal.cuh"
#include "reduce.cuh"

namespace ebb {

enum { S_RHO = 0, S_PQ = 1, S_RZ = 2, S_FIRST = 3, S_PAR = 4, S_ALPHA = 5, S_VAR = 6, S_RZ0 = 7, S_ITERS = 8,
       S_DONE = 9, S_DSUM = 10, S_GSUM = 11, S_NSCAL = 12 };
// S_VAR: single-reduction phase scalars pending (multi-GPU phase mode): 0 none,
// 1 after the prologue, 2 after an iteration; S_DSUM / S_GSUM hold the
// rank-local w.z / r.z sums the host allreduces between phases

template <typename R>
struct V4;
template <>
struct V4<double> {
    using T = double4;
};
template <>
struct V4<float> {
    using T = float4;
};

template <typename R>
__device__ __forceinline__ typename V4<R>::T ld4(const R* p, uint64_t v) {
    return reinterpret_cast<const typename V4<R>::T*>(p)[v];
}
// L1-bypassing (L2-coherent) 4-wide load: data written by other CTAs earlier in
// the same (persistent) kernel must not be served from a stale L1 line
__device__ __forceinline__ double4 ld4cg(const double* p, uint64_t v) {
    double4 r;
    asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
                 : "l"(p + 4 * v));
    return r;
}
__device__ __forceinline__ float4 ld4cg(const float* p, uint64_t v) {
    float4 r;
    asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p + 4 * v));
    return r;
}

template <typename R>
__device__ __forceinline__ void st4(R* p, uint64_t v, typename V4<R>::T x) {
    reinterpret_cast<typename V4<R>::T*>(p)[v] = x;
}

// Edge-relation matvec chunks streamed through shared memory by the TMA engine
// (solver.cu k_spmv_tma and the persistent PCG kernels)
#define TMA_VCH 16
#define TMA_NS 4
#define TMA_CONSUMERS 8
#define PCG_GROUPS 2                          // persistent PCG: consumer warp groups
#define PCG_WPG (TMA_CONSUMERS / PCG_GROUPS)  // warps per group
#ifndef CG1_NS
#define CG1_NS 4        // TMA ring depth of the single-reduction PCG
#endif
constexpr unsigned kCg1PartStride = 2048;   // partial slots per phase parity (grid <= 2048)

#ifndef EBB_BAR_SLEEP_NS
#define EBB_BAR_SLEEP_NS 64
#endif
// sum of the per-CTA partials in block order, same value in every CTA
__device__ __forceinline__ double grid_sum_partials(const double* partials, unsigned int n, double* sm_tot) {
    double s = 0.0;
    for (unsigned int i = threadIdx.x; i < n; i += blockDim.x) s += __ldcg(&partials[i]);
    s = block_reduce<ROP_SUM>(s);
    if (threadIdx.x == 0) *sm_tot = s;
    __syncthreads();
    return *sm_tot;
}


// Stage capacity (rows) of the TMA-fed matvecs: the rows of the largest
// 16-vertex chunk (measured per chunk at grouping time, not 16 x the longest
// group: one hub vertex no longer inflates every stage) + the 16-byte
// alignment slack of the 9 plane copies and the head copy.
// (a multiple of 4 rows: every plane of a stage starts 16-byte aligned, as
// the bulk copies require)
template <typename R>
uint32_t tma_cap(uint32_t chunk_rows) {
    return ((chunk_rows ? chunk_rows : 1u) + 2 * (16 / sizeof(R)) + 4 + 3) & ~3u;
}
constexpr size_t kTmaSmemMax = 200 * 1024;   // beyond it: the warp-per-vertex path (no staging)


// host-side checks of an ebb_cg (solver.cu)
ebb_status check_mask(Ctx* c, ebb_field m, ebb_rel rel, const uint8_t** out);
double cg_tol2(const ebb_cg* cg);
int cg_variant(const ebb_cg* cg, const EdgeGraph& G, ebb_dtype dt);
ebb_status cg_validate(Ctx* c, const ebb_cg* cg, EdgeGraph* G, ebb_dtype* dt);

}  // namespace ebb
