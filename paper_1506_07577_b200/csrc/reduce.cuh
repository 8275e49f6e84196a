// reduce.cuh -- global reductions fused into the producing kernel:
// warp shuffle tree -> block tree -> per-block partial -> the last block to
// finish (ticket counter) reduces the partials in block order.  The shuffle
// pattern and the partial order are fixed, so the result is deterministic for
// a fixed grid (no floating-point atomics).
#pragma once
#include <cuda_runtime.h>

namespace ebb {

enum { ROP_SUM = 0, ROP_MAX = 1, ROP_MIN = 2 };

template <int OP>
__device__ __forceinline__ double rop(double a, double b) {
    if (OP == ROP_SUM) return a + b;
    if (OP == ROP_MAX) return fmax(a, b);
    return fmin(a, b);
}

template <int OP>
__device__ __forceinline__ double rop_identity() {
    if (OP == ROP_SUM) return 0.0;
    if (OP == ROP_MAX) return -INFINITY;
    return INFINITY;
}

template <int OP>
__device__ __forceinline__ double warp_reduce(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = rop<OP>(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block reduction; result valid in every thread.  All threads must call.
template <int OP>
__device__ __forceinline__ double block_reduce(double v) {
    __shared__ double sw[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_reduce<OP>(v);
    __syncthreads();  // protect sw from a previous call
    if (lane == 0) sw[warp] = v;
    __syncthreads();
    double r = lane < nw ? sw[lane] : rop_identity<OP>();
    r = warp_reduce<OP>(r);
    return r;
}

// Two-pass grid reduction.  Returns true in thread 0 of the last block, with
// the grid total in *out.  `counter` must be 0 on entry; it is reset to 0.
template <int OP = ROP_SUM>
__device__ __forceinline__ bool block_reduce_last_done(double v, double* partials, unsigned int* counter,
                                                       double* out) {
    __shared__ bool am_last;
    double b = block_reduce<OP>(v);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = b;
        __threadfence();
        unsigned int ticket = atomicAdd(counter, 1u);
        am_last = (ticket == gridDim.x - 1);
    }
    __syncthreads();
    if (!am_last) return false;
    __threadfence();
    double s = rop_identity<OP>();
    for (unsigned int i = threadIdx.x; i < gridDim.x; i += blockDim.x) s = rop<OP>(s, __ldcg(&partials[i]));
    s = block_reduce<OP>(s);
    if (threadIdx.x == 0) {
        *counter = 0u;
        *out = s;
        return true;
    }
    return false;
}

__device__ __forceinline__ bool block_sum_last_done(double v, double* partials, unsigned int* counter, double* out) {
    return block_reduce_last_done<ROP_SUM>(v, partials, counter, out);
}

}  // namespace ebb
