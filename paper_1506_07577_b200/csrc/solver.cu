// solver.cu -- edge-relation matvec, Jacobi-PCG, implicit assembly, integrator
// updates and global reductions.
//
// The matvec is the paper's query-loop `for e in v.edges do ... e.head ... end`
// over the edge relation grouped by tail (CSR) with the
// 3x3 stiffness stored per edge.  PCG follows Saad Alg. 9.1
// with the Jacobi preconditioner; every scalar stays on the device.
//
// PCG iteration (one stream, no host synchronisation), two kernels:
//   spmv (CG)    beta = rz/rho (0 on the first iteration); p = z + beta p_old,
//                formed on the fly for every gathered head and stored for the
//                owned vertex (p double-buffered); q = (A p) * mask; local p.q
//   k_cg_update  alpha = rho / p.q; x += alpha p; r -= alpha q; z = r * dinv; local r.z
// Between kernels the scalars p.q and r.z are the only cross-CTA (and, on
// several GPUs, cross-rank) reductions; z is the only vector a halo needs.
// CG work vectors are padded 4-component records (32 B fp64 / 16 B fp32) so a
// vertex is one 256-/128-bit access.
#include <cstdlib>
#include <type_traits>

#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "async_copy.cuh"
#include "cg_common.cuh"
#include "ebb_internal.cuh"
#include "reduce.cuh"

using namespace ebb;

namespace {

// ---------------------------------------------------------------------------
// Edge-relation matvec, register path (used for borrowed, unpadded columns):
// two phases per CTA chunk of SPMV_VC vertices -- flat coalesced row loads
// into shared memory, then 4 lanes per vertex sum the vertex's rows.
#define SPMV_VC 64
#define SPMV_BATCH 4
template <typename R, bool MPQ>
__global__ void __launch_bounds__(256) k_spmv(uint64_t nv, const uint32_t* __restrict__ index,
                                              const uint32_t* __restrict__ head, const R* __restrict__ A, uint64_t ne,
                                              const R* __restrict__ p, R* __restrict__ q,
                                              const uint8_t* __restrict__ mask, double* __restrict__ partials,
                                              unsigned int* __restrict__ counter, double* __restrict__ pq_out) {
    extern __shared__ __align__(16) unsigned char spmv_smem[];
    R* ys = reinterpret_cast<R*>(spmv_smem);
    double pq = 0.0;
    const uint64_t nchunks = (nv + SPMV_VC - 1) / SPMV_VC;
    for (uint64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const uint64_t v0 = ch * SPMV_VC;
        const uint64_t v1 = v0 + SPMV_VC < nv ? v0 + SPMV_VC : nv;
        const uint32_t e0 = index[v0], nr = index[v1] - e0;
        for (uint32_t kb = threadIdx.x; kb < nr; kb += SPMV_BATCH * 256) {
            R a[SPMV_BATCH][9];
            uint32_t hh[SPMV_BATCH];
#pragma unroll
            for (int u = 0; u < SPMV_BATCH; ++u) {
                const uint32_t k = kb + u * 256;
                if (k < nr) {
                    const uint64_t e = e0 + k;
                    hh[u] = __ldcs(head + e);
#pragma unroll
                    for (int c = 0; c < 9; ++c) a[u][c] = __ldcs(A + c * ne + e);
                }
            }
#pragma unroll
            for (int u = 0; u < SPMV_BATCH; ++u) {
                const uint32_t k = kb + u * 256;
                if (k < nr) {
                    const uint64_t h = 3ull * hh[u];
                    const R px = p[h], py = p[h + 1], pz = p[h + 2];
                    ys[3 * k] = a[u][0] * px + a[u][1] * py + a[u][2] * pz;
                    ys[3 * k + 1] = a[u][3] * px + a[u][4] * py + a[u][5] * pz;
                    ys[3 * k + 2] = a[u][6] * px + a[u][7] * py + a[u][8] * pz;
                }
            }
        }
        __syncthreads();
        const uint64_t v = v0 + (threadIdx.x >> 2);
        const unsigned sub = threadIdx.x & 3;
        const bool valid = v < v1;
        R a0 = 0, a1 = 0, a2 = 0;
        if (valid) {
            const uint32_t r1 = index[v + 1] - e0;
            for (uint32_t r = index[v] - e0 + sub; r < r1; r += 4) {
                a0 += ys[3 * r];
                a1 += ys[3 * r + 1];
                a2 += ys[3 * r + 2];
            }
        }
#pragma unroll
        for (int o = 2; o > 0; o >>= 1) {
            a0 += __shfl_xor_sync(0xffffffffu, a0, o, 4);
            a1 += __shfl_xor_sync(0xffffffffu, a1, o, 4);
            a2 += __shfl_xor_sync(0xffffffffu, a2, o, 4);
        }
        if (sub == 0 && valid) {
            if (MPQ && mask && !mask[v]) a0 = a1 = a2 = 0;
            q[3 * v] = a0;
            q[3 * v + 1] = a1;
            q[3 * v + 2] = a2;
            if (MPQ) pq += (double)p[3 * v] * a0 + (double)p[3 * v + 1] * a1 + (double)p[3 * v + 2] * a2;
        }
        __syncthreads();
    }
    if (MPQ) {
        double tot;
        if (block_sum_last_done(pq, partials, counter, &tot)) *pq_out = tot;
    }
}

// ---------------------------------------------------------------------------
// Edge-relation matvec streamed through shared memory by the TMA engine,
// warp-specialized.  A persistent CTA walks chunks of TMA_VCH consecutive
// vertices; the rows of a chunk are one contiguous range of the grouped edge
// relation, so its 9 A planes and its head keys are 10 contiguous segments.
//   producer warp (warp 8, one lane): for each chunk, waits until the ring
//     stage is empty, then issues 10 1-D bulk async copies (cp.async.bulk,
//     L2 evict-first) that complete on the stage's "full" mbarrier;
//   consumer warps 0..7: each owns 2 vertices of every chunk (16 lanes per
//     vertex), waits on "full", reads A and head from shared memory, gathers
//     p through head (L2-resident; one 256-bit load per head in CG mode),
//     reduces with shuffles, then arrives on the stage's "empty" mbarrier.
//     No block-wide barrier inside the loop: consumer warps run ahead of each
//     other by up to TMA_NS chunks.
// CG = true: p, q are padded vec4 records; MPQ: q *= mask, fused local p.q.
template <typename R, bool CG, bool MPQ, bool DIR = false, bool GRP = true>
__global__ void __launch_bounds__(32 * (TMA_CONSUMERS + 1))
    k_spmv_tma(uint64_t nv, const uint32_t* __restrict__ index, const uint32_t* __restrict__ head,
               const R* __restrict__ A, uint64_t ne, const R* __restrict__ p, R* __restrict__ q,
               const uint8_t* __restrict__ mask, double* __restrict__ partials, unsigned int* __restrict__ counter,
               double* __restrict__ pq_out, uint32_t cap, R* pbuf0 = nullptr, R* pbuf1 = nullptr,
               double* __restrict__ scal = nullptr) {
    extern __shared__ __align__(128) unsigned char tma_smem[];
    __shared__ __align__(8) uint64_t full_bar[TMA_NS], empty_bar[TMA_NS];
    constexpr uint32_t AE = 16 / sizeof(R);   // elements per 16 B
    const size_t stage_bytes = ((size_t)9 * cap * sizeof(R) + (size_t)cap * 4 + 127) & ~(size_t)127;
    if (DIR && scal[S_DONE] != 0.0) return;   // PCG converged (tolerance mode): no-op
    const uint64_t nchunks = (nv + TMA_VCH - 1) / TMA_VCH;
    const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < TMA_NS; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], GRP ? PCG_WPG : TMA_CONSUMERS);
        }
        mbar_fence_init();
    }
    __syncthreads();
    double pq = 0.0;
    if (warp == TMA_CONSUMERS) {
        if (lane == 0) {
            uint32_t k = 0;
            for (uint64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x, ++k) {
                const int s = k % TMA_NS;
                const uint64_t v0 = ch * TMA_VCH;
                const uint64_t v1 = v0 + TMA_VCH < nv ? v0 + TMA_VCH : nv;
                const uint64_t e0 = index[v0], e1 = index[v1];
                if (k >= TMA_NS) mbar_wait(&empty_bar[s], ((k / TMA_NS) + 1) & 1u);
                unsigned char* base = tma_smem + s * stage_bytes;
                uint32_t tot = 0;
#pragma unroll
                for (int c = 0; c < 9; ++c) {
                    const uint64_t a0 = (c * ne + e0) & ~(uint64_t)(AE - 1);
                    const uint64_t a1 = (c * ne + e1 + AE - 1) & ~(uint64_t)(AE - 1);
                    tot += (uint32_t)((a1 - a0) * sizeof(R));
                }
                const uint64_t h0 = e0 & ~3ull, h1 = (e1 + 3) & ~3ull;
                tot += (uint32_t)((h1 - h0) * 4);
                fence_proxy_async_smem();
                mbar_arrive_expect_tx(&full_bar[s], tot);
#pragma unroll
                for (int c = 0; c < 9; ++c) {
                    const uint64_t a0 = (c * ne + e0) & ~(uint64_t)(AE - 1);
                    const uint64_t a1 = (c * ne + e1 + AE - 1) & ~(uint64_t)(AE - 1);
                    bulk_g2s_evict_first(base + (size_t)c * cap * sizeof(R), A + a0,
                                         (uint32_t)((a1 - a0) * sizeof(R)), &full_bar[s]);
                }
                bulk_g2s_evict_first(base + (size_t)9 * cap * sizeof(R), head + h0, (uint32_t)((h1 - h0) * 4),
                                     &full_bar[s]);
            }
        }
    } else {
        // GRP: consumer group g (warps 4g..4g+3) takes the chunks k = g mod 2,
        // 8 lanes per vertex, two rows per lane per pass (both gathers in
        // flight); else all 8 warps take every chunk, 16 lanes per vertex
        const unsigned grp = GRP ? warp / PCG_WPG : 0u, wig = GRP ? warp % PCG_WPG : warp;
        constexpr unsigned LPV = GRP ? 8u : 16u;
        const unsigned sub = lane & (LPV - 1);
        // DIR (CG): p = z + beta p_old on the fly -- `p` holds z, p is double-buffered
        const R* __restrict__ pold = nullptr;
        R* __restrict__ pnew = nullptr;
        R beta = 0;
        if (DIR) {
            const int cur = scal[S_PAR] != 0.0;
            pold = cur ? pbuf1 : pbuf0;
            pnew = cur ? pbuf0 : pbuf1;
            const double rho = scal[S_RHO], rz = scal[S_RZ];
            beta = (scal[S_FIRST] != 0.0 || rho == 0.0) ? R(0) : (R)(rz / rho);
        }
        uint32_t k = grp;
        for (uint64_t ch = blockIdx.x + (uint64_t)grp * gridDim.x; ch < nchunks;
             ch += (uint64_t)gridDim.x * (GRP ? PCG_GROUPS : 1), k += (GRP ? PCG_GROUPS : 1)) {
            const int s = k % TMA_NS;
            const uint64_t v0 = ch * TMA_VCH;
            const uint64_t v1 = v0 + TMA_VCH < nv ? v0 + TMA_VCH : nv;
            const uint64_t v = GRP ? v0 + 4 * wig + (lane >> 3) : v0 + 2 * warp + (lane >> 4);
            const bool valid = v < v1;
            const uint32_t e0 = index[v0];
            const uint32_t r0 = valid ? index[v] - e0 : 0u, r1 = valid ? index[v + 1] - e0 : 0u;
            R own0 = 0, own1 = 0, own2 = 0;
            uint8_t mk = 1;
            if (MPQ && valid && sub == 0) {
                if (DIR) {
                    const auto zv = ld4(p, v);
                    const auto ov = ld4(pold, v);
                    own0 = zv.x + beta * ov.x;
                    own1 = zv.y + beta * ov.y;
                    own2 = zv.z + beta * ov.z;
                } else if (CG) {
                    const auto pv = ld4(p, v);
                    own0 = pv.x;
                    own1 = pv.y;
                    own2 = pv.z;
                } else {
                    own0 = p[3 * v];
                    own1 = p[3 * v + 1];
                    own2 = p[3 * v + 2];
                }
                if (mask) mk = mask[v];
            }
            mbar_wait(&full_bar[s], (k / TMA_NS) & 1u);
            const unsigned char* base = tma_smem + s * stage_bytes;
            const uint32_t* hs = reinterpret_cast<const uint32_t*>(base + (size_t)9 * cap * sizeof(R)) + (e0 & 3u);
            auto gather = [&](uint32_t hv, R& px, R& py, R& pz) {
                if (DIR) {
                    const auto zv = ld4(p, hv);
                    const auto ov = ld4(pold, hv);
                    px = zv.x + beta * ov.x;
                    py = zv.y + beta * ov.y;
                    pz = zv.z + beta * ov.z;
                } else if (CG) {
                    const auto pv = ld4(p, hv);
                    px = pv.x;
                    py = pv.y;
                    pz = pv.z;
                } else {
                    px = p[3ull * hv];
                    py = p[3ull * hv + 1];
                    pz = p[3ull * hv + 2];
                }
            };
            R a0 = 0, a1 = 0, a2 = 0;
            constexpr unsigned STEP = GRP ? 2 * LPV : LPV;
            for (uint32_t r = r0 + sub; r < r1; r += STEP) {
                const uint32_t rr = r + LPV;
                const bool two = GRP && rr < r1;
                const uint32_t hv = hs[r], hw = two ? hs[rr] : hv;
                R px, py, pz, qx = 0, qy = 0, qz = 0;
                gather(hv, px, py, pz);
                if (GRP) gather(hw, qx, qy, qz);
                R av[9], bv[9];
#pragma unroll
                for (int c = 0; c < 9; ++c) {
                    const uint32_t off = (uint32_t)((c * ne + e0) & (AE - 1));
                    const R* pl = reinterpret_cast<const R*>(base + (size_t)c * cap * sizeof(R)) + off;
                    av[c] = pl[r];
                    bv[c] = two ? pl[rr] : R(0);
                }
                a0 += av[0] * px + av[1] * py + av[2] * pz + (bv[0] * qx + bv[1] * qy + bv[2] * qz);
                a1 += av[3] * px + av[4] * py + av[5] * pz + (bv[3] * qx + bv[4] * qy + bv[5] * qz);
                a2 += av[6] * px + av[7] * py + av[8] * pz + (bv[6] * qx + bv[7] * qy + bv[8] * qz);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[s]);
#pragma unroll
            for (int o = LPV / 2; o > 0; o >>= 1) {
                a0 += __shfl_xor_sync(0xffffffffu, a0, o, LPV);
                a1 += __shfl_xor_sync(0xffffffffu, a1, o, LPV);
                a2 += __shfl_xor_sync(0xffffffffu, a2, o, LPV);
            }
            if (sub == 0 && valid) {
                if (MPQ && !mk) a0 = a1 = a2 = 0;
                if (CG) {
                    typename V4<R>::T qv;
                    qv.x = a0;
                    qv.y = a1;
                    qv.z = a2;
                    qv.w = 0;
                    st4(q, v, qv);
                    if (DIR) {
                        typename V4<R>::T pv;
                        pv.x = own0;
                        pv.y = own1;
                        pv.z = own2;
                        pv.w = 0;
                        st4(pnew, v, pv);
                    }
                } else {
                    q[3 * v] = a0;
                    q[3 * v + 1] = a1;
                    q[3 * v + 2] = a2;
                }
                if (MPQ) pq += (double)own0 * a0 + (double)own1 * a1 + (double)own2 * a2;
            }
        }
    }
    if (MPQ) {
        double tot;
        if (block_sum_last_done(pq, partials, counter, &tot)) {
            *pq_out = tot;
            if (DIR) {   // every block has read rho/rz/parity: retire them
                scal[S_RHO] = scal[S_RZ];
                scal[S_FIRST] = 0.0;
                scal[S_PAR] = scal[S_PAR] != 0.0 ? 0.0 : 1.0;
            }
        }
    }
}


// ---------------------------------------------------------------------------
// Edge-relation matvec without any staging: one warp per vertex, lanes stride
// its rows (any group length: the fallback when the largest chunk does not fit
// the TMA stages or the register path's shared memory, e.g. a hub vertex of
// thousands of edges).  Same modes and outputs as k_spmv_tma (CG padded
// records, DIR direction update formed on the fly, MPQ mask + fused p.q).
template <typename R, bool CG, bool MPQ, bool DIR>
__global__ void __launch_bounds__(256) k_spmv_warp(uint64_t nv, const uint32_t* __restrict__ index,
                                                   const uint32_t* __restrict__ head, const R* __restrict__ A,
                                                   uint64_t ne, const R* __restrict__ p, R* __restrict__ q,
                                                   const uint8_t* __restrict__ mask, double* __restrict__ partials,
                                                   unsigned int* __restrict__ counter, double* __restrict__ pq_out,
                                                   R* pbuf0, R* pbuf1, double* __restrict__ scal) {
    if (DIR && scal[S_DONE] != 0.0) return;   // PCG converged (tolerance mode): no-op
    const unsigned lane = threadIdx.x & 31;
    const R* __restrict__ pold = nullptr;
    R* __restrict__ pnew = nullptr;
    R beta = 0;
    if (DIR) {
        const int cur = scal[S_PAR] != 0.0;
        pold = cur ? pbuf1 : pbuf0;
        pnew = cur ? pbuf0 : pbuf1;
        const double rho = scal[S_RHO], rz = scal[S_RZ];
        beta = (scal[S_FIRST] != 0.0 || rho == 0.0) ? R(0) : (R)(rz / rho);
    }
    auto gather = [&](uint64_t hv, R& px, R& py, R& pz) {
        if (DIR) {
            const auto zv = ld4(p, hv);
            const auto ov = ld4(pold, hv);
            px = zv.x + beta * ov.x;
            py = zv.y + beta * ov.y;
            pz = zv.z + beta * ov.z;
        } else if (CG) {
            const auto pv = ld4(p, hv);
            px = pv.x;
            py = pv.y;
            pz = pv.z;
        } else {
            px = p[3 * hv];
            py = p[3 * hv + 1];
            pz = p[3 * hv + 2];
        }
    };
    double pq = 0.0;
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t v = wid; v < nv; v += nw) {
        R a0 = 0, a1 = 0, a2 = 0;
        for (uint32_t r = index[v] + lane; r < index[v + 1]; r += 32) {
            R px, py, pz;
            gather(head[r], px, py, pz);
            a0 += A[r] * px + A[ne + r] * py + A[2 * ne + r] * pz;
            a1 += A[3 * ne + r] * px + A[4 * ne + r] * py + A[5 * ne + r] * pz;
            a2 += A[6 * ne + r] * px + A[7 * ne + r] * py + A[8 * ne + r] * pz;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a0 += __shfl_xor_sync(0xffffffffu, a0, o);
            a1 += __shfl_xor_sync(0xffffffffu, a1, o);
            a2 += __shfl_xor_sync(0xffffffffu, a2, o);
        }
        if (lane == 0) {
            R own0 = 0, own1 = 0, own2 = 0;
            if (MPQ) gather(v, own0, own1, own2);
            if (MPQ && mask && !mask[v]) a0 = a1 = a2 = 0;
            if (CG) {
                typename V4<R>::T qv;
                qv.x = a0;
                qv.y = a1;
                qv.z = a2;
                qv.w = 0;
                st4(q, v, qv);
                if (DIR) {
                    typename V4<R>::T pv;
                    pv.x = own0;
                    pv.y = own1;
                    pv.z = own2;
                    pv.w = 0;
                    st4(pnew, v, pv);
                }
            } else {
                q[3 * v] = a0;
                q[3 * v + 1] = a1;
                q[3 * v + 2] = a2;
            }
            if (MPQ) pq += (double)own0 * a0 + (double)own1 * a1 + (double)own2 * a2;
        }
    }
    if (MPQ) {
        double tot;
        if (block_sum_last_done(pq, partials, counter, &tot)) {
            *pq_out = tot;
            if (DIR) {
                scal[S_RHO] = scal[S_RZ];
                scal[S_FIRST] = 0.0;
                scal[S_PAR] = scal[S_PAR] != 0.0 ? 0.0 : 1.0;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Persistent PCG (single GPU): all `iters` iterations in one cooperative
// launch.  Every CTA runs the warp-specialized TMA matvec of k_spmv_tma over
// its chunks, then a software grid barrier, then the vector update over a
// grid-stride range of vertices, then a grid barrier.  The two dots are
// per-CTA partials summed by every CTA in block order (deterministic, no
// last-block second pass), so alpha and beta are known everywhere right after
// each barrier.  The producer warp keeps streaming: when a matvec phase ends
// it immediately issues the first TMA_NS chunks of the next iteration, so the
// HBM stream of A overlaps the latency-bound update phase and the barriers.
__device__ __forceinline__ void grid_barrier(unsigned int* count, unsigned int* gen, unsigned int nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int g = *reinterpret_cast<volatile unsigned int*>(gen);
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *reinterpret_cast<volatile unsigned int*>(count) = 0u;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*reinterpret_cast<volatile unsigned int*>(gen) == g) __nanosleep(EBB_BAR_SLEEP_NS);
        }
        __threadfence();
    }
    __syncthreads();
}

// fp32 solves use the cooperative-groups grid sync, fp64 the counter barrier
// above (measured per dtype, profiles/r01_c4_cg_barrier.txt: grid.sync is
// 5-16 % faster in fp32, up to 8 % slower in fp64 at 1e7 tets)
template <typename R>
__device__ __forceinline__ void grid_barrier_t(unsigned int* count, unsigned int* gen, unsigned int nblocks) {
    if constexpr (sizeof(R) == 4) {
        (void)count;
        (void)gen;
        (void)nblocks;
        cooperative_groups::this_grid().sync();
    } else {
        grid_barrier(count, gen, nblocks);
    }
}

#ifdef CG_PROF   // measurement-only build: per-phase clock split of thread 0 of every CTA
__device__ unsigned long long g_cg_prof[8];
#define CG_MARK(q)                                  \
    do {                                            \
        if (threadIdx.x == 0) {                     \
            const long long tn_ = clock64();        \
            cg_tp[q] += tn_ - cg_t0[0];             \
            cg_t0[0] = tn_;                         \
        }                                           \
    } while (0)
#else
#define CG_MARK(q) \
    do {           \
    } while (0)
#endif
template <typename R>
__global__ void __launch_bounds__(32 * (TMA_CONSUMERS + 1))
    k_cg_persistent(uint64_t nv, const uint32_t* __restrict__ index, const uint32_t* __restrict__ head,
                    const R* __restrict__ A, uint64_t ne, R* __restrict__ z, R* pb0, R* pb1, R* __restrict__ q,
                    const R* __restrict__ dinv, R* __restrict__ x, R* __restrict__ r,
                    const uint8_t* __restrict__ mask, double* __restrict__ part_pq, double* __restrict__ part_rz,
                    unsigned int* __restrict__ bar_count, unsigned int* __restrict__ bar_gen,
                    double* __restrict__ scal, double* __restrict__ rho_user, unsigned long long* __restrict__ err,
                    uint32_t cap, int iters, double tol2) {
    extern __shared__ __align__(128) unsigned char tma_smem[];
    __shared__ __align__(8) uint64_t full_bar[TMA_NS], empty_bar[TMA_NS];
    __shared__ double sm_tot;
    constexpr uint32_t AE = 16 / sizeof(R);
    const size_t stage_bytes = ((size_t)9 * cap * sizeof(R) + (size_t)cap * 4 + 127) & ~(size_t)127;
    const uint64_t nchunks = (nv + TMA_VCH - 1) / TMA_VCH;
    const uint64_t my_chunks = nchunks > blockIdx.x ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < TMA_NS; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], PCG_WPG);
        }
        mbar_fence_init();
    }
    __syncthreads();
    // scalars (identical in every CTA)
    double rho = scal[S_RHO];
    int first = scal[S_FIRST] != 0.0;
    int cur = scal[S_PAR] != 0.0;
    double rz_new = scal[S_RZ];
    const double rz0 = scal[S_RZ0];
    if (scal[S_DONE] != 0.0) iters = 0;   // converged in an earlier call (tolerance mode)
    int done_it = 0;
    bool conv = false;
    // producer state: global chunk sequence number (continues across iterations)
    uint64_t issued = 0;          // stage uses issued so far
    auto issue = [&](uint64_t ch, uint64_t seq) {
        const int s = seq % TMA_NS;
        const uint64_t v0 = ch * TMA_VCH;
        const uint64_t v1 = v0 + TMA_VCH < nv ? v0 + TMA_VCH : nv;
        const uint64_t e0 = index[v0], e1 = index[v1];
        if (seq >= TMA_NS) mbar_wait(&empty_bar[s], (uint32_t)(((seq / TMA_NS) + 1) & 1u));
        unsigned char* base = tma_smem + s * stage_bytes;
        uint32_t tot = 0;
#pragma unroll
        for (int c = 0; c < 9; ++c) {
            const uint64_t a0 = (c * ne + e0) & ~(uint64_t)(AE - 1);
            const uint64_t a1 = (c * ne + e1 + AE - 1) & ~(uint64_t)(AE - 1);
            tot += (uint32_t)((a1 - a0) * sizeof(R));
        }
        const uint64_t h0 = e0 & ~3ull, h1 = (e1 + 3) & ~3ull;
        tot += (uint32_t)((h1 - h0) * 4);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&full_bar[s], tot);
#pragma unroll
        for (int c = 0; c < 9; ++c) {
            const uint64_t a0 = (c * ne + e0) & ~(uint64_t)(AE - 1);
            const uint64_t a1 = (c * ne + e1 + AE - 1) & ~(uint64_t)(AE - 1);
            bulk_g2s_evict_first(base + (size_t)c * cap * sizeof(R), A + a0, (uint32_t)((a1 - a0) * sizeof(R)),
                                 &full_bar[s]);
        }
        bulk_g2s_evict_first(base + (size_t)9 * cap * sizeof(R), head + h0, (uint32_t)((h1 - h0) * 4), &full_bar[s]);
    };
    // prologue: the first TMA_NS chunks of iteration 0
    if (iters > 0 && warp == TMA_CONSUMERS && lane == 0)
        for (uint64_t j = 0; j < my_chunks && j < TMA_NS; ++j) issue(blockIdx.x + j * gridDim.x, issued++);
    const uint64_t gthreads = (uint64_t)gridDim.x * blockDim.x;
#ifdef CG_PROF
    __shared__ long long cg_tp[5], cg_t0[1];
    if (threadIdx.x == 0) {
        for (int q = 0; q < 5; ++q) cg_tp[q] = 0;
        cg_t0[0] = clock64();
    }
#endif
    for (int it = 0; it < iters; ++it) {
        const R beta = (first || rho == 0.0) ? R(0) : (R)(rz_new / rho);
        const R* __restrict__ pold = cur ? pb1 : pb0;
        R* __restrict__ pnew = cur ? pb0 : pb1;
        double pq = 0.0;
        if (warp == TMA_CONSUMERS) {
            // producer: remaining chunks of this iteration, then the head of the next one
            if (lane == 0) {
                for (uint64_t j = TMA_NS; j < my_chunks; ++j) issue(blockIdx.x + j * gridDim.x, issued++);
                if (it + 1 < iters)
                    for (uint64_t j = 0; j < my_chunks && j < TMA_NS; ++j) issue(blockIdx.x + j * gridDim.x, issued++);
            }
        } else {
            // consumer group g (warps 4g..4g+3) takes the chunks of sequence
            // number = g (mod 2); 8 lanes per vertex, 4 vertices per warp
            const unsigned grp = warp / PCG_WPG, wig = warp % PCG_WPG;
            const unsigned sub = lane & 7;
            const uint64_t seq0 = (uint64_t)it * my_chunks;
            for (uint64_t j = grp; j < my_chunks; j += PCG_GROUPS) {
                const uint64_t seq = seq0 + j;
                const uint64_t ch = blockIdx.x + j * gridDim.x;
                const int s = seq % TMA_NS;
                const uint64_t v0 = ch * TMA_VCH;
                const uint64_t v1 = v0 + TMA_VCH < nv ? v0 + TMA_VCH : nv;
                const uint64_t v = v0 + 4 * wig + (lane >> 3);
                const bool valid = v < v1;
                const uint32_t e0 = index[v0];
                const uint32_t r0 = valid ? index[v] - e0 : 0u, r1 = valid ? index[v + 1] - e0 : 0u;
                R own0 = 0, own1 = 0, own2 = 0;
                uint8_t mk = 1;
                if (valid && sub == 0) {
                    const auto zv = ld4cg(z, v);
                    const auto ov = ld4cg(pold, v);
                    own0 = zv.x + beta * ov.x;
                    own1 = zv.y + beta * ov.y;
                    own2 = zv.z + beta * ov.z;
                    if (mask) mk = mask[v];
                }
                mbar_wait(&full_bar[s], (uint32_t)((seq / TMA_NS) & 1u));
                const unsigned char* base = tma_smem + s * stage_bytes;
                const uint32_t* hs = reinterpret_cast<const uint32_t*>(base + (size_t)9 * cap * sizeof(R)) + (e0 & 3u);
                uint32_t off[9];
#pragma unroll
                for (int c = 0; c < 9; ++c) off[c] = (uint32_t)((c * ne + e0) & (AE - 1));
                R a0 = 0, a1 = 0, a2 = 0;
                for (uint32_t rb = r0 + sub; rb < r1; rb += 16) {
                    // two rows per lane per pass: both gathers in flight together
                    const uint32_t rr1 = rb + 8;
                    const bool two = rr1 < r1;
                    const uint32_t h0 = hs[rb], h1 = two ? hs[rr1] : h0;
                    const auto z0 = ld4cg(z, h0);
                    const auto o0 = ld4cg(pold, h0);
                    const auto z1 = ld4cg(z, h1);
                    const auto o1 = ld4cg(pold, h1);
                    R av[9], bv[9];
#pragma unroll
                    for (int c = 0; c < 9; ++c) {
                        const R* pl = reinterpret_cast<const R*>(base + (size_t)c * cap * sizeof(R)) + off[c];
                        av[c] = pl[rb];
                        bv[c] = two ? pl[rr1] : R(0);
                    }
                    const R px = z0.x + beta * o0.x, py = z0.y + beta * o0.y, pz = z0.z + beta * o0.z;
                    const R qx = z1.x + beta * o1.x, qy = z1.y + beta * o1.y, qz = z1.z + beta * o1.z;
                    a0 += av[0] * px + av[1] * py + av[2] * pz + (bv[0] * qx + bv[1] * qy + bv[2] * qz);
                    a1 += av[3] * px + av[4] * py + av[5] * pz + (bv[3] * qx + bv[4] * qy + bv[5] * qz);
                    a2 += av[6] * px + av[7] * py + av[8] * pz + (bv[6] * qx + bv[7] * qy + bv[8] * qz);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[s]);
#pragma unroll
                for (int o = 4; o > 0; o >>= 1) {
                    a0 += __shfl_xor_sync(0xffffffffu, a0, o, 8);
                    a1 += __shfl_xor_sync(0xffffffffu, a1, o, 8);
                    a2 += __shfl_xor_sync(0xffffffffu, a2, o, 8);
                }
                if (sub == 0 && valid) {
                    if (!mk) a0 = a1 = a2 = 0;
                    typename V4<R>::T qv, pv;
                    qv.x = a0; qv.y = a1; qv.z = a2; qv.w = 0;
                    pv.x = own0; pv.y = own1; pv.z = own2; pv.w = 0;
                    st4(q, v, qv);
                    st4(pnew, v, pv);
                    pq += (double)own0 * a0 + (double)own1 * a1 + (double)own2 * a2;
                }
            }
        }
        CG_MARK(0);   // this thread's matvec work
        pq = block_reduce<ROP_SUM>(pq);
        CG_MARK(1);   // the CTA's other warps
        if (threadIdx.x == 0) part_pq[blockIdx.x] = pq;
        grid_barrier_t<R>(bar_count, bar_gen, gridDim.x);
        const double pqs = grid_sum_partials(part_pq, gridDim.x, &sm_tot);
        CG_MARK(2);   // grid barrier 1 (the other CTAs)
        if (blockIdx.x == 0 && threadIdx.x == 0 && pqs < 0.0) atomicAdd(&err[ERR_NOT_SPD], 1ull);
        rho = rz_new;                   // rho_k = r_k . z_k (beta above used the previous rho)
        first = 0;
        cur ^= 1;
        const R alpha = (pqs != 0.0) ? (R)(rho / pqs) : R(0);
        // update phase over every thread of the grid
        double acc = 0.0;
        for (uint64_t vv = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; vv < nv; vv += gthreads) {
            const auto pv = ld4cg(pnew, vv);
            const auto qv = ld4cg(q, vv);
            const auto dv = ld4(dinv, vv);
            auto rv = ld4(r, vv);
            rv.x -= alpha * qv.x;
            rv.y -= alpha * qv.y;
            rv.z -= alpha * qv.z;
            typename V4<R>::T zv;
            zv.x = rv.x * dv.x;
            zv.y = rv.y * dv.y;
            zv.z = rv.z * dv.z;
            zv.w = 0;
            st4(r, vv, rv);
            st4(z, vv, zv);
            x[3 * vv] += alpha * pv.x;
            x[3 * vv + 1] += alpha * pv.y;
            x[3 * vv + 2] += alpha * pv.z;
            acc += (double)rv.x * zv.x + (double)rv.y * zv.y + (double)rv.z * zv.z;
        }
        acc = block_reduce<ROP_SUM>(acc);
        CG_MARK(3);   // update phase
        if (threadIdx.x == 0) part_rz[blockIdx.x] = acc;
        grid_barrier_t<R>(bar_count, bar_gen, gridDim.x);
        rz_new = grid_sum_partials(part_rz, gridDim.x, &sm_tot);
        CG_MARK(4);   // grid barrier 2
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            scal[S_PQ] = pqs;
            *rho_user = rz_new;
        }
        ++done_it;
        if (tol2 > 0.0 && rz_new <= tol2 * rz0) {   // same value in every CTA: a uniform exit
            conv = true;
            break;
        }
    }
    // an early exit leaves the next iteration's prefetched chunks in flight
    if (warp == TMA_CONSUMERS && lane == 0)
        for (uint64_t sq = (uint64_t)done_it * my_chunks; sq < issued; ++sq)
            mbar_wait(&full_bar[sq % TMA_NS], (uint32_t)((sq / TMA_NS) & 1u));
#ifdef CG_PROF
    if (threadIdx.x == 0) {
        for (int q = 0; q < 5; ++q) atomicAdd(&g_cg_prof[q], (unsigned long long)cg_tp[q]);
        atomicAdd(&g_cg_prof[5], 1ull);
        atomicAdd(&g_cg_prof[6], (unsigned long long)done_it);
    }
#endif
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        scal[S_RHO] = rho;
        scal[S_RZ] = rz_new;
        scal[S_FIRST] = first ? 1.0 : 0.0;
        scal[S_PAR] = cur ? 1.0 : 0.0;
        scal[S_ITERS] += (double)done_it;
        if (conv) scal[S_DONE] = 1.0;
    }
}

// ---------------------------------------------------------------------------
// Symmetric-storage persistent PCG (Saad Alg. 9.1 iterates): A = A^T
// (the stiffness of edge (a, b) is the transpose of (b, a)), so the
// matvec streams only the upper triangle (rows tail <= head: ~half the bytes
// of A, the dominant stream of every iteration).  Row (v, w) of the upper
// CSR adds A_vw p_w to q_v (owner, in registers) and, for w != v, A_vw^T p_v
// to q_w with red.global.add (the paper's field `+=`) -- q is zeroed
// by the update phase of the previous iteration.  p.q needs no q:
//   p.q = sum_v p_v.A_vv p_v + 2 sum_{v<w} p_v.A_vw p_w,
// accumulated from the streamed blocks, so the structure is Saad's: matvec
// phase -> grid barrier -> update phase (reads the complete q) -> barrier.
template <typename R>
__global__ void __launch_bounds__(32 * (TMA_CONSUMERS + 1), 3)
    k_cg_sym_persistent(uint64_t nv, const uint32_t* __restrict__ index, const uint32_t* __restrict__ head,
                        const R* __restrict__ A, uint64_t ne, R* __restrict__ z, R* pb0, R* pb1, R* __restrict__ q,
                        const R* __restrict__ dinv, R* __restrict__ x, R* __restrict__ r,
                        const uint8_t* __restrict__ mask, double* __restrict__ part_pq, double* __restrict__ part_rz,
                        unsigned int* __restrict__ bar_count, unsigned int* __restrict__ bar_gen,
                        double* __restrict__ scal, double* __restrict__ rho_user, unsigned long long* __restrict__ err,
                        uint32_t cap, int iters, double tol2) {
    extern __shared__ __align__(128) unsigned char tma_smem[];
    __shared__ __align__(8) uint64_t full_bar[TMA_NS], empty_bar[TMA_NS];
    __shared__ double sm_tot;
    constexpr uint32_t AE = 16 / sizeof(R);
    const size_t stage_bytes = ((size_t)9 * cap * sizeof(R) + (size_t)cap * 4 + 127) & ~(size_t)127;
    const uint64_t nchunks = (nv + TMA_VCH - 1) / TMA_VCH;
    const uint64_t my_chunks = nchunks > blockIdx.x ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < TMA_NS; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], PCG_WPG);
        }
        mbar_fence_init();
    }
    __syncthreads();
    double rho = scal[S_RHO];
    int first = scal[S_FIRST] != 0.0;
    int cur = scal[S_PAR] != 0.0;
    double rz_new = scal[S_RZ];
    const double rz0 = scal[S_RZ0];
    if (scal[S_DONE] != 0.0) iters = 0;
    int done_it = 0;
    bool conv = false;
    uint64_t issued = 0;
    auto issue = [&](uint64_t ch, uint64_t seq) {
        const int s = seq % TMA_NS;
        const uint64_t v0 = ch * TMA_VCH;
        const uint64_t v1 = v0 + TMA_VCH < nv ? v0 + TMA_VCH : nv;
        const uint64_t e0 = index[v0], e1 = index[v1];
        if (seq >= TMA_NS) mbar_wait(&empty_bar[s], (uint32_t)(((seq / TMA_NS) + 1) & 1u));
        unsigned char* base = tma_smem + s * stage_bytes;
        uint32_t tot = 0;
#pragma unroll
        for (int c = 0; c < 9; ++c) {
            const uint64_t a0 = (c * ne + e0) & ~(uint64_t)(AE - 1);
            const uint64_t a1 = (c * ne + e1 + AE - 1) & ~(uint64_t)(AE - 1);
            tot += (uint32_t)((a1 - a0) * sizeof(R));
        }
        const uint64_t h0 = e0 & ~3ull, h1 = (e1 + 3) & ~3ull;
        tot += (uint32_t)((h1 - h0) * 4);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&full_bar[s], tot);
#pragma unroll
        for (int c = 0; c < 9; ++c) {
            const uint64_t a0 = (c * ne + e0) & ~(uint64_t)(AE - 1);
            const uint64_t a1 = (c * ne + e1 + AE - 1) & ~(uint64_t)(AE - 1);
            bulk_g2s_evict_first(base + (size_t)c * cap * sizeof(R), A + a0, (uint32_t)((a1 - a0) * sizeof(R)),
                                 &full_bar[s]);
        }
        bulk_g2s_evict_first(base + (size_t)9 * cap * sizeof(R), head + h0, (uint32_t)((h1 - h0) * 4), &full_bar[s]);
    };
    if (iters > 0 && warp == TMA_CONSUMERS && lane == 0)
        for (uint64_t j = 0; j < my_chunks && j < TMA_NS; ++j) issue(blockIdx.x + j * gridDim.x, issued++);
    const uint64_t gthreads = (uint64_t)gridDim.x * blockDim.x;
#ifdef CG_PROF
    __shared__ long long cg_tp[5], cg_t0[1];
    if (threadIdx.x == 0) {
        for (int q = 0; q < 5; ++q) cg_tp[q] = 0;
        cg_t0[0] = clock64();
    }
#endif
    for (int it = 0; it < iters; ++it) {
        const R beta = (first || rho == 0.0) ? R(0) : (R)(rz_new / rho);
        const R* __restrict__ pold = cur ? pb1 : pb0;
        R* __restrict__ pnew = cur ? pb0 : pb1;
        double pq = 0.0;
        if (warp == TMA_CONSUMERS) {
            if (lane == 0) {
                for (uint64_t j = TMA_NS; j < my_chunks; ++j) issue(blockIdx.x + j * gridDim.x, issued++);
                if (it + 1 < iters)
                    for (uint64_t j = 0; j < my_chunks && j < TMA_NS; ++j) issue(blockIdx.x + j * gridDim.x, issued++);
            }
        } else {
            const unsigned grp = warp / PCG_WPG, wig = warp % PCG_WPG;
            const unsigned sub = lane & 7;
            const uint64_t seq0 = (uint64_t)it * my_chunks;
            for (uint64_t j = grp; j < my_chunks; j += PCG_GROUPS) {
                const uint64_t seq = seq0 + j;
                const uint64_t ch = blockIdx.x + j * gridDim.x;
                const int s = seq % TMA_NS;
                const uint64_t v0 = ch * TMA_VCH;
                const uint64_t v1 = v0 + TMA_VCH < nv ? v0 + TMA_VCH : nv;
                const uint64_t v = v0 + 4 * wig + (lane >> 3);
                const bool valid = v < v1;
                const uint32_t e0 = index[v0];
                const uint32_t r0 = valid ? index[v] - e0 : 0u, r1 = valid ? index[v + 1] - e0 : 0u;
                R own0 = 0, own1 = 0, own2 = 0;
                if (valid && sub == 0) {
                    const auto zv = ld4cg(z, v);
                    const auto ov = ld4cg(pold, v);
                    own0 = zv.x + beta * ov.x;
                    own1 = zv.y + beta * ov.y;
                    own2 = zv.z + beta * ov.z;
                }
                // p_v to every lane of the vertex (the transposed blocks need it)
                const int src = (int)(lane & ~7u);
                const R pv0 = __shfl_sync(0xffffffffu, own0, src);
                const R pv1 = __shfl_sync(0xffffffffu, own1, src);
                const R pv2 = __shfl_sync(0xffffffffu, own2, src);
                mbar_wait(&full_bar[s], (uint32_t)((seq / TMA_NS) & 1u));
                const unsigned char* base = tma_smem + s * stage_bytes;
                const uint32_t* hs = reinterpret_cast<const uint32_t*>(base + (size_t)9 * cap * sizeof(R)) + (e0 & 3u);
                uint32_t off[9];
#pragma unroll
                for (int c = 0; c < 9; ++c) off[c] = (uint32_t)((c * ne + e0) & (AE - 1));
                R a0 = 0, a1 = 0, a2 = 0;
                double dsum = 0.0;
                for (uint32_t rb = r0 + sub; rb < r1; rb += 8) {
                    const uint32_t h = hs[rb];
                    const auto zh = ld4cg(z, h);
                    const auto oh = ld4cg(pold, h);
                    R av[9];
#pragma unroll
                    for (int c = 0; c < 9; ++c)
                        av[c] = reinterpret_cast<const R*>(base + (size_t)c * cap * sizeof(R))[off[c] + rb];
                    const R px = zh.x + beta * oh.x, py = zh.y + beta * oh.y, pz = zh.z + beta * oh.z;
                    const R m0 = av[0] * px + av[1] * py + av[2] * pz;
                    const R m1 = av[3] * px + av[4] * py + av[5] * pz;
                    const R m2 = av[6] * px + av[7] * py + av[8] * pz;
                    a0 += m0;
                    a1 += m1;
                    a2 += m2;
                    const double d = (double)pv0 * m0 + (double)pv1 * m1 + (double)pv2 * m2;
                    if (h != (uint32_t)v) {
                        dsum += 2.0 * d;
                        // q_h += A_vh^T p_v
                        atomicAdd(q + 4ull * h + 0, av[0] * pv0 + av[3] * pv1 + av[6] * pv2);
                        atomicAdd(q + 4ull * h + 1, av[1] * pv0 + av[4] * pv1 + av[7] * pv2);
                        atomicAdd(q + 4ull * h + 2, av[2] * pv0 + av[5] * pv1 + av[8] * pv2);
                    } else {
                        dsum += d;
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[s]);
#pragma unroll
                for (int o = 4; o > 0; o >>= 1) {
                    a0 += __shfl_xor_sync(0xffffffffu, a0, o, 8);
                    a1 += __shfl_xor_sync(0xffffffffu, a1, o, 8);
                    a2 += __shfl_xor_sync(0xffffffffu, a2, o, 8);
                }
                pq += dsum;
                if (sub == 0 && valid) {
                    atomicAdd(q + 4ull * v + 0, a0);
                    atomicAdd(q + 4ull * v + 1, a1);
                    atomicAdd(q + 4ull * v + 2, a2);
                    typename V4<R>::T pv;
                    pv.x = own0; pv.y = own1; pv.z = own2; pv.w = 0;
                    st4(pnew, v, pv);
                }
            }
        }
        pq = block_reduce<ROP_SUM>(pq);
        if (threadIdx.x == 0) part_pq[blockIdx.x] = pq;
        grid_barrier_t<R>(bar_count, bar_gen, gridDim.x);
        const double pqs = grid_sum_partials(part_pq, gridDim.x, &sm_tot);
        if (blockIdx.x == 0 && threadIdx.x == 0 && pqs < 0.0) atomicAdd(&err[ERR_NOT_SPD], 1ull);
        rho = rz_new;
        first = 0;
        cur ^= 1;
        const R alpha = (pqs != 0.0) ? (R)(rho / pqs) : R(0);
        double acc = 0.0;
        typename V4<R>::T zero4;
        zero4.x = zero4.y = zero4.z = zero4.w = R(0);
        for (uint64_t vv = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; vv < nv; vv += gthreads) {
            const auto pv = ld4cg(pnew, vv);
            auto qv = ld4cg(q, vv);
            st4(q, vv, zero4);                       // ready for the next iteration's red.add
            if (mask && !mask[vv]) qv = zero4;       // q = (A p) * mask
            const auto dv = ld4(dinv, vv);
            auto rv = ld4(r, vv);
            rv.x -= alpha * qv.x;
            rv.y -= alpha * qv.y;
            rv.z -= alpha * qv.z;
            typename V4<R>::T zv;
            zv.x = rv.x * dv.x;
            zv.y = rv.y * dv.y;
            zv.z = rv.z * dv.z;
            zv.w = 0;
            st4(r, vv, rv);
            st4(z, vv, zv);
            x[3 * vv] += alpha * pv.x;
            x[3 * vv + 1] += alpha * pv.y;
            x[3 * vv + 2] += alpha * pv.z;
            acc += (double)rv.x * zv.x + (double)rv.y * zv.y + (double)rv.z * zv.z;
        }
        acc = block_reduce<ROP_SUM>(acc);
        CG_MARK(3);   // update phase
        if (threadIdx.x == 0) part_rz[blockIdx.x] = acc;
        grid_barrier_t<R>(bar_count, bar_gen, gridDim.x);
        rz_new = grid_sum_partials(part_rz, gridDim.x, &sm_tot);
        CG_MARK(4);   // grid barrier 2
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            scal[S_PQ] = pqs;
            *rho_user = rz_new;
        }
        ++done_it;
        if (tol2 > 0.0 && rz_new <= tol2 * rz0) {
            conv = true;
            break;
        }
    }
    if (warp == TMA_CONSUMERS && lane == 0)
        for (uint64_t sq = (uint64_t)done_it * my_chunks; sq < issued; ++sq)
            mbar_wait(&full_bar[sq % TMA_NS], (uint32_t)((sq / TMA_NS) & 1u));
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        scal[S_RHO] = rho;
        scal[S_RZ] = rz_new;
        scal[S_FIRST] = first ? 1.0 : 0.0;
        scal[S_PAR] = cur ? 1.0 : 0.0;
        scal[S_ITERS] += (double)done_it;
        if (conv) scal[S_DONE] = 1.0;
    }
}

// upper-triangle CSR of a grouped edge relation
__global__ void k_upper_count(uint64_t nv, const uint32_t* __restrict__ index, const uint32_t* __restrict__ head,
                              uint32_t* __restrict__ rself, uint32_t* __restrict__ cnt) {
    const uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (v >= nv) return;
    uint32_t lo = index[v], hi = index[v + 1];
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (head[mid] < (uint32_t)v) lo = mid + 1;
        else hi = mid;
    }
    rself[v] = lo;
    cnt[v] = index[v + 1] - lo;
}

__global__ void k_upper_fill(uint64_t nv, const uint32_t* __restrict__ head, const uint32_t* __restrict__ rself,
                             const uint32_t* __restrict__ uptr, uint32_t* __restrict__ uhead,
                             uint32_t* __restrict__ usrc) {
    const uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (v >= nv) return;
    const uint32_t n = uptr[v + 1] - uptr[v];
    for (uint32_t j = 0; j < n; ++j) {
        uhead[uptr[v] + j] = head[rself[v] + j];
        usrc[uptr[v] + j] = rself[v] + j;
    }
}

template <typename R>
__global__ void k_compress_upper(uint64_t nu, uint64_t ne, const uint32_t* __restrict__ usrc, const R* __restrict__ A,
                                 R* __restrict__ Ah) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= nu) return;
    const uint64_t src = usrc[k];
#pragma unroll
    for (int c = 0; c < 9; ++c) Ah[(uint64_t)c * nu + k] = A[(uint64_t)c * ne + src];
}

// ---------------------------------------------------------------------------
// Single-reduction persistent PCG (Chronopoulos-Gear):
// the same iterates as Saad Alg. 9.1 in exact arithmetic, with ONE grid
// barrier and ONE gathered vector per iteration (Saad: two barriers, two
// gathered vectors).  D = diag(A)^-1 (Jacobi), all operators masked.
//   s_i = w_i + b_i s_{i-1} (= A p_i),  p_i = z_i + b_i p_{i-1},
//   y_i = A u_i + b_i y_{i-1} (= A D s_i),  u_i = D w_i,
//   x_{i+1} = x_i + a_i p_i,  r_{i+1} = r_i - a_i s_i,  z_{i+1} = D r_{i+1},
//   w_{i+1} = w_i - a_i y_i (= A z_{i+1}),  u_{i+1} = D w_{i+1},
//   g_{i+1} = r.z,  d_{i+1} = w.z  (one fused reduction),
//   b_{i+1} = g_{i+1} / g_i,  a_{i+1} = g_{i+1} / (d_{i+1} - b_{i+1} g_{i+1} / a_i).
// The matvec operand u_i is complete when the phase starts (it does not
// depend on a_i, b_i), so each phase is: stream A, gather u_i, and the owner
// of each vertex applies every recurrence as it finishes the vertex's row.
// Only u is read by neighbours (double-buffered); the rest is owner-local.
// The first call after ebb_cg_init runs one extra matvec (w_0 = A z_0).
// The body is shared by two kernels that differ only in their launch bounds
// (measured, profiles/r02_cg1_launch_bounds.jsonl): fp64 with min 3 CTAs per
// SM (72 registers, no spills; without a min-blocks ptxas keeps 72 but
// spills 56 bytes and runs 2.7 % slower at C2; min 1 takes 146 and runs
// 1.45x slower), fp32 without one (72 registers, no spills).
template <typename R>
__device__ __forceinline__ void cg1_persistent_body(uint64_t nv, const uint32_t* __restrict__ index, const uint32_t* __restrict__ head,
                     const R* __restrict__ A, uint64_t ne, const R* __restrict__ dinv, R* __restrict__ x,
                     R* __restrict__ r, const R* __restrict__ z0, R* __restrict__ p, R* __restrict__ sv,
                     R* __restrict__ yv, R* __restrict__ wv, R* ub0, R* ub1, const uint8_t* __restrict__ mask,
                     double* __restrict__ part_g, double* __restrict__ part_d, unsigned int* __restrict__ bar_count,
                     unsigned int* __restrict__ bar_gen, double* __restrict__ scal, double* __restrict__ rho_user,
                     unsigned long long* __restrict__ err, uint32_t cap, int iters,
                     double tol2, int dist) {
    extern __shared__ __align__(128) unsigned char tma_smem[];
    __shared__ __align__(8) uint64_t full_bar[CG1_NS], empty_bar[CG1_NS];
    __shared__ double sm_tot;
    constexpr uint32_t AE = 16 / sizeof(R);
    const size_t stage_bytes = ((size_t)9 * cap * sizeof(R) + (size_t)cap * 4 + 127) & ~(size_t)127;
    const uint64_t nchunks = (nv + TMA_VCH - 1) / TMA_VCH;
    const uint64_t my_chunks = nchunks > blockIdx.x ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < CG1_NS; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], PCG_WPG);
        }
        mbar_fence_init();
    }
    __syncthreads();
    // scalars (identical in every CTA)
    double gam = scal[S_RHO];                 // g_i = r_i . z_i
    double alpha = scal[S_ALPHA];             // a_i
    double beta = scal[S_PQ];                 // b_i
    int first = scal[S_FIRST] != 0.0;         // w_0 not yet formed
    int par = scal[S_PAR] != 0.0;             // u_i in buffer par
    const double rz0 = scal[S_RZ0];
    if (scal[S_DONE] != 0.0) iters = 0;       // converged in an earlier call (tolerance mode)
    int done_it = 0, done_ph = 0;
    bool conv = false;
    if (dist && scal[S_VAR] != 0.0 && scal[S_DONE] == 0.0) {
        // multi-GPU phase mode: finish the previous phase's scalar recurrences
        // from the globally summed (allreduced) w.z and r.z -- the same
        // formulas as below, every CTA reads the same slots
        const double dsum = scal[S_DSUM];
        if (scal[S_VAR] == 1.0) {
            if (blockIdx.x == 0 && threadIdx.x == 0 && dsum < 0.0) atomicAdd(&err[ERR_NOT_SPD], 1ull);
            alpha = dsum != 0.0 ? gam / dsum : 0.0;
            beta = 0.0;
            first = 0;
        } else {
            const double gnew = scal[S_GSUM];
            const double bn = gam != 0.0 ? gnew / gam : 0.0;
            const double den = dsum - (alpha != 0.0 ? bn * gnew / alpha : 0.0);
            if (blockIdx.x == 0 && threadIdx.x == 0 && den < 0.0) atomicAdd(&err[ERR_NOT_SPD], 1ull);
            alpha = den != 0.0 ? gnew / den : 0.0;
            beta = bn;
            gam = gnew;
            par ^= 1;
            if (blockIdx.x == 0 && threadIdx.x == 0) *rho_user = gam;
            if (tol2 > 0.0 && gam <= tol2 * rz0) {
                conv = true;
                iters = 0;
            }
        }
    }
    uint64_t issued = 0;
    auto issue = [&](uint64_t ch, uint64_t seq) {
        const int s = seq % CG1_NS;
        const uint64_t v0 = ch * TMA_VCH;
        const uint64_t v1 = v0 + TMA_VCH < nv ? v0 + TMA_VCH : nv;
        const uint64_t e0 = index[v0], e1 = index[v1];
        if (seq >= CG1_NS) mbar_wait(&empty_bar[s], (uint32_t)(((seq / CG1_NS) + 1) & 1u));
        unsigned char* base = tma_smem + s * stage_bytes;
        uint32_t tot = 0;
#pragma unroll
        for (int c = 0; c < 9; ++c) {
            const uint64_t a0 = (c * ne + e0) & ~(uint64_t)(AE - 1);
            const uint64_t a1 = (c * ne + e1 + AE - 1) & ~(uint64_t)(AE - 1);
            tot += (uint32_t)((a1 - a0) * sizeof(R));
        }
        const uint64_t h0 = e0 & ~3ull, h1 = (e1 + 3) & ~3ull;
        tot += (uint32_t)((h1 - h0) * 4);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&full_bar[s], tot);
#pragma unroll
        for (int c = 0; c < 9; ++c) {
            const uint64_t a0 = (c * ne + e0) & ~(uint64_t)(AE - 1);
            const uint64_t a1 = (c * ne + e1 + AE - 1) & ~(uint64_t)(AE - 1);
            bulk_g2s_evict_first(base + (size_t)c * cap * sizeof(R), A + a0, (uint32_t)((a1 - a0) * sizeof(R)),
                                 &full_bar[s]);
        }
        bulk_g2s_evict_first(base + (size_t)9 * cap * sizeof(R), head + h0, (uint32_t)((h1 - h0) * 4), &full_bar[s]);
    };
    const int nphase = dist ? (iters > 0 ? 1 : 0) : iters + (first && iters > 0 ? 1 : 0);
    if (warp == TMA_CONSUMERS && lane == 0 && nphase > 0)
        for (uint64_t j = 0; j < my_chunks && j < CG1_NS; ++j) issue(blockIdx.x + j * gridDim.x, issued++);
    for (int ph = 0; ph < nphase; ++ph) {
        const bool pro = first != 0;          // prologue: w_0 = A z_0, u_0 = D w_0
        const R a = (R)alpha, b = (R)beta;
        const R* __restrict__ op = pro ? z0 : (par ? ub1 : ub0);   // the gathered operand (z_0 or u_i)
        R* __restrict__ un = pro ? (par ? ub1 : ub0) : (par ? ub0 : ub1);   // u_0 in place / u_{i+1}
        double pg = 0.0, pd = 0.0;
        if (warp == TMA_CONSUMERS) {
            if (lane == 0) {
                for (uint64_t j = CG1_NS; j < my_chunks; ++j) issue(blockIdx.x + j * gridDim.x, issued++);
                if (ph + 1 < nphase)
                    for (uint64_t j = 0; j < my_chunks && j < CG1_NS; ++j) issue(blockIdx.x + j * gridDim.x, issued++);
            }
        } else {
            const unsigned grp = warp / PCG_WPG, wig = warp % PCG_WPG;
            const unsigned sub = lane & 7;
            const uint64_t seq0 = (uint64_t)ph * my_chunks;
            for (uint64_t j = grp; j < my_chunks; j += PCG_GROUPS) {
                const uint64_t seq = seq0 + j;
                const uint64_t ch = blockIdx.x + j * gridDim.x;
                const int s = seq % CG1_NS;
                const uint64_t v0 = ch * TMA_VCH;
                const uint64_t v1 = v0 + TMA_VCH < nv ? v0 + TMA_VCH : nv;
                const uint64_t v = v0 + 4 * wig + (lane >> 3);
                const bool valid = v < v1;
                const uint32_t e0 = index[v0];
                const uint32_t r0 = valid ? index[v] - e0 : 0u, r1 = valid ? index[v + 1] - e0 : 0u;
                mbar_wait(&full_bar[s], (uint32_t)((seq / CG1_NS) & 1u));
                const unsigned char* base = tma_smem + s * stage_bytes;
                const uint32_t* hs = reinterpret_cast<const uint32_t*>(base + (size_t)9 * cap * sizeof(R)) + (e0 & 3u);
                uint32_t off[9];
#pragma unroll
                for (int c = 0; c < 9; ++c) off[c] = (uint32_t)((c * ne + e0) & (AE - 1));
                R a0 = 0, a1 = 0, a2 = 0;
                for (uint32_t rb = r0 + sub; rb < r1; rb += 16) {
                    // two rows per lane per pass: both gathers in flight together
                    const uint32_t rr1 = rb + 8;
                    const bool two = rr1 < r1;
                    const uint32_t h0 = hs[rb], h1 = two ? hs[rr1] : h0;
                    const auto o0 = ld4cg(op, h0);
                    const auto o1 = ld4cg(op, h1);
                    R av[9], bv[9];
#pragma unroll
                    for (int c = 0; c < 9; ++c) {
                        const R* pl = reinterpret_cast<const R*>(base + (size_t)c * cap * sizeof(R)) + off[c];
                        av[c] = pl[rb];
                        bv[c] = two ? pl[rr1] : R(0);
                    }
                    a0 += av[0] * o0.x + av[1] * o0.y + av[2] * o0.z + (bv[0] * o1.x + bv[1] * o1.y + bv[2] * o1.z);
                    a1 += av[3] * o0.x + av[4] * o0.y + av[5] * o0.z + (bv[3] * o1.x + bv[4] * o1.y + bv[5] * o1.z);
                    a2 += av[6] * o0.x + av[7] * o0.y + av[8] * o0.z + (bv[6] * o1.x + bv[7] * o1.y + bv[8] * o1.z);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[s]);
#pragma unroll
                for (int o = 4; o > 0; o >>= 1) {
                    a0 += __shfl_xor_sync(0xffffffffu, a0, o, 8);
                    a1 += __shfl_xor_sync(0xffffffffu, a1, o, 8);
                    a2 += __shfl_xor_sync(0xffffffffu, a2, o, 8);
                }
                if (sub == 0 && valid) {
                    if (mask && !mask[v]) a0 = a1 = a2 = 0;   // m = (A op) * mask
                    const auto dv = ld4(dinv, v);
                    typename V4<R>::T t;
                    t.w = 0;
                    if (pro) {
                        // w_0 = A z_0, u_0 = D w_0, d_0 = w_0 . z_0
                        const auto zv = ld4(z0, v);
                        t.x = a0; t.y = a1; t.z = a2;
                        st4(wv, v, t);
                        t.x = a0 * dv.x; t.y = a1 * dv.y; t.z = a2 * dv.z;
                        st4(un, v, t);
                        pd += (double)a0 * zv.x + (double)a1 * zv.y + (double)a2 * zv.z;
                    } else {
                        auto rv = ld4(r, v);
                        auto wi = ld4(wv, v);
                        typename V4<R>::T si = wi, yi, pi;
                        yi.x = a0; yi.y = a1; yi.z = a2; yi.w = 0;
                        pi.x = rv.x * dv.x; pi.y = rv.y * dv.y; pi.z = rv.z * dv.z; pi.w = 0;   // z_i
                        if (b != R(0)) {
                            const auto so = ld4(sv, v), yo = ld4(yv, v), po = ld4(p, v);
                            si.x += b * so.x; si.y += b * so.y; si.z += b * so.z;
                            yi.x += b * yo.x; yi.y += b * yo.y; yi.z += b * yo.z;
                            pi.x += b * po.x; pi.y += b * po.y; pi.z += b * po.z;
                        }
                        si.w = 0;
                        st4(sv, v, si);
                        st4(yv, v, yi);
                        st4(p, v, pi);
                        x[3 * v] += a * pi.x;
                        x[3 * v + 1] += a * pi.y;
                        x[3 * v + 2] += a * pi.z;
                        rv.x -= a * si.x; rv.y -= a * si.y; rv.z -= a * si.z; rv.w = 0;
                        wi.x -= a * yi.x; wi.y -= a * yi.y; wi.z -= a * yi.z; wi.w = 0;
                        st4(r, v, rv);
                        st4(wv, v, wi);
                        t.x = wi.x * dv.x; t.y = wi.y * dv.y; t.z = wi.z * dv.z;
                        st4(un, v, t);
                        const R zx = rv.x * dv.x, zy = rv.y * dv.y, zz = rv.z * dv.z;
                        pg += (double)rv.x * zx + (double)rv.y * zy + (double)rv.z * zz;
                        pd += (double)wi.x * zx + (double)wi.y * zy + (double)wi.z * zz;
                    }
                }
            }
        }
        pg = block_reduce<ROP_SUM>(pg);
        pd = block_reduce<ROP_SUM>(pd);
        // one grid barrier per phase: the partial slots alternate by phase
        // parity, so a CTA that leaves the barrier first and writes the next
        // phase's partials cannot overwrite ones a slower CTA is still summing
        // (it reaches the phase after next only once every CTA has passed the
        // next barrier, i.e. has finished reading this phase's slots)
        double* const pgb = part_g + (ph & 1) * kCg1PartStride;
        double* const pdb = part_d + (ph & 1) * kCg1PartStride;
        if (threadIdx.x == 0) {
            pgb[blockIdx.x] = pg;
            pdb[blockIdx.x] = pd;
        }
        grid_barrier_t<R>(bar_count, bar_gen, gridDim.x);
        const double dsum = grid_sum_partials(pdb, gridDim.x, &sm_tot);
        if (dist) {
            // phase mode: publish the rank-local sums; the recurrences finish
            // at the next launch, after the host's allreduce of S_DSUM..S_GSUM
            const double gl = pro ? 0.0 : grid_sum_partials(pgb, gridDim.x, &sm_tot);
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                scal[S_DSUM] = dsum;
                scal[S_GSUM] = gl;
                scal[S_VAR] = pro ? 1.0 : 2.0;
            }
            ++done_ph;
            if (!pro) ++done_it;
            break;
        }
        if (pro) {
            // a_0 = g_0 / (p_0 . A p_0), p_0 = z_0
            if (blockIdx.x == 0 && threadIdx.x == 0 && dsum < 0.0) atomicAdd(&err[ERR_NOT_SPD], 1ull);
            alpha = dsum != 0.0 ? gam / dsum : 0.0;
            beta = 0.0;
            first = 0;
        } else {
            const double gnew = grid_sum_partials(pgb, gridDim.x, &sm_tot);
            const double bn = gam != 0.0 ? gnew / gam : 0.0;
            const double den = dsum - (alpha != 0.0 ? bn * gnew / alpha : 0.0);   // = p_{i+1} . A p_{i+1}
            if (blockIdx.x == 0 && threadIdx.x == 0 && den < 0.0) atomicAdd(&err[ERR_NOT_SPD], 1ull);
            alpha = den != 0.0 ? gnew / den : 0.0;
            beta = bn;
            gam = gnew;
            par ^= 1;
            if (blockIdx.x == 0 && threadIdx.x == 0) *rho_user = gam;
        }
        ++done_ph;
        if (!pro) {
            ++done_it;
            if (tol2 > 0.0 && gam <= tol2 * rz0) {   // same value in every CTA: a uniform exit
                conv = true;
                break;
            }
        }
    }
    // an early exit leaves the next phase's prefetched chunks in flight
    if (warp == TMA_CONSUMERS && lane == 0)
        for (uint64_t sq = (uint64_t)done_ph * my_chunks; sq < issued; ++sq)
            mbar_wait(&full_bar[sq % CG1_NS], (uint32_t)((sq / CG1_NS) & 1u));
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        scal[S_ITERS] += (double)done_it;
        if (conv) scal[S_DONE] = 1.0;
        if (dist && done_ph == 0) scal[S_VAR] = 0.0;   // pending scalars consumed, no new phase
        scal[S_RHO] = gam;
        scal[S_RZ] = gam;
        scal[S_ALPHA] = alpha;
        scal[S_PQ] = beta;
        scal[S_FIRST] = first ? 1.0 : 0.0;
        scal[S_PAR] = par ? 1.0 : 0.0;
    }
}

#define EBB_CG1_PARAMS                                                                                              \
    uint64_t nv, const uint32_t *__restrict__ index, const uint32_t *__restrict__ head, const R *__restrict__ A,  \
        uint64_t ne, const R *__restrict__ dinv, R *__restrict__ x, R *__restrict__ r, const R *__restrict__ z0,    \
        R *__restrict__ p, R *__restrict__ sv, R *__restrict__ yv, R *__restrict__ wv, R *ub0, R *ub1,              \
        const uint8_t *__restrict__ mask, double *__restrict__ part_g, double *__restrict__ part_d,                  \
        unsigned int *__restrict__ bar_count, unsigned int *__restrict__ bar_gen, double *__restrict__ scal,        \
        double *__restrict__ rho_user, unsigned long long *__restrict__ err, uint32_t cap, int iters, double tol2,   \
        int dist
#define EBB_CG1_ARGS                                                                                                \
    nv, index, head, A, ne, dinv, x, r, z0, p, sv, yv, wv, ub0, ub1, mask, part_g, part_d, bar_count, bar_gen,     \
        scal, rho_user, err, cap, iters, tol2, dist
template <typename R>
__global__ void __launch_bounds__(32 * (TMA_CONSUMERS + 1), 3) k_cg1_persistent_f64(EBB_CG1_PARAMS) {
    cg1_persistent_body<R>(EBB_CG1_ARGS);
}
template <typename R>
__global__ void __launch_bounds__(32 * (TMA_CONSUMERS + 1)) k_cg1_persistent_f32(EBB_CG1_PARAMS) {
    cg1_persistent_body<R>(EBB_CG1_ARGS);
}
#undef EBB_CG1_PARAMS
#undef EBB_CG1_ARGS
// the kernel of a dtype
template <typename R>
constexpr auto cg1_kernel() {
    if constexpr (sizeof(R) == 8) return k_cg1_persistent_f64<R>;
    else return k_cg1_persistent_f32<R>;
}

// ---------------------------------------------------------------------------
// PCG kernels on padded vec4 work vectors (one thread per vertex)
// init: dinv = 1/diag(A) on free DOFs (Jacobi), x = 0, r = b*m,
//       z = r*dinv, p = z, local r.z -> scal[S_RZ]; scal[S_FIRST] = 1
template <typename R>
__global__ void __launch_bounds__(256) k_cg_init(uint64_t nv, const uint32_t* __restrict__ self,
                                                 const R* __restrict__ A, uint64_t ne, const R* __restrict__ b,
                                                 const uint8_t* __restrict__ mask, R* __restrict__ dinv,
                                                 R* __restrict__ x, R* __restrict__ r, R* __restrict__ z,
                                                 R* __restrict__ p, double* __restrict__ partials,
                                                 unsigned int* __restrict__ counter, double* __restrict__ scal,
                                                 double* __restrict__ rho_user) {
    double acc = 0.0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x) {
        const bool fr = !mask || mask[v];
        const uint32_t e = self[v];
        typename V4<R>::T dv, rv, zv;
        dv.x = fr ? R(1) / A[e] : R(0);
        dv.y = fr ? R(1) / A[4 * ne + e] : R(0);
        dv.z = fr ? R(1) / A[8 * ne + e] : R(0);
        dv.w = 0;
        rv.x = fr ? b[3 * v] : R(0);
        rv.y = fr ? b[3 * v + 1] : R(0);
        rv.z = fr ? b[3 * v + 2] : R(0);
        rv.w = 0;
        zv.x = rv.x * dv.x;
        zv.y = rv.y * dv.y;
        zv.z = rv.z * dv.z;
        zv.w = 0;
        st4(dinv, v, dv);
        st4(r, v, rv);
        st4(z, v, zv);
        st4(p, v, zv);
        x[3 * v] = 0;
        x[3 * v + 1] = 0;
        x[3 * v + 2] = 0;
        acc += (double)rv.x * zv.x + (double)rv.y * zv.y + (double)rv.z * zv.z;
    }
    double tot;
    if (block_sum_last_done(acc, partials, counter, &tot)) {
        scal[S_RZ] = tot;
        scal[S_RHO] = tot;
        scal[S_PQ] = 0.0;
        scal[S_FIRST] = 1.0;
        scal[S_PAR] = 0.0;
        scal[S_RZ0] = tot;
        scal[S_ITERS] = 0.0;
        scal[S_DONE] = 0.0;
        scal[S_VAR] = 0.0;
        if (rho_user) *rho_user = tot;
    }
}

// alpha = rho / p.q; x += alpha p; r -= alpha q; z = r*dinv; local r.z -> scal[S_RZ]
template <typename R>
__global__ void __launch_bounds__(256) k_cg_update(uint64_t nv, const R* pbuf0, const R* pbuf1, const R* __restrict__ q,
                                                   const R* __restrict__ dinv, R* __restrict__ x, R* __restrict__ r,
                                                   R* __restrict__ z, double* __restrict__ partials,
                                                   unsigned int* __restrict__ counter, double* __restrict__ scal,
                                                   double* __restrict__ rho_user, unsigned long long* __restrict__ err,
                                                   double tol2) {
    if (scal[S_DONE] != 0.0) return;   // converged (tolerance mode): the remaining launches are no-ops
    const double pqs = scal[S_PQ];
    const R alpha = (pqs != 0.0) ? (R)(scal[S_RHO] / pqs) : R(0);
    const R* __restrict__ p = scal[S_PAR] != 0.0 ? pbuf1 : pbuf0;   // the current direction
    double acc = 0.0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x) {
        const auto pv = ld4(p, v);
        const auto qv = ld4(q, v);
        const auto dv = ld4(dinv, v);
        auto rv = ld4(r, v);
        rv.x -= alpha * qv.x;
        rv.y -= alpha * qv.y;
        rv.z -= alpha * qv.z;
        typename V4<R>::T zv;
        zv.x = rv.x * dv.x;
        zv.y = rv.y * dv.y;
        zv.z = rv.z * dv.z;
        zv.w = 0;
        st4(r, v, rv);
        st4(z, v, zv);
        x[3 * v] += alpha * pv.x;
        x[3 * v + 1] += alpha * pv.y;
        x[3 * v + 2] += alpha * pv.z;
        acc += (double)rv.x * zv.x + (double)rv.y * zv.y + (double)rv.z * zv.z;
    }
    double tot;
    if (block_sum_last_done(acc, partials, counter, &tot)) {
        if (pqs < 0.0) atomicAdd(&err[ERR_NOT_SPD], 1ull);
        scal[S_RZ] = tot;
        if (rho_user) *rho_user = tot;
        scal[S_ITERS] += 1.0;
        if (tol2 > 0.0 && tot <= tol2 * scal[S_RZ0]) scal[S_DONE] = 1.0;
    }
}

// a9 in one pass over K: A = M + h D + h^2 K (D = alpha M + beta K) written
// row by row while the same rows accumulate (K v)_v, then
// b_v = h (f + M g - D v - h K v).  LPV lanes per vertex (shuffle reduce);
// A may alias K (every element is read, then written, by one thread).
template <typename R, int LPV, bool CONS, bool NEWTON>
__global__ void __launch_bounds__(256) k_assemble_fused(uint64_t nv, const uint32_t* __restrict__ index,
                                                        const uint32_t* __restrict__ head, const R* K, R* A,
                                                        uint64_t ne, const R* __restrict__ mass,
                                                        const R* __restrict__ f, const R* __restrict__ vel,
                                                        const R* __restrict__ vel0, R* __restrict__ b, R h, R alpha,
                                                        R beta, R g0, R g1, R g2) {
    // CONS: mass is the consistent edge mass (M_e = mass[e] I), M v and the
    // row sum for M g are accumulated with K v; else the lumped mass[v].
    // NEWTON: vel = the velocity iterate w, vel0 = v_n, and
    // b = h (f + M g - D w) + M (v_n - w) (no -h^2 K v term)
    const unsigned lane = threadIdx.x % LPV;
    const uint64_t v = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / LPV;
    const bool live = v < nv;   // every lane reaches the shuffles
    const R m = (!CONS && live) ? mass[v] : R(0);
    R k0 = 0, k1 = 0, k2 = 0, m0 = 0, m1 = 0, m2 = 0, ms = 0, n0 = 0, n1 = 0, n2 = 0;
    if (live) {
        for (uint32_t e = index[v] + lane; e < index[v + 1]; e += LPV) {
            const uint32_t hd = head[e];
            const bool diag = hd == (uint32_t)v;
            const R w0 = vel[3ull * hd], w1 = vel[3ull * hd + 1], w2 = vel[3ull * hd + 2];
            R Ke[9];
#pragma unroll
            for (int c = 0; c < 9; ++c) Ke[c] = K[(uint64_t)c * ne + e];
            k0 += Ke[0] * w0 + Ke[1] * w1 + Ke[2] * w2;
            k1 += Ke[3] * w0 + Ke[4] * w1 + Ke[5] * w2;
            k2 += Ke[6] * w0 + Ke[7] * w1 + Ke[8] * w2;
            R me = diag ? m : R(0);
            if (CONS) {
                me = mass[e];
                m0 += me * w0;
                m1 += me * w1;
                m2 += me * w2;
                ms += me;
                if (NEWTON) {
                    n0 += me * vel0[3ull * hd];
                    n1 += me * vel0[3ull * hd + 1];
                    n2 += me * vel0[3ull * hd + 2];
                }
            }
#pragma unroll
            for (int c = 0; c < 9; ++c) {
                const R Me = (c == 0 || c == 4 || c == 8) ? me : R(0);
                const R De = alpha * Me + beta * Ke[c];
                A[(uint64_t)c * ne + e] = Me + h * De + h * h * Ke[c];
            }
        }
    }
#pragma unroll
    for (int o = LPV / 2; o > 0; o >>= 1) {
        k0 += __shfl_xor_sync(0xffffffffu, k0, o, LPV);
        k1 += __shfl_xor_sync(0xffffffffu, k1, o, LPV);
        k2 += __shfl_xor_sync(0xffffffffu, k2, o, LPV);
        if (CONS) {
            m0 += __shfl_xor_sync(0xffffffffu, m0, o, LPV);
            m1 += __shfl_xor_sync(0xffffffffu, m1, o, LPV);
            m2 += __shfl_xor_sync(0xffffffffu, m2, o, LPV);
            ms += __shfl_xor_sync(0xffffffffu, ms, o, LPV);
            if (NEWTON) {
                n0 += __shfl_xor_sync(0xffffffffu, n0, o, LPV);
                n1 += __shfl_xor_sync(0xffffffffu, n1, o, LPV);
                n2 += __shfl_xor_sync(0xffffffffu, n2, o, LPV);
            }
        }
    }
    if (live && lane == 0) {
        const R kv[3] = {k0, k1, k2}, mv[3] = {m0, m1, m2}, nv0[3] = {n0, n1, n2}, g[3] = {g0, g1, g2};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const uint64_t i = 3 * v + a;
            const R Mv = CONS ? mv[a] : m * vel[i];
            const R Mg = CONS ? ms * g[a] : m * g[a];
            const R Dv = alpha * Mv + beta * kv[a];
            if (NEWTON) {
                const R Mv0 = CONS ? nv0[a] : m * vel0[i];
                b[i] = h * (f[i] + Mg - Dv) + (Mv0 - Mv);
            } else {
                b[i] = h * (f[i] + Mg - Dv - h * kv[a]);
            }
        }
    }
}

// O8: a = (f + m g)/m; u += v h + a h^2/2; v += a h (Fig. 2 applyForces)
template <typename R>
__global__ void k_explicit(uint64_t nv, const R* __restrict__ f, const R* __restrict__ mass,
                           const uint8_t* __restrict__ mask, R* __restrict__ u, R* __restrict__ vel, R h, R g0, R g1,
                           R g2) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= 3 * nv) return;
    if (mask && !mask[i / 3]) return;
    const R g = (i % 3 == 0) ? g0 : ((i % 3 == 1) ? g1 : g2);
    const R m = mass[i / 3];
    R a = (f[i] + m * g) / m;
    u[i] += vel[i] * h + R(0.5) * a * h * h;
    vel[i] += a * h;
}

// NEWTON = false: vel += dv, u += h vel (the one-linearisation step);
// NEWTON = true:  vel += dv, u += h dv (a later Newton iteration: u = u_n + h vel)
template <typename R, bool NEWTON>
__global__ void k_implicit_update(uint64_t ndof, const R* __restrict__ dv, R h, R* __restrict__ u, R* __restrict__ vel) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= ndof) return;
    const R d = dv[i];
    R v = vel[i] + d;
    vel[i] = v;
    u[i] += h * (NEWTON ? d : v);
}

// generic global reduction over all components of a field
template <typename R, int OP, bool DOT>
__global__ void k_global_reduce(uint64_t n, uint32_t comps, int soa, const R* __restrict__ a, const R* __restrict__ b,
                                const uint8_t* __restrict__ mask, double* __restrict__ partials,
                                unsigned int* __restrict__ counter, double* __restrict__ out) {
    double acc = rop_identity<OP>();
    const uint64_t tot = n * comps;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < tot; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t el = soa ? (i % n) : (i / comps);
        if (mask && !mask[el]) continue;
        double x = (double)a[i];
        if (DOT) x *= (double)b[i];
        acc = rop<OP>(acc, x);
    }
    double r;
    if (block_reduce_last_done<OP>(acc, partials, counter, &r)) *out = r;
}

}  // namespace

// grouped edge relation of a query-loop (declared in ebb_internal.cuh)
namespace ebb {
ebb_status edge_graph(Ctx* c, ebb_rel edges, EdgeGraph* g) {
    Relation* E = get_rel(c, edges);
    if (!E) return fail(c, EBB_E_ARG, "bad edges relation");
    if (E->grouped_by == EBB_NONE || E->index == EBB_NONE)
        return fail(c, EBB_E_STATE, "relation '%s' is not grouped (query-loops need GroupBy, P:696-700)", E->name.c_str());
    Field* key = get_field(c, E->grouped_by);
    ebb_field hf = EBB_NONE;
    for (ebb_field f : E->fields)
        if (c->fields[f].alive && c->fields[f].name == "head") hf = f;
    if (hf == EBB_NONE) return fail(c, EBB_E_STATE, "relation '%s' has no 'head' key-field", E->name.c_str());
    Field* H = &c->fields[hf];
    if (H->dtype != EBB_KEY || H->comps() != 1 || H->key_target != key->key_target)
        return fail(c, EBB_E_TYPE, "'head' must be a scalar key into the grouping source");
    g->verts = key->key_target;
    g->nv = c->rels[g->verts].size;
    g->ne = E->size;
    g->index = (const uint32_t*)c->fields[E->index].ptr;
    g->head = (const uint32_t*)H->ptr;
    g->max_group = E->max_group;
    g->max_chunk16 = E->max_chunk16 ? E->max_chunk16 : TMA_VCH * E->max_group;
    g->max_chunk64 = E->max_chunk64 ? E->max_chunk64 : SPMV_VC * E->max_group;
    return EBB_OK;
}
}  // namespace ebb

namespace {

template <typename R, bool CG, bool MPQ, bool DIR = false>
ebb_status launch_tma(Ctx* c, const EdgeGraph& G, const R* A, const R* p, R* q, const uint8_t* mask, double* pq_out,
                      unsigned int* counter, cudaStream_t s, R* pb0 = nullptr, R* pb1 = nullptr,
                      double* scal = nullptr) {
    const uint32_t cap = tma_cap<R>(G.max_chunk16);
    const size_t stage = ((size_t)9 * cap * sizeof(R) + (size_t)cap * 4 + 127) & ~(size_t)127;
    const size_t smem = stage * TMA_NS;
    if (smem > kTmaSmemMax) return EBB_E_SIZE;   // caller falls back to a path without staging
    // consumer layout: grouped 8 lanes per vertex (default, measured faster:
    // DESIGN.md §5.3); EBB_SPMV_GRP=0 selects 16 lanes per vertex
    static const bool grp = !(getenv("EBB_SPMV_GRP") && getenv("EBB_SPMV_GRP")[0] == '0');
    auto kern = grp ? k_spmv_tma<R, CG, MPQ, DIR, true> : k_spmv_tma<R, CG, MPQ, DIR, false>;
    static thread_local size_t configured_dev[kMaxDevices][2] = {};
    size_t* const configured = configured_dev[c->device % kMaxDevices];
    if (smem > configured[grp]) {
        EBB_CUDA(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured[grp] = smem;
    }
    const int block = 32 * (TMA_CONSUMERS + 1);
    const uint64_t nch = (G.nv + TMA_VCH - 1) / TMA_VCH;
    const unsigned grid = occ_grid(c, kern, block, smem, nch * block);
    kern<<<grid, block, smem, s>>>(G.nv, G.index, G.head, A, G.ne, p, q, mask, c->d_partials, counter, pq_out, cap,
                                   pb0, pb1, scal);
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

template <typename R, bool CG, bool MPQ, bool DIR>
ebb_status launch_spmv_warp(Ctx* c, const EdgeGraph& G, const R* A, const R* p, R* q, const uint8_t* mask,
                            double* pq_out, unsigned int* counter, cudaStream_t s, R* pb0 = nullptr,
                            R* pb1 = nullptr, double* scal = nullptr) {
    const unsigned grid = occ_grid(c, k_spmv_warp<R, CG, MPQ, DIR>, 256, 0, G.nv * 32);
    k_spmv_warp<R, CG, MPQ, DIR><<<grid, 256, 0, s>>>(G.nv, G.index, G.head, A, G.ne, p, q, mask, c->d_partials,
                                                      counter, pq_out, pb0, pb1, scal);
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

// matvec on AOS vec3 p, q (the ebb_map_edge_matvec ABI and the K v of assembly)
template <typename R, bool MPQ>
ebb_status launch_spmv3(Ctx* c, const EdgeGraph& G, const R* A, const R* p, R* q, const uint8_t* mask, double* pq_out,
                        unsigned int* counter, cudaStream_t s, bool padded) {
    KernelTimer kt(c, EBB_K_EDGE_MATVEC, s);
    const char* env = getenv("EBB_SPMV");
    if (padded && !(env && env[0] == 'p')) {
        ebb_status st = launch_tma<R, false, MPQ>(c, G, A, p, q, mask, pq_out, counter, s);
        if (st != EBB_E_SIZE) return st;
    }
    const size_t smem = (size_t)(G.max_chunk64 ? G.max_chunk64 : 1) * 3 * sizeof(R);   // rows of the largest chunk
    if (smem > kTmaSmemMax) return launch_spmv_warp<R, false, MPQ, false>(c, G, A, p, q, mask, pq_out, counter, s);
    if (smem > 48 * 1024)
        EBB_CUDA(c, cudaFuncSetAttribute(k_spmv<R, MPQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const unsigned grid = occ_grid(c, k_spmv<R, MPQ>, 256, smem, ((G.nv + SPMV_VC - 1) / SPMV_VC) * 256);
    k_spmv<R, MPQ><<<grid, 256, smem, s>>>(G.nv, G.index, G.head, A, G.ne, p, q, mask, c->d_partials, counter, pq_out);
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status check_vec(Ctx* c, Field* F, ebb_rel rel, ebb_dtype dt, const char* what) {
    if (!F) return fail(c, EBB_E_ARG, "bad field handle (%s)", what);
    if (F->rel != rel || F->comps() != 3 || F->dtype != dt || F->layout != EBB_AOS)
        return fail(c, EBB_E_TYPE, "'%s' (%s) must be an AOS vec3 field of the map dtype on verts", F->name.c_str(), what);
    return EBB_OK;
}

ebb_status check_mat(Ctx* c, Field* F, ebb_rel rel, ebb_dtype dt, const char* what) {
    if (!F) return fail(c, EBB_E_ARG, "bad field handle (%s)", what);
    if (F->rel != rel || F->comps() != 9 || F->dtype != dt || F->layout != EBB_SOA)
        return fail(c, EBB_E_TYPE, "'%s' (%s) must be a SOA 3x3 field on edges", F->name.c_str(), what);
    return EBB_OK;
}

}  // namespace

namespace ebb {
ebb_status check_mask(Ctx* c, ebb_field m, ebb_rel rel, const uint8_t** out) {
    *out = nullptr;
    if (m == EBB_NONE) return EBB_OK;
    Field* M = get_field(c, m);
    if (!M || M->dtype != EBB_U8 || M->comps() != 1 || M->rel != rel)
        return fail(c, EBB_E_TYPE, "mask must be a U8 scalar field on verts");
    *out = (const uint8_t*)M->ptr;
    return EBB_OK;
}

}  // namespace ebb

namespace {



// upper-triangle CSR of `edges` (cached until the next relation permutation)
ebb_status upper_csr(Ctx* c, ebb_rel edges, const EdgeGraph& G, UpperCSR** out) {
    for (UpperCSR* U : c->uppers)
        if (U->edges == edges) {
            *out = U;
            return EBB_OK;
        }
    const uint64_t nv = G.nv;
    uint32_t *rself = nullptr, *cnt = nullptr, *tmp = nullptr;
    UpperCSR* U = new UpperCSR();
    U->edges = edges;
    U->max_group = G.max_group;
    auto cleanup = [&]() {
        cudaFree(rself);
        cudaFree(cnt);
        cudaFree(tmp);
    };
    if (cudaMalloc(&rself, nv * 4 + 16) != cudaSuccess || cudaMalloc(&cnt, (nv + 1) * 4 + 16) != cudaSuccess ||
        cudaMalloc(&U->uptr, (nv + 1) * 4 + 16) != cudaSuccess) {
        cleanup();
        U->release();
        delete U;
        return fail(c, EBB_E_CUDA, "cg: upper CSR allocation failed");
    }
    cudaMemset(cnt, 0, (nv + 1) * 4);
    k_upper_count<<<grid_for(nv, 256), 256>>>(nv, G.index, G.head, rself, cnt);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, U->uptr, (int)(nv + 1));
    cudaMalloc(&tmp, tb);
    cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, U->uptr, (int)(nv + 1));
    uint32_t nu = 0;
    cudaMemcpy(&nu, U->uptr + nv, 4, cudaMemcpyDeviceToHost);
    U->nu = nu;
    if (cudaMalloc(&U->uhead, (uint64_t)nu * 4 + 64) != cudaSuccess ||
        cudaMalloc(&U->usrc, (uint64_t)nu * 4 + 64) != cudaSuccess) {
        cleanup();
        U->release();
        delete U;
        return fail(c, EBB_E_CUDA, "cg: upper CSR allocation failed");
    }
    k_upper_fill<<<grid_for(nv, 256), 256>>>(nv, G.head, rself, U->uptr, U->uhead, U->usrc);
    const cudaError_t e = cudaDeviceSynchronize();
    cleanup();
    if (e != cudaSuccess) {
        U->release();
        delete U;
        return cuda_fail(c, e, "upper_csr");
    }
    uint32_t st[3];
    if (index_stats(c, U->uptr, nv, st) != EBB_OK) {
        U->release();
        delete U;
        return EBB_E_CUDA;
    }
    U->max_chunk16 = st[1];
    c->uppers.push_back(U);
    *out = U;
    return EBB_OK;
}

// the compressed (upper rows) copy of system matrix `Af`
ebb_status upper_matrix(Ctx* c, UpperCSR* U, ebb_field Af, size_t esize, void** out) {
    for (auto& a : U->ahalf)
        if (a.first == Af) {
            *out = a.second;
            return EBB_OK;
        }
    void* p = nullptr;
    EBB_CUDA(c, cudaMalloc(&p, 9 * U->nu * esize + 256));
    U->ahalf.push_back({Af, p});
    *out = p;
    return EBB_OK;
}

// tolerance mode (ebb_cg.tol > 0): stop once r.z <= tol^2 r0.z0
}  // namespace

namespace ebb {
double cg_tol2(const ebb_cg* cg) { return cg->tol > 0.0 ? cg->tol * cg->tol : 0.0; }

}  // namespace ebb

namespace {

template <typename R>
ebb_status cg_sym_launch(Ctx* c, const ebb_cg* cg, const EdgeGraph& G, int iters, cudaStream_t s) {
    UpperCSR* U;
    EBB_TRY(upper_csr(c, cg->edges, G, &U));
    void* Ah;
    EBB_TRY(upper_matrix(c, U, cg->A, sizeof(R), &Ah));
    const uint8_t* mask;
    EBB_TRY(check_mask(c, cg->mask, G.verts, &mask));
    auto F = [&](ebb_field f) { return (R*)c->fields[f].ptr; };
    const uint32_t cap = tma_cap<R>(U->max_chunk16);
    const size_t stage = ((size_t)9 * cap * sizeof(R) + (size_t)cap * 4 + 127) & ~(size_t)127;
    const size_t smem = stage * TMA_NS;
    if (smem > kTmaSmemMax) return EBB_E_SIZE;   // the caller falls back to Saad
    static thread_local size_t configured_dev[kMaxDevices] = {};
    size_t& configured = configured_dev[c->device % kMaxDevices];
    if (smem > configured) {
        EBB_CUDA(c, cudaFuncSetAttribute(k_cg_sym_persistent<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
        configured = smem;
    }
    const int block = 32 * (TMA_CONSUMERS + 1);
    int nb = 0;
    EBB_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_cg_sym_persistent<R>, block, smem));
    if (nb < 1) return fail(c, EBB_E_CUDA, "cg: persistent kernel does not fit on an SM");
    const uint64_t nch = (G.nv + TMA_VCH - 1) / TMA_VCH;
    uint64_t grid = (uint64_t)nb * c->num_sms;
    if (grid > nch) grid = nch;
    if (grid > 4096) grid = 4096;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    KernelTimer kt(c, EBB_K_CG_SOLVE, s);
    EBB_CUDA(c, cudaLaunchKernelEx(&cfg, k_cg_sym_persistent<R>, G.nv, (const uint32_t*)U->uptr,
                                   (const uint32_t*)U->uhead, (const R*)Ah, (uint64_t)U->nu, F(cg->z), F(cg->p),
                                   F(cg->p2), F(cg->q), (const R*)F(cg->dinv), F(cg->x), F(cg->r), mask,
                                   c->d_partials, c->d_partials + 4096, c->d_counter + 10, c->d_counter + 11,
                                   (double*)c->fields[cg->scal].ptr, (double*)c->fields[cg->rho].ptr, c->d_err, cap,
                                   iters, cg_tol2(cg)));
    return EBB_OK;
}

// symmetric variant, at ebb_cg_init: the upper rows of A and q = 0
template <typename R>
ebb_status cg_sym_prepare(Ctx* c, const ebb_cg* cg, const EdgeGraph& G, cudaStream_t s) {
    UpperCSR* U;
    EBB_TRY(upper_csr(c, cg->edges, G, &U));
    void* Ah;
    EBB_TRY(upper_matrix(c, U, cg->A, sizeof(R), &Ah));
    c->launches++;
    k_compress_upper<R><<<grid_for(U->nu, 256), 256, 0, s>>>(U->nu, G.ne, U->usrc, (const R*)c->fields[cg->A].ptr,
                                                             (R*)Ah);
    EBB_CUDA(c, cudaGetLastError());
    EBB_CUDA(c, cudaMemsetAsync(c->fields[cg->q].ptr, 0, G.nv * 4 * sizeof(R), s));
    return EBB_OK;
}

template <typename R>
ebb_status cg1_launch(Ctx* c, const ebb_cg* cg, const EdgeGraph& G, int iters, cudaStream_t s, int dist = 0) {
    for (ebb_field f : {cg->s, cg->y, cg->w, cg->u, cg->u2})
        if (!get_field(c, f)) return fail(c, EBB_E_STATE, "cg: single-reduction work vectors missing (ebb_cg_init "
                                                           "with this variant first)");
    auto F = [&](ebb_field f) { return (R*)c->fields[f].ptr; };
    const uint8_t* mask;
    EBB_TRY(check_mask(c, cg->mask, G.verts, &mask));
    const uint32_t cap = tma_cap<R>(G.max_chunk16);
    const size_t stage = ((size_t)9 * cap * sizeof(R) + (size_t)cap * 4 + 127) & ~(size_t)127;
    const size_t smem = stage * CG1_NS;
    if (smem > kTmaSmemMax) return EBB_E_SIZE;   // the caller falls back to Saad
    static thread_local size_t configured_dev[kMaxDevices] = {};
    size_t& configured = configured_dev[c->device % kMaxDevices];
    if (smem > configured) {
        EBB_CUDA(c, cudaFuncSetAttribute(cg1_kernel<R>(), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    const int block = 32 * (TMA_CONSUMERS + 1);
    int nb = 0;
    EBB_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, cg1_kernel<R>(), block, smem));
    if (nb < 1) return fail(c, EBB_E_CUDA, "cg: persistent kernel does not fit on an SM");
    const uint64_t nch = (G.nv + TMA_VCH - 1) / TMA_VCH;
    uint64_t grid = (uint64_t)nb * c->num_sms;
    if (grid > nch) grid = nch;
    if (grid > kCg1PartStride) grid = kCg1PartStride;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    KernelTimer kt(c, EBB_K_CG_SOLVE, s);
    EBB_CUDA(c, cudaLaunchKernelEx(&cfg, cg1_kernel<R>(), G.nv, G.index, G.head, (const R*)c->fields[cg->A].ptr,
                                   G.ne, (const R*)c->fields[cg->dinv].ptr, F(cg->x), F(cg->r), (const R*)F(cg->z),
                                   F(cg->p), F(cg->s), F(cg->y), F(cg->w), F(cg->u), F(cg->u2), mask, c->d_partials,
                                   c->d_partials + 4096, c->d_counter + 10, c->d_counter + 11,
                                   (double*)c->fields[cg->scal].ptr, (double*)c->fields[cg->rho].ptr, c->d_err, cap,
                                   iters, cg_tol2(cg), dist));
    return EBB_OK;
}

template <typename R>
ebb_status cg_iterate(Ctx* c, const ebb_cg* cg, const EdgeGraph& G, int iters, cudaStream_t s, int only_phase = -1) {
    const R* A = (const R*)c->fields[cg->A].ptr;
    R* x = (R*)c->fields[cg->x].ptr;
    R* r = (R*)c->fields[cg->r].ptr;
    R* p = (R*)c->fields[cg->p].ptr;
    R* p2 = (R*)c->fields[cg->p2].ptr;
    R* z = (R*)c->fields[cg->z].ptr;
    R* q = (R*)c->fields[cg->q].ptr;
    const R* dinv = (const R*)c->fields[cg->dinv].ptr;
    const uint8_t* mask;
    EBB_TRY(check_mask(c, cg->mask, G.verts, &mask));
    double* scal = (double*)c->fields[cg->scal].ptr;
    double* rho_user = (double*)c->fields[cg->rho].ptr;
    const unsigned ug = occ_grid(c, k_cg_update<R>, 256, 0, G.nv);
    const int variant = cg_variant(cg, G, sizeof(R) == 8 ? EBB_F64 : EBB_F32);
    if (only_phase < 0 && iters > 0 && variant == EBB_CG_SINGLE_REDUCTION) return cg1_launch<R>(c, cg, G, iters, s);
    if (only_phase == EBB_CG_SR_PHASE) {
        const ebb_status st = cg1_launch<R>(c, cg, G, 1, s, 1);
        if (st == EBB_E_SIZE)
            return fail(c, EBB_E_RANGE, "cg: single-reduction phase: the largest 16-vertex chunk (%u rows) does not "
                                        "fit the TMA stages (use the Saad phases)", G.max_chunk16);
        return st;
    }
    if (only_phase < 0 && iters > 0 && variant == EBB_CG_SYMMETRIC) return cg_sym_launch<R>(c, cg, G, iters, s);
    const char* mode = getenv("EBB_CG");
    if (only_phase < 0 && iters > 0 && !(mode && mode[0] == '2')) {
        // single launch, all iterations (cooperative: every CTA resident)
        const uint32_t cap = tma_cap<R>(G.max_chunk16);
        const size_t stage = ((size_t)9 * cap * sizeof(R) + (size_t)cap * 4 + 127) & ~(size_t)127;
        const size_t smem = stage * TMA_NS;
        if (smem <= kTmaSmemMax) {
            static thread_local size_t configured_dev[kMaxDevices] = {};
            size_t& configured = configured_dev[c->device % kMaxDevices];
            if (smem > configured) {
                EBB_CUDA(c, cudaFuncSetAttribute(k_cg_persistent<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem));
                configured = smem;
            }
            const int block = 32 * (TMA_CONSUMERS + 1);
            int nb = 0;
            EBB_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_cg_persistent<R>, block, smem));
            if (nb >= 1) {
                const uint64_t nch = (G.nv + TMA_VCH - 1) / TMA_VCH;
                uint64_t grid = (uint64_t)nb * c->num_sms;
                if (grid > nch) grid = nch;
                if (grid > 4096) grid = 4096;
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3((unsigned)grid);
                cfg.blockDim = dim3(block);
                cfg.dynamicSmemBytes = smem;
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeCooperative;
                at[0].val.cooperative = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                KernelTimer kt(c, EBB_K_CG_SOLVE, s);
                EBB_CUDA(c, cudaLaunchKernelEx(&cfg, k_cg_persistent<R>, G.nv, G.index, G.head, A, G.ne, z, p, p2, q,
                                               dinv, x, r, mask, c->d_partials, c->d_partials + 4096,
                                               c->d_counter + 10, c->d_counter + 11, scal, rho_user, c->d_err, cap,
                                               iters, cg_tol2(cg)));
#ifdef CG_PROF
                {
                    unsigned long long h[8];
                    cudaDeviceSynchronize();
                    cudaMemcpyFromSymbol(h, g_cg_prof, sizeof(h));
                    const unsigned long long zr[8] = {0};
                    cudaMemcpyToSymbol(g_cg_prof, zr, sizeof(zr));
                    const double n = (double)h[6];   // CTA-iterations
                    fprintf(stderr, "CG_PROF grid %llu: per iteration (cycles, thread 0 of a CTA): matvec own %.0f, "
                            "CTA wait %.0f, barrier1 %.0f, update %.0f, barrier2 %.0f\n", h[5], h[0] / n, h[1] / n,
                            h[2] / n, h[3] / n, h[4] / n);
                }
#endif
                return EBB_OK;
            }
        }
    }
    for (int k = 0; k < iters; ++k) {
        // EBB_CG_DIR is fused into the matvec (p = z + beta p_old gathered on the fly)
        if (only_phase < 0 || only_phase == EBB_CG_MATVEC) {
            KernelTimer kt(c, EBB_K_EDGE_MATVEC, s);
            ebb_status st = launch_tma<R, true, true, true>(c, G, A, z, q, mask, scal + S_PQ, c->d_counter + 1, s, p,
                                                            p2, scal);
            if (st == EBB_E_SIZE)   // the largest chunk does not fit the stages: no staging
                st = launch_spmv_warp<R, true, true, true>(c, G, A, z, q, mask, scal + S_PQ, c->d_counter + 1, s, p,
                                                           p2, scal);
            EBB_TRY(st);
        }
        if (only_phase < 0 || only_phase == EBB_CG_UPDATE) {
            KernelTimer kt(c, EBB_K_CG_UPDATE, s);
            k_cg_update<R><<<ug, 256, 0, s>>>(G.nv, p, p2, q, dinv, x, r, z, c->d_partials, c->d_counter + 2, scal,
                                              rho_user, c->d_err, only_phase < 0 ? cg_tol2(cg) : 0.0);
        }
    }
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

// AUTO = the measured faster variant: the single-reduction
// kernel saves a grid barrier and a gathered vector per iteration but moves
// ~9 owner-local vector records per vertex; it wins while they stay in L2
// (C2: 1M tets, fp64) and loses once they stream from HBM (1e7 tets).
}  // namespace

namespace ebb {
int cg_variant(const ebb_cg* cg, const EdgeGraph& G, ebb_dtype dt) {
    int v = cg->variant;
    if (v == EBB_CG_AUTO) {
        const char* e = getenv("EBB_CG_VARIANT");
        if (e && atoi(e) >= EBB_CG_SAAD && atoi(e) <= EBB_CG_SYMMETRIC) v = atoi(e);
        // measured crossover (fp64 and fp32 alike): between 1.8e5 and 3.0e5 vertices
        else v = G.nv <= 232000 ? EBB_CG_SINGLE_REDUCTION : EBB_CG_SAAD;
    }
    // a variant whose ring of TMA stages (sized by the largest 16-vertex chunk)
    // does not fit runs as Saad, which has a path without staging
    if (v == EBB_CG_SINGLE_REDUCTION || v == EBB_CG_SYMMETRIC) {
        const size_t bf = dt == EBB_F64 ? 8 : 4;
        const size_t cap = ((G.max_chunk16 ? G.max_chunk16 : 1) + 2 * (16 / bf) + 4 + 3) & ~(size_t)3;
        const size_t stage = (9 * cap * bf + cap * 4 + 127) & ~(size_t)127;
        if (stage * (v == EBB_CG_SINGLE_REDUCTION ? CG1_NS : TMA_NS) > kTmaSmemMax) v = EBB_CG_SAAD;
    }
    return v;
}

}  // namespace ebb

namespace {

}  // namespace

namespace ebb {
ebb_status cg_validate(Ctx* c, const ebb_cg* cg, EdgeGraph* G, ebb_dtype* dt) {
    EBB_TRY(edge_graph(c, cg->edges, G));
    Field* A = get_field(c, cg->A);
    if (!A) return fail(c, EBB_E_ARG, "cg: bad A");
    *dt = A->dtype;
    EBB_TRY(check_mat(c, A, cg->edges, *dt, "A"));
    if (!A->owned) return fail(c, EBB_E_TYPE, "cg: A must be a library-allocated field (padded for bulk copies)");
    EBB_TRY(check_vec(c, get_field(c, cg->b), G->verts, *dt, "b"));
    EBB_TRY(check_vec(c, get_field(c, cg->x), G->verts, *dt, "x"));
    return EBB_OK;
}

}  // namespace ebb

namespace {


}  // namespace


extern "C" {

ebb_status ebb_map_edge_matvec(ebb_ctx ctx, ebb_rel edges, ebb_field A, ebb_field p, ebb_field q, ebb_field mask,
                               ebb_field pq_global, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c) return EBB_E_ARG;
    EdgeGraph G;
    EBB_TRY(edge_graph(c, edges, &G));
    Field* Af = get_field(c, A);
    if (!Af) return fail(c, EBB_E_ARG, "matvec: bad A");
    ebb_dtype dt = Af->dtype;
    EBB_TRY(check_mat(c, Af, edges, dt, "A"));
    Field* P = get_field(c, p);
    Field* Q = get_field(c, q);
    EBB_TRY(check_vec(c, P, G.verts, dt, "p"));
    EBB_TRY(check_vec(c, Q, G.verts, dt, "q"));
    if (P->ptr == Q->ptr) return fail(c, EBB_E_PHASE, "matvec: p and q alias (read and write phase)");
    const uint8_t* m;
    EBB_TRY(check_mask(c, mask, G.verts, &m));
    double* pq = nullptr;
    if (pq_global != EBB_NONE) {
        Field* PQ = get_field(c, pq_global);
        if (!PQ || !PQ->is_global || PQ->dtype != EBB_F64) return fail(c, EBB_E_TYPE, "pq_global must be an F64 global");
        pq = (double*)PQ->ptr;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const bool fused = pq || m;
    double* pqo = pq ? pq : (double*)c->d_partials + 8191;
    if (dt == EBB_F64) {
        if (fused)
            return launch_spmv3<double, true>(c, G, (const double*)Af->ptr, (const double*)P->ptr, (double*)Q->ptr, m,
                                              pqo, c->d_counter + 3, s, Af->owned);
        return launch_spmv3<double, false>(c, G, (const double*)Af->ptr, (const double*)P->ptr, (double*)Q->ptr,
                                           nullptr, nullptr, c->d_counter + 3, s, Af->owned);
    }
    if (dt == EBB_F32) {
        if (fused)
            return launch_spmv3<float, true>(c, G, (const float*)Af->ptr, (const float*)P->ptr, (float*)Q->ptr, m,
                                             pqo, c->d_counter + 3, s, Af->owned);
        return launch_spmv3<float, false>(c, G, (const float*)Af->ptr, (const float*)P->ptr, (float*)Q->ptr, nullptr,
                                          nullptr, c->d_counter + 3, s, Af->owned);
    }
    return fail(c, EBB_E_TYPE, "matvec: dtype must be F32 or F64");
}

ebb_status ebb_global_reduce(ebb_ctx ctx, int32_t op, ebb_field a, ebb_field b, ebb_field mask, ebb_field out,
                             ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c) return EBB_E_ARG;
    Field* Af = get_field(c, a);
    Field* O = get_field(c, out);
    if (!Af || !O) return fail(c, EBB_E_ARG, "global_reduce: bad handle");
    if (!O->is_global || O->dtype != EBB_F64) return fail(c, EBB_E_TYPE, "global_reduce: out must be an F64 global");
    if (Af->dtype != EBB_F32 && Af->dtype != EBB_F64) return fail(c, EBB_E_TYPE, "global_reduce: F32/F64 fields only");
    Field* Bf = nullptr;
    if (op == EBB_RED_DOT) {
        Bf = get_field(c, b);
        if (!Bf || Bf->dtype != Af->dtype || Bf->comps() != Af->comps() || Bf->rel != Af->rel || Bf->layout != Af->layout)
            return fail(c, EBB_E_TYPE, "global_reduce DOT: b must match a");
    } else if (op != EBB_RED_SUM && op != EBB_RED_MAX && op != EBB_RED_MIN) {
        return fail(c, EBB_E_ARG, "global_reduce: unknown op %d", op);
    }
    const uint8_t* m;
    EBB_TRY(check_mask(c, mask, Af->rel, &m));
    uint64_t n = c->rels[Af->rel].size;
    unsigned grid = occ_grid(c, k_global_reduce<double, ROP_SUM, true>, 256, 0, n * Af->comps());
    cudaStream_t s = (cudaStream_t)stream;
    int soa = Af->layout == EBB_SOA;
    double* o = (double*)O->ptr;
    unsigned int* cnt = c->d_counter + 4;
    c->launches++;
#define EBB_RED(R)                                                                                                    \
    do {                                                                                                              \
        const R* pa = (const R*)Af->ptr;                                                                              \
        const R* pb = Bf ? (const R*)Bf->ptr : nullptr;                                                               \
        if (op == EBB_RED_SUM) k_global_reduce<R, ROP_SUM, false><<<grid, 256, 0, s>>>(n, Af->comps(), soa, pa, pb, m, c->d_partials, cnt, o); \
        else if (op == EBB_RED_DOT) k_global_reduce<R, ROP_SUM, true><<<grid, 256, 0, s>>>(n, Af->comps(), soa, pa, pb, m, c->d_partials, cnt, o); \
        else if (op == EBB_RED_MAX) k_global_reduce<R, ROP_MAX, false><<<grid, 256, 0, s>>>(n, Af->comps(), soa, pa, pb, m, c->d_partials, cnt, o); \
        else k_global_reduce<R, ROP_MIN, false><<<grid, 256, 0, s>>>(n, Af->comps(), soa, pa, pb, m, c->d_partials, cnt, o); \
    } while (0)
    if (Af->dtype == EBB_F64) EBB_RED(double);
    else EBB_RED(float);
#undef EBB_RED
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status ebb_implicit_assemble(ebb_ctx ctx, const ebb_implicit_desc* d, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !d) return fail(c, EBB_E_ARG, "null argument");
    EdgeGraph G;
    EBB_TRY(edge_graph(c, d->edges, &G));
    Field* K = get_field(c, d->K);
    Field* A = get_field(c, d->A);
    if (!K || !A) return fail(c, EBB_E_ARG, "assemble: bad K/A");
    ebb_dtype dt = K->dtype;
    EBB_TRY(check_mat(c, K, d->edges, dt, "K"));
    EBB_TRY(check_mat(c, A, d->edges, dt, "A"));
    Field* M = get_field(c, d->mass);
    if (!M || M->dtype != dt || M->comps() != 1 || (M->rel != G.verts && M->rel != d->edges))
        return fail(c, EBB_E_TYPE, "assemble: mass must be a scalar field of the map dtype on verts (lumped) or "
                                   "on the edges (consistent)");
    const bool cons = M->rel == d->edges;
    Field* F = get_field(c, d->f);
    Field* V = get_field(c, d->vel);
    Field* B = get_field(c, d->b);
    EBB_TRY(check_vec(c, F, G.verts, dt, "f"));
    EBB_TRY(check_vec(c, V, G.verts, dt, "vel"));
    EBB_TRY(check_vec(c, B, G.verts, dt, "b"));
    if (B->ptr == F->ptr || B->ptr == V->ptr) return fail(c, EBB_E_PHASE, "assemble: b aliases a read field");
    if (d->rhs_form != EBB_RHS_LINEARISED && d->rhs_form != EBB_RHS_NEWTON)
        return fail(c, EBB_E_ARG, "assemble: unknown rhs_form %d", d->rhs_form);
    const bool newton = d->rhs_form == EBB_RHS_NEWTON;
    Field* V0 = nullptr;
    if (newton) {
        V0 = get_field(c, d->vel0);
        EBB_TRY(check_vec(c, V0, G.verts, dt, "vel0"));
        if (B->ptr == V0->ptr) return fail(c, EBB_E_PHASE, "assemble: b aliases vel0");
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int lpv = G.max_group <= 16 ? 16 : 32;
#define EBB_ASM(R)                                                                                                  \
    do {                                                                                                            \
        KernelTimer kt(c, EBB_K_ASSEMBLE, s);                                                                       \
        decltype(&k_assemble_fused<R, 16, false, false>) kern;                                                     \
        if (newton)                                                                                                 \
            kern = lpv == 16 ? (cons ? k_assemble_fused<R, 16, true, true> : k_assemble_fused<R, 16, false, true>)   \
                             : (cons ? k_assemble_fused<R, 32, true, true> : k_assemble_fused<R, 32, false, true>);  \
        else                                                                                                        \
            kern = lpv == 16 ? (cons ? k_assemble_fused<R, 16, true, false> : k_assemble_fused<R, 16, false, false>) \
                             : (cons ? k_assemble_fused<R, 32, true, false> : k_assemble_fused<R, 32, false, false>);\
        kern<<<grid_for(G.nv * lpv, 256), 256, 0, s>>>(G.nv, G.index, G.head, (const R*)K->ptr, (R*)A->ptr, G.ne,    \
                                                       (const R*)M->ptr, (const R*)F->ptr, (const R*)V->ptr,        \
                                                       V0 ? (const R*)V0->ptr : nullptr, (R*)B->ptr, (R)d->h,       \
                                                       (R)d->alpha, (R)d->beta, (R)d->g[0], (R)d->g[1], (R)d->g[2]);\
    } while (0)
    if (dt == EBB_F64) EBB_ASM(double);
    else EBB_ASM(float);
#undef EBB_ASM
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status ebb_cg_init(ebb_ctx ctx, ebb_cg* cg, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !cg) return fail(c, EBB_E_ARG, "null argument");
    EdgeGraph G;
    ebb_dtype dt;
    EBB_TRY(cg_validate(c, cg, &G, &dt));
    Field* S = get_field(c, cg->self);
    if (!S || S->dtype != EBB_KEY || S->rel != G.verts || S->key_target != cg->edges)
        return fail(c, EBB_E_TYPE, "cg: self must be the verts -> edges self-loop key");
    const uint8_t* mask;
    EBB_TRY(check_mask(c, cg->mask, G.verts, &mask));
    // work vectors: padded 4-component records, allocated on first use
    static int serial = 0;
    char nm[64];
    if (cg->variant < EBB_CG_AUTO || cg->variant > EBB_CG_SYMMETRIC)
        return fail(c, EBB_E_ARG, "cg: unknown variant %d", cg->variant);
    ebb_field* work[] = {&cg->r, &cg->p, &cg->z, &cg->q, &cg->dinv, &cg->p2, &cg->s, &cg->y, &cg->w, &cg->u, &cg->u2};
    const char* wn[] = {"r", "p", "z", "q", "dinv", "p2", "s", "y", "w", "u", "u2"};
    const int nwork = cg_variant(cg, G, dt) == EBB_CG_SINGLE_REDUCTION ? 11 : 6;
    int id = -1;
    for (int i = 0; i < nwork; ++i) {
        Field* W = *work[i] == EBB_NONE ? nullptr : get_field(c, *work[i]);
        if (!W) {
            if (id < 0) id = serial++;
            snprintf(nm, sizeof(nm), "__cg%d_%s", id, wn[i]);
            EBB_TRY(new_internal_field(c, G.verts, nm, dt, 4, 1, EBB_AOS, work[i]));
        } else if (W->rel != G.verts || W->comps() != 4 || W->dtype != dt || W->layout != EBB_AOS) {
            return fail(c, EBB_E_TYPE, "cg: work field '%s' must be an AOS 4x1 (padded vec3) field on verts",
                        W->name.c_str());
        }
    }
    if (cg->rho == EBB_NONE) {
        if (id < 0) id = serial++;
        snprintf(nm, sizeof(nm), "__cg%d_rho", id);
        EBB_TRY(ebb_global_new(ctx, nm, EBB_F64, 0.0, &cg->rho));
    }
    if (cg->scal == EBB_NONE) {
        if (id < 0) id = serial++;
        snprintf(nm, sizeof(nm), "__cg%d_scal", id);
        ebb_rel sr;
        EBB_TRY(ebb_relation_new(ctx, (std::string(nm) + "_rel").c_str(), S_NSCAL, &sr));
        EBB_TRY(new_internal_field(c, sr, nm, EBB_F64, 1, 1, EBB_AOS, &cg->scal));
    }
    cudaStream_t s = (cudaStream_t)stream;
    double* scal = (double*)c->fields[cg->scal].ptr;
    double* rho = (double*)c->fields[cg->rho].ptr;
    const uint32_t* self = (const uint32_t*)c->fields[cg->self].ptr;
    c->launches++;
#define EBB_INIT(R)                                                                                                  \
    do {                                                                                                             \
        const unsigned g = occ_grid(c, k_cg_init<R>, 256, 0, G.nv);                                                  \
        k_cg_init<R><<<g, 256, 0, s>>>(G.nv, self, (const R*)c->fields[cg->A].ptr, G.ne,                             \
                                       (const R*)c->fields[cg->b].ptr, mask, (R*)c->fields[cg->dinv].ptr,            \
                                       (R*)c->fields[cg->x].ptr, (R*)c->fields[cg->r].ptr, (R*)c->fields[cg->z].ptr, \
                                       (R*)c->fields[cg->p].ptr, c->d_partials, c->d_counter + 6, scal, rho);        \
    } while (0)
    if (dt == EBB_F64) EBB_INIT(double);
    else EBB_INIT(float);
#undef EBB_INIT
    EBB_CUDA(c, cudaGetLastError());
    if (cg_variant(cg, G, dt) == EBB_CG_SYMMETRIC) {
        if (dt == EBB_F64) return cg_sym_prepare<double>(c, cg, G, s);
        return cg_sym_prepare<float>(c, cg, G, s);
    }
    return EBB_OK;
}

ebb_status ebb_cg_iterations(ebb_ctx ctx, const ebb_cg* cg, ebb_stream stream, int32_t* iters, int32_t* converged) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !cg) return fail(c, EBB_E_ARG, "null argument");
    Field* S = get_field(c, cg->scal);
    if (!S) return fail(c, EBB_E_STATE, "cg: call ebb_cg_init first");
    if (S->dtype != EBB_F64 || c->rels[S->rel].size < S_NSCAL) return fail(c, EBB_E_TYPE, "cg: bad scal field");
    double v[S_NSCAL];
    EBB_CUDA(c, cudaMemcpyAsync(v, S->ptr, sizeof(v), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    EBB_CUDA(c, cudaStreamSynchronize((cudaStream_t)stream));
    if (iters) *iters = (int32_t)v[S_ITERS];
    if (converged) *converged = v[S_DONE] != 0.0 ? 1 : 0;
    return EBB_OK;
}

ebb_status ebb_cg_variant(ebb_ctx ctx, const ebb_cg* cg, int32_t* out) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !cg || !out) return fail(c, EBB_E_ARG, "null argument");
    EdgeGraph G;
    ebb_dtype dt;
    EBB_TRY(cg_validate(c, cg, &G, &dt));
    *out = cg_variant(cg, G, dt);
    return EBB_OK;
}

ebb_status ebb_cg_step(ebb_ctx ctx, const ebb_cg* cg, int32_t iters, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !cg) return fail(c, EBB_E_ARG, "null argument");
    if (iters < 0) return fail(c, EBB_E_ARG, "negative iteration count");
    EdgeGraph G;
    ebb_dtype dt;
    EBB_TRY(cg_validate(c, cg, &G, &dt));
    ebb_field w[] = {cg->r, cg->p, cg->z, cg->q, cg->dinv, cg->rho, cg->scal, cg->p2};
    for (ebb_field f : w)
        if (!get_field(c, f)) return fail(c, EBB_E_STATE, "cg: call ebb_cg_init first");
    if (c->rels[get_field(c, cg->scal)->rel].size < S_NSCAL)
        return fail(c, EBB_E_TYPE, "cg: scal must hold %d F64 values", (int)S_NSCAL);
    if (!(cg->tol >= 0.0)) return fail(c, EBB_E_ARG, "cg: tol must be >= 0");
    cudaStream_t s = (cudaStream_t)stream;
    if (dt == EBB_F64) return cg_iterate<double>(c, cg, G, iters, s);
    return cg_iterate<float>(c, cg, G, iters, s);
}

ebb_status ebb_cg_phase(ebb_ctx ctx, const ebb_cg* cg, int32_t phase, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !cg) return fail(c, EBB_E_ARG, "null argument");
    if (phase < EBB_CG_DIR || phase > EBB_CG_SR_PHASE) return fail(c, EBB_E_ARG, "unknown CG phase %d", phase);
    EdgeGraph G;
    ebb_dtype dt;
    EBB_TRY(cg_validate(c, cg, &G, &dt));
    ebb_field w[] = {cg->r, cg->p, cg->z, cg->q, cg->dinv, cg->rho, cg->scal, cg->p2};
    for (ebb_field f : w)
        if (!get_field(c, f)) return fail(c, EBB_E_STATE, "cg: call ebb_cg_init first");
    cudaStream_t s = (cudaStream_t)stream;
    if (dt == EBB_F64) return cg_iterate<double>(c, cg, G, 1, s, phase);
    return cg_iterate<float>(c, cg, G, 1, s, phase);
}

ebb_status ebb_explicit_update(ebb_ctx ctx, const ebb_explicit_desc* d, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !d) return fail(c, EBB_E_ARG, "null argument");
    Field* U = get_field(c, d->u);
    if (!U) return fail(c, EBB_E_ARG, "explicit: bad u");
    ebb_rel verts = U->rel;
    ebb_dtype dt = U->dtype;
    EBB_TRY(check_vec(c, U, verts, dt, "u"));
    EBB_TRY(check_vec(c, get_field(c, d->vel), verts, dt, "vel"));
    EBB_TRY(check_vec(c, get_field(c, d->f), verts, dt, "f"));
    Field* M = get_field(c, d->mass);
    if (!M || M->dtype != dt || M->comps() != 1 || M->rel != verts) return fail(c, EBB_E_TYPE, "explicit: bad mass");
    const uint8_t* mask;
    EBB_TRY(check_mask(c, d->mask, verts, &mask));
    uint64_t nv = c->rels[verts].size;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned g = grid_for(3 * nv, 256);
    c->launches++;
    if (dt == EBB_F64)
        k_explicit<double><<<g, 256, 0, s>>>(nv, (const double*)c->fields[d->f].ptr, (const double*)M->ptr, mask,
                                             (double*)U->ptr, (double*)c->fields[d->vel].ptr, d->h, d->g[0], d->g[1], d->g[2]);
    else
        k_explicit<float><<<g, 256, 0, s>>>(nv, (const float*)c->fields[d->f].ptr, (const float*)M->ptr, mask,
                                            (float*)U->ptr, (float*)c->fields[d->vel].ptr, (float)d->h, (float)d->g[0],
                                            (float)d->g[1], (float)d->g[2]);
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

namespace {
ebb_status implicit_update_impl(ebb_ctx ctx, ebb_field dv, double h, ebb_field u, ebb_field vel, ebb_stream stream,
                                bool newton) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c) return EBB_E_ARG;
    Field* U = get_field(c, u);
    if (!U) return fail(c, EBB_E_ARG, "implicit_update: bad u");
    ebb_dtype dt = U->dtype;
    EBB_TRY(check_vec(c, U, U->rel, dt, "u"));
    EBB_TRY(check_vec(c, get_field(c, vel), U->rel, dt, "vel"));
    EBB_TRY(check_vec(c, get_field(c, dv), U->rel, dt, "dv"));
    uint64_t ndof = 3 * c->rels[U->rel].size;
    cudaStream_t s = (cudaStream_t)stream;
    c->launches++;
    if (dt == EBB_F64) {
        auto k = newton ? k_implicit_update<double, true> : k_implicit_update<double, false>;
        k<<<grid_for(ndof, 256), 256, 0, s>>>(ndof, (const double*)c->fields[dv].ptr, h, (double*)U->ptr,
                                              (double*)c->fields[vel].ptr);
    } else {
        auto k = newton ? k_implicit_update<float, true> : k_implicit_update<float, false>;
        k<<<grid_for(ndof, 256), 256, 0, s>>>(ndof, (const float*)c->fields[dv].ptr, (float)h, (float*)U->ptr,
                                              (float*)c->fields[vel].ptr);
    }
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}
}  // namespace

ebb_status ebb_implicit_update(ebb_ctx ctx, ebb_field dv, double h, ebb_field u, ebb_field vel, ebb_stream stream) {
    return implicit_update_impl(ctx, dv, h, u, vel, stream, false);
}

ebb_status ebb_newton_update(ebb_ctx ctx, ebb_field dv, double h, ebb_field u, ebb_field vel, ebb_stream stream) {
    return implicit_update_impl(ctx, dv, h, u, vel, stream, true);
}

}  // extern "C"
