// peer_cg.cu -- the fused multi-GPU PCG over peer memory and the peer halos
// (the halo exchange of positions and of the partial force
// sums and the allreduce of the CG scalars, without NCCL on the path; the
// paper is single-device).  Kernels: cg1_peer_body (single-
// reduction) and cg_saad_peer_body (Saad) as k_cg_peer1 (one rank per
// launch, the record a kernel parameter) / k_cg_peer (ranks emulated on one
// device in one cooperative launch), k_peer_halo (COPY / ADD halos); the
// C-ABI bind / step / push entry points.  The send lists and CUDA IPC of
// fields are in peer.cu; include/ebb.h documents the protocol.
#include <cstring>
#include <type_traits>
#include <vector>

#include "async_copy.cuh"
#include "cg_common.cuh"
#include "ebb_internal.cuh"
#include "reduce.cuh"

using namespace ebb;

namespace {

// ---------------------------------------------------------------------------
// Fused multi-GPU single-reduction PCG over peer memory (ebb_cg_peer_step;
// SURVEY §8(e); include/ebb.h).  One launch runs every iteration of every
// rank whose system lives on this device: a real multi-GPU job launches it
// once per process (one rank), ranks emulated on one device share one
// cooperative launch, CTAs [lr*G, (lr+1)*G) working for local rank lr.  The
// per-phase work is k_cg1_persistent's on the rank's OWNED rows (ghost rows
// are never solved), plus:
//   * the owner of a row that peers hold as a ghost stores its new u (the
//     next gathered operand) and x straight into the peers' buffers as it
//     finishes the row (send CSR: per owned vertex, (peer, peer row));
//   * the phase's rank-local (w.z, r.z) go through mailboxes: after the
//     rank's grid barrier (every CTA fenced at system scope, so its peer
//     stores are visible first), block 0 writes them into every peer's
//     mailbox slot [epoch & 1][rank] and releases the slot's sequence word
//     (epoch + 1); every CTA of every rank acquires the P-1 sequence words of
//     its own mailbox and sums the P values in rank order -- the same sums,
//     bitwise, on every rank, so alpha, beta and the tolerance stop agree.
// Safety of the buffers without further barriers: a rank writes a peer's
// ghost rows of u(par') only in the phase after the one in which that peer
// last gathered u(par'), and it can be there only after the peer published
// that phase's sums, i.e. after every CTA of the peer finished the phase; a
// mailbox slot is rewritten two exchanges later, which needs this rank's
// next publication, made after all its CTAs read the slot.  The first
// launch after ebb_cg_init exchanges r.z once (everyone has initialised,
// so nobody's ebb_cg_init can zero a ghost row after a peer filled it),
// then pushes z_0 and exchanges again before the w_0 = A z_0 prologue.
constexpr int kPeerMax = EBB_MAX_RANKS;
constexpr int kMbEpoch = 2 * kPeerMax * 4;   // mailbox word holding the rank's exchange count
static_assert(kMbEpoch < EBB_PEER_MBOX_WORDS, "mailbox layout");
struct PeerRankArgs {
    uint64_t nv, ne;                   // owned rows (solved), edge rows of the local relation
    const uint32_t* index;
    const uint32_t* head;
    const void* A;
    const void* dinv;
    void *x, *r, *z0, *p, *sv, *yv, *wv, *ub0, *ub1;
    void *q, *p2;                      // Saad: q = A p, the second direction buffer
    uint64_t nv_all;                   // local rows (owned + ghost)
    const uint8_t* mask;
    double* part;                      // 4 x kCg1PartStride: (g, d) x phase parity
    unsigned int* bar;                 // rank grid barrier: count, generation
    double* scal;
    double* rho_user;
    const uint32_t* send_off;
    const uint2* send_dst;
    unsigned long long* mbox;          // own mailbox
    void* peer_ub0[kPeerMax];
    void* peer_ub1[kPeerMax];
    void* peer_x[kPeerMax];
    void* peer_z0[kPeerMax];
    unsigned long long* peer_mbox[kPeerMax];
    int rank, nranks;
    uint32_t cap, pad;
};

__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// grid barrier over the G CTAs of one rank; a CTA that stored to peer memory
// since its last barrier fences at system scope before it arrives (those
// stores precede the rank's publication), the others at GPU scope (nothing
// of theirs is read by a peer)
__device__ __forceinline__ void rank_barrier(unsigned int* bar, unsigned int nblocks, bool sent) {
    const int any = __syncthreads_or(sent ? 1 : 0);
    if (threadIdx.x == 0) {
        unsigned int* count = bar;
        unsigned int* gen = bar + 1;
        const unsigned int g = *reinterpret_cast<volatile unsigned int*>(gen);
        if (any) asm volatile("fence.acq_rel.sys;" ::: "memory");
        else __threadfence();
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

#ifndef EBB_PEER_TIMEOUT_NS
#define EBB_PEER_TIMEOUT_NS 20000000000ull   // 20 s: a peer that never arrives
#endif
// exchange number `epoch` of (d, g) between the ranks; returns the sums over
// ranks in rank order (every CTA, every rank: the same values).  Call after a
// rank_barrier that follows this CTA's last read of the previous exchange.
template <typename ARGS>   // PeerRankArgs or HaloRankArgs: rank, nranks, mbox, peer_mbox
__device__ __forceinline__ void peer_exchange(const ARGS& a, unsigned bid, uint64_t epoch, double d, double g,
                                              double* sm2, unsigned long long* err, double& dsum, double& gsum) {
    const unsigned slot = (unsigned)(epoch & 1u);
    const unsigned long long seq = epoch + 1;
    const unsigned q = threadIdx.x;
    if (bid == 0 && q < (unsigned)a.nranks && q != (unsigned)a.rank) {
        unsigned long long* mb = a.peer_mbox[q] + (slot * kPeerMax + a.rank) * 4;
        st_relaxed_sys(mb, (unsigned long long)__double_as_longlong(d));
        st_relaxed_sys(mb + 1, (unsigned long long)__double_as_longlong(g));
        st_release_sys(mb + 2, seq);
    }
    if (q < (unsigned)a.nranks && q != (unsigned)a.rank) {
        const unsigned long long* sw = a.mbox + (slot * kPeerMax + q) * 4 + 2;
        // after one abandoned wait every later one is skipped (the results are
        // invalid anyway; the launch must still end)
        if (ld_acquire_sys(sw) != seq && *reinterpret_cast<volatile unsigned long long*>(&err[ERR_PEER]) == 0) {
            const unsigned long long t0 = global_ns();
            while (ld_acquire_sys(sw) != seq) {
                __nanosleep(32);
                if (global_ns() - t0 > EBB_PEER_TIMEOUT_NS) {
                    atomicAdd(&err[ERR_PEER], 1ull);
                    break;
                }
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double sd = 0.0, sg = 0.0;
        for (int r = 0; r < a.nranks; ++r) {
            if (r == a.rank) {
                sd += d;
                sg += g;
            } else {
                const unsigned long long* mb = a.mbox + (slot * kPeerMax + r) * 4;
                sd += __longlong_as_double((long long)ld_relaxed_sys(mb));
                sg += __longlong_as_double((long long)ld_relaxed_sys(mb + 1));
            }
        }
        sm2[0] = sd;
        sm2[1] = sg;
    }
    __syncthreads();
    dsum = sm2[0];
    gsum = sm2[1];
}

// The body of one rank's CTA (lr: local rank of the launch, bid: CTA within
// the rank, G CTAs per rank); `a` is a kernel parameter (one rank per launch,
// the production multi-GPU form: its fields are constant-bank operands, no
// registers) or a record in global memory (ranks emulated on one device).
template <typename R>
__device__ __forceinline__ void cg1_peer_body(const PeerRankArgs& a, const unsigned lr, const unsigned bid,
                                              const unsigned G, unsigned long long* __restrict__ err, int iters,
                                              const double tol2) {
    extern __shared__ __align__(128) unsigned char tma_smem[];
    __shared__ __align__(8) uint64_t full_bar[CG1_NS], empty_bar[CG1_NS];
    __shared__ double sm_tot, sm2[2];
    constexpr uint32_t AE = 16 / sizeof(R);
    const uint64_t nv = a.nv, ne = a.ne;
    const uint32_t cap = a.cap;
    const uint32_t* __restrict__ index = a.index;
    const uint32_t* __restrict__ head = a.head;
    const R* __restrict__ A = (const R*)a.A;
    const R* __restrict__ dinv = (const R*)a.dinv;
    R* __restrict__ x = (R*)a.x;
    R* __restrict__ r = (R*)a.r;
    const R* __restrict__ z0 = (const R*)a.z0;
    R* __restrict__ p = (R*)a.p;
    R* __restrict__ sv = (R*)a.sv;
    R* __restrict__ yv = (R*)a.yv;
    R* __restrict__ wv = (R*)a.wv;
    R* ub0 = (R*)a.ub0;
    R* ub1 = (R*)a.ub1;
    const uint8_t* __restrict__ mask = a.mask;
    double* __restrict__ scal = a.scal;
    const uint32_t* __restrict__ send_off = a.send_off;
    const uint2* __restrict__ send_dst = a.send_dst;
    const size_t stage_bytes = ((size_t)9 * cap * sizeof(R) + (size_t)cap * 4 + 127) & ~(size_t)127;
    const uint64_t nchunks = (nv + TMA_VCH - 1) / TMA_VCH;
    const uint64_t my_chunks = nchunks > bid ? (nchunks - bid + G - 1) / G : 0;
    const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < CG1_NS; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], PCG_WPG);
        }
        mbar_fence_init();
    }
    __syncthreads();
    uint64_t epoch = a.mbox[kMbEpoch];
    double gam = scal[S_RHO];                 // g_i = r_i . z_i (rank-local after ebb_cg_init)
    double alpha = scal[S_ALPHA];
    double beta = scal[S_PQ];
    int first = scal[S_FIRST] != 0.0;
    int par = scal[S_PAR] != 0.0;
    double rz0 = scal[S_RZ0];
    if (scal[S_DONE] != 0.0) iters = 0;
    int done_it = 0, done_ph = 0;
    bool conv = false;
    if (first && iters > 0) {
        // 1) every rank has run ebb_cg_init; the global r_0.z_0
        double g0, unused;
        peer_exchange(a, bid, epoch++, gam, 0.0, sm2, err, g0, unused);
        gam = g0;
        rz0 = g0;
        // 2) z_0 halo: owners store their rows into the peers' ghost rows
        bool sent = false;
        for (uint64_t v = (uint64_t)bid * blockDim.x + threadIdx.x; v < nv; v += (uint64_t)G * blockDim.x) {
            const uint32_t s0 = send_off[v], s1 = send_off[v + 1];
            if (s0 == s1) continue;
            const auto zv = ld4(z0, v);
            for (uint32_t k = s0; k < s1; ++k) {
                const uint2 d = send_dst[k];
                st4((R*)a.peer_z0[d.x], d.y, zv);
            }
            sent = true;
        }
        rank_barrier(a.bar, G, sent);
        peer_exchange(a, bid, epoch++, 0.0, 0.0, sm2, err, g0, unused);
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
    const int nphase = iters + (first && iters > 0 ? 1 : 0);
    if (warp == TMA_CONSUMERS && lane == 0 && nphase > 0)
        for (uint64_t j = 0; j < my_chunks && j < CG1_NS; ++j) issue(bid + j * G, issued++);
    for (int ph = 0; ph < nphase; ++ph) {
        const bool pro = first != 0;
        const R aa = (R)alpha, b = (R)beta;
        const R* __restrict__ op = pro ? z0 : (par ? ub1 : ub0);
        const bool un1 = pro ? par != 0 : par == 0;          // u_{i+1} goes to buffer 1 (u2)
        R* __restrict__ un = un1 ? ub1 : ub0;
        double pg = 0.0, pd = 0.0;
        bool sent = false;
        if (warp == TMA_CONSUMERS) {
            if (lane == 0) {
                for (uint64_t j = CG1_NS; j < my_chunks; ++j) issue(bid + j * G, issued++);
                if (ph + 1 < nphase)
                    for (uint64_t j = 0; j < my_chunks && j < CG1_NS; ++j) issue(bid + j * G, issued++);
            }
        } else {
            const unsigned grp = warp / PCG_WPG, wig = warp % PCG_WPG;
            const unsigned sub = lane & 7;
            const uint64_t seq0 = (uint64_t)ph * my_chunks;
            for (uint64_t j = grp; j < my_chunks; j += PCG_GROUPS) {
                const uint64_t seq = seq0 + j;
                const uint64_t ch = bid + j * G;
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
                    if (mask && !mask[v]) a0 = a1 = a2 = 0;
                    const auto dv = ld4(dinv, v);
                    const uint32_t s0 = send_off[v], s1 = send_off[v + 1];
                    typename V4<R>::T t;
                    t.w = 0;
                    if (pro) {
                        const auto zv = ld4(z0, v);
                        t.x = a0; t.y = a1; t.z = a2;
                        st4(wv, v, t);
                        t.x = a0 * dv.x; t.y = a1 * dv.y; t.z = a2 * dv.z;
                        st4(un, v, t);
                        for (uint32_t k = s0; k < s1; ++k) {
                            const uint2 d = send_dst[k];
                            st4((R*)(un1 ? a.peer_ub1[d.x] : a.peer_ub0[d.x]), d.y, t);
                        }
                        sent |= s0 != s1;
                        pd += (double)a0 * zv.x + (double)a1 * zv.y + (double)a2 * zv.z;
                    } else {
                        auto rv = ld4(r, v);
                        auto wi = ld4(wv, v);
                        typename V4<R>::T si = wi, yi, pi;
                        yi.x = a0; yi.y = a1; yi.z = a2; yi.w = 0;
                        pi.x = rv.x * dv.x; pi.y = rv.y * dv.y; pi.z = rv.z * dv.z; pi.w = 0;
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
                        const R x0 = x[3 * v] + aa * pi.x, x1 = x[3 * v + 1] + aa * pi.y, x2 = x[3 * v + 2] + aa * pi.z;
                        x[3 * v] = x0;
                        x[3 * v + 1] = x1;
                        x[3 * v + 2] = x2;
                        rv.x -= aa * si.x; rv.y -= aa * si.y; rv.z -= aa * si.z; rv.w = 0;
                        wi.x -= aa * yi.x; wi.y -= aa * yi.y; wi.z -= aa * yi.z; wi.w = 0;
                        st4(r, v, rv);
                        st4(wv, v, wi);
                        t.x = wi.x * dv.x; t.y = wi.y * dv.y; t.z = wi.z * dv.z;
                        st4(un, v, t);
                        for (uint32_t k = s0; k < s1; ++k) {
                            const uint2 d = send_dst[k];
                            st4((R*)(un1 ? a.peer_ub1[d.x] : a.peer_ub0[d.x]), d.y, t);
                            R* px = (R*)a.peer_x[d.x] + 3 * (uint64_t)d.y;
                            px[0] = x0;
                            px[1] = x1;
                            px[2] = x2;
                        }
                        sent |= s0 != s1;
                        const R zx = rv.x * dv.x, zy = rv.y * dv.y, zz = rv.z * dv.z;
                        pg += (double)rv.x * zx + (double)rv.y * zy + (double)rv.z * zz;
                        pd += (double)wi.x * zx + (double)wi.y * zy + (double)wi.z * zz;
                    }
                }
            }
        }
        pg = block_reduce<ROP_SUM>(pg);
        pd = block_reduce<ROP_SUM>(pd);
        double* const pgb = a.part + (ph & 1) * 2 * kCg1PartStride;
        double* const pdb = pgb + kCg1PartStride;
        if (threadIdx.x == 0) {
            pgb[bid] = pg;
            pdb[bid] = pd;
        }
        rank_barrier(a.bar, G, sent);
        const double dl = grid_sum_partials(pdb, G, &sm_tot);
        const double gl = pro ? 0.0 : grid_sum_partials(pgb, G, &sm_tot);
        double dsum, gnew;
        peer_exchange(a, bid, epoch++, dl, gl, sm2, err, dsum, gnew);
        if (pro) {
            if (lr == 0 && bid == 0 && threadIdx.x == 0 && dsum < 0.0) atomicAdd(&err[ERR_NOT_SPD], 1ull);
            alpha = dsum != 0.0 ? gam / dsum : 0.0;
            beta = 0.0;
            first = 0;
        } else {
            const double bn = gam != 0.0 ? gnew / gam : 0.0;
            const double den = dsum - (alpha != 0.0 ? bn * gnew / alpha : 0.0);
            if (lr == 0 && bid == 0 && threadIdx.x == 0 && den < 0.0) atomicAdd(&err[ERR_NOT_SPD], 1ull);
            alpha = den != 0.0 ? gnew / den : 0.0;
            beta = bn;
            gam = gnew;
            par ^= 1;
        }
        ++done_ph;
        if (!pro) {
            ++done_it;
            if (tol2 > 0.0 && gam <= tol2 * rz0) {   // global sums: the same exit on every rank
                conv = true;
                break;
            }
        }
    }
    if (warp == TMA_CONSUMERS && lane == 0)
        for (uint64_t sq = (uint64_t)done_ph * my_chunks; sq < issued; ++sq)
            mbar_wait(&full_bar[sq % CG1_NS], (uint32_t)((sq / CG1_NS) & 1u));
    if (bid == 0 && threadIdx.x == 0) {
        scal[S_ITERS] += (double)done_it;
        if (conv) scal[S_DONE] = 1.0;
        scal[S_RHO] = gam;
        scal[S_RZ] = gam;
        scal[S_RZ0] = rz0;
        scal[S_ALPHA] = alpha;
        scal[S_PQ] = beta;
        scal[S_FIRST] = first ? 1.0 : 0.0;
        scal[S_PAR] = par ? 1.0 : 0.0;
        *a.rho_user = gam;
        a.mbox[kMbEpoch] = epoch;
    }
}

// Saad Alg. 9.1 (the single-GPU k_cg_persistent's iterates and phases) with
// the same peer-memory halo and mailbox exchanges, for ranks whose vector
// records stream from HBM (~1e7 tets per GPU), where Saad's two gathered
// vectors cost less than the single-reduction form's nine owner records
// (DESIGN.md §5.4).  Per iteration two exchanges (p.q after the matvec, r.z
// after the update).  Ghost rows: z arrives from the owners (stored by the
// owner's update phase); the direction p = z + beta p_old of a ghost row is
// formed by the receiver (a ghost pass in the matvec phase writes it into the
// new p buffer; gatherers form it on the fly as on one GPU); x arrives from
// the owners.  Owners store z and x rows during the update phase, which
// peers reach only after the p.q exchange, i.e. after this rank's matvec
// phase (including the ghost pass) read the old z.
template <typename R>
__device__ __forceinline__ void cg_saad_peer_body(const PeerRankArgs& a, const unsigned lr, const unsigned bid,
                                                  const unsigned G, unsigned long long* __restrict__ err,
                                                  int iters, const double tol2) {
    extern __shared__ __align__(128) unsigned char tma_smem[];
    __shared__ __align__(8) uint64_t full_bar[TMA_NS], empty_bar[TMA_NS];
    __shared__ double sm_tot, sm2[2];
    constexpr uint32_t AE = 16 / sizeof(R);
    const uint64_t nv = a.nv, ne = a.ne, nv_all = a.nv_all;
    const uint32_t cap = a.cap;
    const uint32_t* __restrict__ index = a.index;
    const uint32_t* __restrict__ head = a.head;
    const R* __restrict__ A = (const R*)a.A;
    const R* __restrict__ dinv = (const R*)a.dinv;
    R* __restrict__ x = (R*)a.x;
    R* __restrict__ r = (R*)a.r;
    R* __restrict__ z = (R*)a.z0;
    R* __restrict__ q = (R*)a.q;
    R* pb0 = (R*)a.p;
    R* pb1 = (R*)a.p2;
    const uint8_t* __restrict__ mask = a.mask;
    double* __restrict__ scal = a.scal;
    const uint32_t* __restrict__ send_off = a.send_off;
    const uint2* __restrict__ send_dst = a.send_dst;
    double* __restrict__ part_pq = a.part;
    double* __restrict__ part_rz = a.part + kCg1PartStride;
    const size_t stage_bytes = ((size_t)9 * cap * sizeof(R) + (size_t)cap * 4 + 127) & ~(size_t)127;
    const uint64_t nchunks = (nv + TMA_VCH - 1) / TMA_VCH;
    const uint64_t my_chunks = nchunks > bid ? (nchunks - bid + G - 1) / G : 0;
    const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < TMA_NS; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], PCG_WPG);
        }
        mbar_fence_init();
    }
    __syncthreads();
    uint64_t epoch = a.mbox[kMbEpoch];
    double rho = scal[S_RHO];
    int first = scal[S_FIRST] != 0.0;
    int cur = scal[S_PAR] != 0.0;
    double rz_new = scal[S_RZ];
    double rz0 = scal[S_RZ0];
    if (scal[S_DONE] != 0.0) iters = 0;
    int done_it = 0;
    bool conv = false;
    const uint64_t gthreads = (uint64_t)G * blockDim.x;
    const uint64_t gtid = (uint64_t)bid * blockDim.x + threadIdx.x;
    if (first && iters > 0) {
        // the global r_0.z_0 (every rank has initialised), then the z_0 halo
        double g0, unused;
        peer_exchange(a, bid, epoch++, rz_new, 0.0, sm2, err, g0, unused);
        rz_new = g0;
        rho = g0;
        rz0 = g0;
        bool sent = false;
        for (uint64_t v = gtid; v < nv; v += gthreads) {
            const uint32_t s0 = send_off[v], s1 = send_off[v + 1];
            if (s0 == s1) continue;
            const auto zv = ld4(z, v);
            for (uint32_t k = s0; k < s1; ++k) {
                const uint2 d = send_dst[k];
                st4((R*)a.peer_z0[d.x], d.y, zv);
            }
            sent = true;
        }
        rank_barrier(a.bar, G, sent);
        peer_exchange(a, bid, epoch++, 0.0, 0.0, sm2, err, g0, unused);
    }
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
        for (uint64_t j = 0; j < my_chunks && j < TMA_NS; ++j) issue(bid + j * G, issued++);
    for (int it = 0; it < iters; ++it) {
        const R beta = (first || rho == 0.0) ? R(0) : (R)(rz_new / rho);
        const R* __restrict__ pold = cur ? pb1 : pb0;
        R* __restrict__ pnew = cur ? pb0 : pb1;
        double pq = 0.0;
        if (warp == TMA_CONSUMERS) {
            if (lane == 0) {
                for (uint64_t j = TMA_NS; j < my_chunks; ++j) issue(bid + j * G, issued++);
                if (it + 1 < iters)
                    for (uint64_t j = 0; j < my_chunks && j < TMA_NS; ++j) issue(bid + j * G, issued++);
            }
        } else {
            const unsigned grp = warp / PCG_WPG, wig = warp % PCG_WPG;
            const unsigned sub = lane & 7;
            const uint64_t seq0 = (uint64_t)it * my_chunks;
            for (uint64_t j = grp; j < my_chunks; j += PCG_GROUPS) {
                const uint64_t seq = seq0 + j;
                const uint64_t ch = bid + j * G;
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
                    const uint32_t rr1 = rb + 8;
                    const bool two = rr1 < r1;
                    const uint32_t h0 = hs[rb], h1 = two ? hs[rr1] : h0;
                    const auto z0v = ld4cg(z, h0);
                    const auto o0 = ld4cg(pold, h0);
                    const auto z1v = ld4cg(z, h1);
                    const auto o1 = ld4cg(pold, h1);
                    R av[9], bv[9];
#pragma unroll
                    for (int c = 0; c < 9; ++c) {
                        const R* pl = reinterpret_cast<const R*>(base + (size_t)c * cap * sizeof(R)) + off[c];
                        av[c] = pl[rb];
                        bv[c] = two ? pl[rr1] : R(0);
                    }
                    const R px = z0v.x + beta * o0.x, py = z0v.y + beta * o0.y, pz = z0v.z + beta * o0.z;
                    const R qx = z1v.x + beta * o1.x, qy = z1v.y + beta * o1.y, qz = z1v.z + beta * o1.z;
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
            // ghost rows: the new direction from the owners' z (they are
            // gathered on the fly in this phase; stored for the next one)
            for (uint64_t g = nv + (uint64_t)bid * (blockDim.x - 32) + threadIdx.x; g < nv_all;
                 g += (uint64_t)G * (blockDim.x - 32)) {
                const auto zv = ld4cg(z, g);
                const auto ov = ld4cg(pold, g);
                typename V4<R>::T pv;
                pv.x = zv.x + beta * ov.x;
                pv.y = zv.y + beta * ov.y;
                pv.z = zv.z + beta * ov.z;
                pv.w = 0;
                st4(pnew, g, pv);
            }
        }
        pq = block_reduce<ROP_SUM>(pq);
        if (threadIdx.x == 0) part_pq[bid] = pq;
        rank_barrier(a.bar, G, false);
        double pqs, unused;
        peer_exchange(a, bid, epoch++, grid_sum_partials(part_pq, G, &sm_tot), 0.0, sm2, err, pqs, unused);
        if (lr == 0 && bid == 0 && threadIdx.x == 0 && pqs < 0.0) atomicAdd(&err[ERR_NOT_SPD], 1ull);
        rho = rz_new;
        first = 0;
        cur ^= 1;
        const R alpha = (pqs != 0.0) ? (R)(rho / pqs) : R(0);
        double acc = 0.0;
        bool sent = false;
        for (uint64_t vv = gtid; vv < nv; vv += gthreads) {
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
            const R x0 = x[3 * vv] + alpha * pv.x, x1 = x[3 * vv + 1] + alpha * pv.y,
                    x2 = x[3 * vv + 2] + alpha * pv.z;
            x[3 * vv] = x0;
            x[3 * vv + 1] = x1;
            x[3 * vv + 2] = x2;
            const uint32_t s0 = send_off[vv], s1 = send_off[vv + 1];
            for (uint32_t k = s0; k < s1; ++k) {
                const uint2 d = send_dst[k];
                st4((R*)a.peer_z0[d.x], d.y, zv);
                R* px = (R*)a.peer_x[d.x] + 3 * (uint64_t)d.y;
                px[0] = x0;
                px[1] = x1;
                px[2] = x2;
            }
            sent |= s0 != s1;
            acc += (double)rv.x * zv.x + (double)rv.y * zv.y + (double)rv.z * zv.z;
        }
        acc = block_reduce<ROP_SUM>(acc);
        if (threadIdx.x == 0) part_rz[bid] = acc;
        rank_barrier(a.bar, G, sent);
        peer_exchange(a, bid, epoch++, grid_sum_partials(part_rz, G, &sm_tot), 0.0, sm2, err, rz_new, unused);
        if (bid == 0 && threadIdx.x == 0) scal[S_PQ] = pqs;
        ++done_it;
        if (tol2 > 0.0 && rz_new <= tol2 * rz0) {   // global sums: the same exit on every rank
            conv = true;
            break;
        }
    }
    if (warp == TMA_CONSUMERS && lane == 0)
        for (uint64_t sq = (uint64_t)done_it * my_chunks; sq < issued; ++sq)
            mbar_wait(&full_bar[sq % TMA_NS], (uint32_t)((sq / TMA_NS) & 1u));
    if (bid == 0 && threadIdx.x == 0) {
        scal[S_RHO] = rho;
        scal[S_RZ] = rz_new;
        scal[S_RZ0] = rz0;
        scal[S_FIRST] = first ? 1.0 : 0.0;
        scal[S_PAR] = cur ? 1.0 : 0.0;
        scal[S_ITERS] += (double)done_it;
        if (conv) scal[S_DONE] = 1.0;
        *a.rho_user = rz_new;
        a.mbox[kMbEpoch] = epoch;
    }
}

// one rank per launch (a process per GPU): the record is a kernel parameter
// (min 3 CTAs per SM, the single-GPU kernels' occupancy: unbounded the
// single-reduction body takes 84 registers, two CTAs per SM)
template <typename R, bool SAAD>
__global__ void __launch_bounds__(32 * (TMA_CONSUMERS + 1), 3)
    k_cg_peer1(const __grid_constant__ PeerRankArgs a, unsigned long long* __restrict__ err, int iters,
               double tol2) {
    if constexpr (SAAD) cg_saad_peer_body<R>(a, 0u, blockIdx.x, gridDim.x, err, iters, tol2);
    else cg1_peer_body<R>(a, 0u, blockIdx.x, gridDim.x, err, iters, tol2);
}

// several ranks emulated on one device in one cooperative launch: records in
// global memory (min 3 CTAs per SM: 72 registers; unbounded, the loaded
// record pointers take 132 registers and one CTA per SM)
#ifndef PEER_MINB
#define PEER_MINB 3
#endif
template <typename R, bool SAAD>
__global__ void __launch_bounds__(32 * (TMA_CONSUMERS + 1), PEER_MINB)
    k_cg_peer(const PeerRankArgs* __restrict__ ranks, unsigned G, unsigned long long* __restrict__ err, int iters,
              double tol2) {
    const unsigned lr = blockIdx.x / G;
    if constexpr (SAAD) cg_saad_peer_body<R>(ranks[lr], lr, blockIdx.x - lr * G, G, err, iters, tol2);
    else cg1_peer_body<R>(ranks[lr], lr, blockIdx.x - lr * G, G, err, iters, tol2);
}

// ---------------------------------------------------------------------------
// Halo of a field over peer memory (ebb_peer_halo_push; SURVEY §8(e) "halo
// exchange of vertex positions and of the partial force sums"):
//   COPY  the owners store the rows peers hold as ghosts straight into the
//         peers' copies of the field (positions: owners -> ghosts);
//   ADD   the partial rows this rank computed for rows another rank owns are
//         added into the owners' rows with red.global.add over peer memory
//         (the reverse add of partial f / K rows: ghost tails -> owners).
// One mailbox exchange first (every rank has reached the push, so no peer
// still reads the ghost rows a COPY overwrites, and every owner has written
// the rows an ADD adds into), the stores / REDs, a rank barrier, one
// exchange more: when the kernel ends on a rank its rows are current.  The
// same mailboxes and epoch counter as the fused PCG.  Element-major fields
// move rows of `comps` elements; component-planar (SOA) fields one element
// per plane (plane stride = the relation's rows, the peer's for its copy).
struct HaloRankArgs {
    const void* src;
    uint64_t n_src;                    // source rows [0, n_src) may send (CSR rows)
    uint64_t n_rows;                   // rows of the source relation (SOA plane stride)
    uint32_t comps, esize;             // elements per row, bytes per element (4 | 8)
    int soa, add, is_f64, pad;
    const uint32_t* send_off;
    const uint2* send_dst;
    unsigned long long* mbox;
    unsigned int* bar;
    void* peer_dst[kPeerMax];
    uint64_t peer_rows[kPeerMax];      // the peers' relation rows (their SOA plane stride)
    unsigned long long* peer_mbox[kPeerMax];
    int rank, nranks;
};

template <typename T>
__device__ __forceinline__ void halo_move(const HaloRankArgs& a, const T* src, uint64_t v, const uint2 d) {
    T* dst = (T*)a.peer_dst[d.x];
    const uint64_t pr = a.peer_rows[d.x];
    for (uint32_t c = 0; c < a.comps; ++c) {
        const T x = a.soa ? src[c * a.n_rows + v] : src[v * a.comps + c];
        T* p = a.soa ? dst + c * pr + d.y : dst + (uint64_t)d.y * a.comps + c;
        if constexpr (sizeof(T) == 8 && !std::is_same<T, double>::value) {
            *p = x;
        } else if constexpr (sizeof(T) == 4 && !std::is_same<T, float>::value) {
            *p = x;
        } else {
            atomicAdd(p, x);   // float / double: ADD mode only (COPY moves integer words)
        }
    }
}

__global__ void __launch_bounds__(256) k_peer_halo(const HaloRankArgs* __restrict__ recs, unsigned G,
                                                   unsigned long long* __restrict__ err) {
    __shared__ double sm2[2];
    const unsigned lr = blockIdx.x / G, bid = blockIdx.x - lr * G;
    const HaloRankArgs& a = recs[lr];
    const uint64_t epoch = a.mbox[kMbEpoch];
    double x0, x1;
    peer_exchange(a, bid, epoch, 0.0, 0.0, sm2, err, x0, x1);   // every rank is here
    bool sent = false;
    for (uint64_t v = (uint64_t)bid * blockDim.x + threadIdx.x; v < a.n_src; v += (uint64_t)G * blockDim.x) {
        const uint32_t s0 = a.send_off[v], s1 = a.send_off[v + 1];
        if (s0 == s1) continue;
        for (uint32_t k = s0; k < s1; ++k) {
            const uint2 d = a.send_dst[k];
            if (!a.add) {
                if (a.esize == 8) halo_move<unsigned long long>(a, (const unsigned long long*)a.src, v, d);
                else halo_move<uint32_t>(a, (const uint32_t*)a.src, v, d);
            } else if (a.is_f64) {
                halo_move<double>(a, (const double*)a.src, v, d);
            } else {
                halo_move<float>(a, (const float*)a.src, v, d);
            }
        }
        sent = true;
    }
    rank_barrier(a.bar, G, sent);
    peer_exchange(a, bid, epoch + 1, 0.0, 0.0, sm2, err, x0, x1);   // every rank's rows have landed
    if (bid == 0 && threadIdx.x == 0) a.mbox[kMbEpoch] = epoch + 2;
}

// launch group of ebb_cg_peer_bind: the per-rank records on the device and
// each rank's grid-barrier words and reduction partials
struct PeerGroup {
    int nlocal = 0;
    unsigned G = 0;                    // CTAs per rank
    size_t smem = 0;
    ebb_dtype dt = EBB_F64;
    bool saad = false;                 // Saad body (else single-reduction)
    double tol2 = 0.0;
    PeerRankArgs* d_args = nullptr;
    PeerRankArgs one;                  // nlocal == 1: the record passed as a kernel parameter
    std::vector<ebb_field> fields;     // every field a record points into (checked at each step)
    HaloRankArgs* d_halo = nullptr;    // halo groups (ebb_peer_halo_bind): the records of k_peer_halo
    bool noop = false;                 // halo group of a one-rank job
    double* d_part = nullptr;
    unsigned int* d_bar = nullptr;
};

// the kernel of a group: one rank per launch or emulated ranks, Saad or
// single-reduction body
template <typename R>
void* peer_kernel(int nlocal, bool saad) {
    if (nlocal == 1) return saad ? (void*)k_cg_peer1<R, true> : (void*)k_cg_peer1<R, false>;
    return saad ? (void*)k_cg_peer<R, true> : (void*)k_cg_peer<R, false>;
}

template <typename R>
ebb_status peer_occupancy(Ctx* c, size_t smem, int nlocal, bool saad, int* nb) {
    static thread_local size_t configured_dev[4][kMaxDevices] = {};
    size_t& configured = configured_dev[(nlocal == 1) * 2 + saad][c->device % kMaxDevices];
    const void* k = peer_kernel<R>(nlocal, saad);
    if (smem > configured) {
        EBB_CUDA(c, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    EBB_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(nb, k, 32 * (TMA_CONSUMERS + 1), smem));
    return EBB_OK;
}

}  // namespace

namespace ebb {
void peer_release(Ctx* c) {
    for (void* g : c->peer_groups) {
        PeerGroup* P = (PeerGroup*)g;
        if (!P) continue;
        cudaFree(P->d_args);
        cudaFree(P->d_part);
        cudaFree(P->d_bar);
        if (P->d_halo) cudaFree(P->d_halo);
        delete P;
    }
    c->peer_groups.clear();
}
}  // namespace ebb

extern "C" {

ebb_status ebb_cg_peer_bind(ebb_ctx ctx, int32_t nlocal, const ebb_cg* cgs, const ebb_peer_cg* peers,
                            int32_t* group_out) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !cgs || !peers || !group_out) return fail(c, EBB_E_ARG, "null argument");
    if (nlocal < 1 || nlocal > EBB_MAX_RANKS) return fail(c, EBB_E_ARG, "peer_bind: nlocal must be 1..%d", EBB_MAX_RANKS);
    std::vector<PeerRankArgs> h(nlocal);
    ebb_dtype dt0 = EBB_F64;
    bool saad = false;
    size_t stage_max = 0;
    std::vector<ebb_field> used;
    for (int i = 0; i < nlocal; ++i) {
        const ebb_cg* cg = &cgs[i];
        const ebb_peer_cg* pc = &peers[i];
        EdgeGraph Gr;
        ebb_dtype dt;
        EBB_TRY(cg_validate(c, cg, &Gr, &dt));
        if (i == 0) dt0 = dt;
        if (dt != dt0) return fail(c, EBB_E_TYPE, "peer_bind: every rank of a group must have the same dtype");
        const int var = cg_variant(cg, Gr, dt);
        if (var != EBB_CG_SAAD && var != EBB_CG_SINGLE_REDUCTION)
            return fail(c, EBB_E_ARG, "peer_bind: rank %d: the fused PCG runs the Saad or the single-reduction "
                        "variant", i);
        if (i == 0) saad = var == EBB_CG_SAAD;
        if ((var == EBB_CG_SAAD) != saad) return fail(c, EBB_E_ARG, "peer_bind: every rank needs the same variant");
        for (ebb_field f : {cg->dinv, cg->r, cg->z, cg->p, cg->scal, cg->rho})
            if (!get_field(c, f))
                return fail(c, EBB_E_STATE, "peer_bind: rank %d: call ebb_cg_init first", i);
        if (saad) {
            for (ebb_field f : {cg->q, cg->p2})
                if (!get_field(c, f)) return fail(c, EBB_E_STATE, "peer_bind: rank %d: call ebb_cg_init first", i);
        } else {
            for (ebb_field f : {cg->s, cg->y, cg->w, cg->u, cg->u2})
                if (!get_field(c, f))
                    return fail(c, EBB_E_STATE, "peer_bind: rank %d: call ebb_cg_init with EBB_CG_SINGLE_REDUCTION "
                                "first (its work vectors are missing)", i);
        }
        if (cg->tol != cgs[0].tol) return fail(c, EBB_E_ARG, "peer_bind: every rank needs the same tol");
        if (pc->nranks < 1 || pc->nranks > EBB_MAX_RANKS || pc->rank < 0 || pc->rank >= pc->nranks ||
            pc->nranks != peers[0].nranks)
            return fail(c, EBB_E_ARG, "peer_bind: rank %d: bad rank / nranks (%d / %d)", i, pc->rank, pc->nranks);
        for (int j = 0; j < i; ++j)
            if (peers[j].rank == pc->rank) return fail(c, EBB_E_ARG, "peer_bind: rank %d bound twice", pc->rank);
        if (pc->n_owned > Gr.nv) return fail(c, EBB_E_SIZE, "peer_bind: n_owned exceeds the local vertex count");
        Field* SO = get_field(c, pc->send_off);
        Field* SD = get_field(c, pc->send_dst);
        Field* MB = get_field(c, pc->mbox);
        if (!SO || SO->dtype != EBB_U32 || SO->comps() != 1 || c->rels[SO->rel].size != pc->n_owned + 1)
            return fail(c, EBB_E_TYPE, "peer_bind: send_off must be a U32 field of n_owned + 1 rows");
        if (!SD || SD->dtype != EBB_U32 || SD->comps() != 2)
            return fail(c, EBB_E_TYPE, "peer_bind: send_dst must be a U32 2x1 field");
        if (!MB || MB->dtype != EBB_F64 || MB->comps() != 1 || c->rels[MB->rel].size < EBB_PEER_MBOX_WORDS)
            return fail(c, EBB_E_TYPE, "peer_bind: mbox must be an F64 field of >= %d rows", EBB_PEER_MBOX_WORDS);
        for (int q = 0; q < pc->nranks; ++q)
            if (q != pc->rank && (!pc->peer_x[q] || !pc->peer_z[q] || !pc->peer_mbox[q] ||
                                  (!saad && (!pc->peer_u[q] || !pc->peer_u2[q]))))
                return fail(c, EBB_E_ARG, "peer_bind: rank %d: missing buffer address of peer %d", pc->rank, q);
        const uint8_t* mask;
        EBB_TRY(check_mask(c, cg->mask, Gr.verts, &mask));
        const uint32_t cap = dt == EBB_F64 ? tma_cap<double>(Gr.max_chunk16) : tma_cap<float>(Gr.max_chunk16);
        const size_t es = dt == EBB_F64 ? 8 : 4;
        const size_t stage = ((size_t)9 * cap * es + (size_t)cap * 4 + 127) & ~(size_t)127;
        if (stage > stage_max) stage_max = stage;
        auto F = [&](ebb_field f) { return c->fields[f].ptr; };
        PeerRankArgs& a = h[i];
        memset(&a, 0, sizeof(a));
        a.nv = pc->n_owned;
        a.ne = Gr.ne;
        a.index = Gr.index;
        a.head = Gr.head;
        a.A = F(cg->A);
        a.dinv = F(cg->dinv);
        a.x = F(cg->x);
        a.r = F(cg->r);
        a.z0 = F(cg->z);
        a.p = F(cg->p);
        if (!saad) {
            a.sv = F(cg->s);
            a.yv = F(cg->y);
            a.wv = F(cg->w);
            a.ub0 = F(cg->u);
            a.ub1 = F(cg->u2);
        } else {
            a.q = F(cg->q);
            a.p2 = F(cg->p2);
        }
        a.nv_all = Gr.nv;
        a.mask = mask;
        a.scal = (double*)F(cg->scal);
        a.rho_user = (double*)F(cg->rho);
        a.send_off = (const uint32_t*)SO->ptr;
        a.send_dst = (const uint2*)SD->ptr;
        a.mbox = (unsigned long long*)MB->ptr;
        for (int q = 0; q < pc->nranks; ++q) {
            a.peer_ub0[q] = (void*)(uintptr_t)pc->peer_u[q];
            a.peer_ub1[q] = (void*)(uintptr_t)pc->peer_u2[q];
            a.peer_x[q] = (void*)(uintptr_t)pc->peer_x[q];
            a.peer_z0[q] = (void*)(uintptr_t)pc->peer_z[q];
            a.peer_mbox[q] = (unsigned long long*)(uintptr_t)pc->peer_mbox[q];
        }
        a.rank = pc->rank;
        a.nranks = pc->nranks;
        a.cap = cap;
        for (ebb_field f : {cg->A, cg->dinv, cg->x, cg->r, cg->z, cg->p, cg->scal, cg->rho, pc->send_off,
                            pc->send_dst, pc->mbox})
            used.push_back(f);
        if (cg->mask != EBB_NONE) used.push_back(cg->mask);
        for (ebb_field f : saad ? std::vector<ebb_field>{cg->q, cg->p2}
                                : std::vector<ebb_field>{cg->s, cg->y, cg->w, cg->u, cg->u2})
            used.push_back(f);
    }
    const size_t smem = stage_max * (saad ? TMA_NS : CG1_NS);
    if (smem > kTmaSmemMax) return fail(c, EBB_E_SIZE, "peer_bind: TMA ring of %zu bytes does not fit", smem);
    int nb = 0;
    if (dt0 == EBB_F64) EBB_TRY(peer_occupancy<double>(c, smem, nlocal, saad, &nb));
    else EBB_TRY(peer_occupancy<float>(c, smem, nlocal, saad, &nb));
    unsigned G = (unsigned)((uint64_t)nb * c->num_sms / (uint64_t)nlocal);
    if (G > kCg1PartStride) G = kCg1PartStride;
    if (G < 1) return fail(c, EBB_E_SIZE, "peer_bind: %d ranks cannot all be resident on one device", nlocal);
    PeerGroup* P = new PeerGroup();
    P->nlocal = nlocal;
    P->G = G;
    P->smem = smem;
    P->dt = dt0;
    P->saad = saad;
    P->fields = used;
    P->tol2 = cg_tol2(&cgs[0]);
    c->peer_groups.push_back(P);
    EBB_CUDA(c, cudaMalloc(&P->d_args, sizeof(PeerRankArgs) * nlocal));
    EBB_CUDA(c, cudaMalloc(&P->d_part, sizeof(double) * 4 * kCg1PartStride * nlocal));
    EBB_CUDA(c, cudaMalloc(&P->d_bar, sizeof(unsigned int) * 2 * nlocal));
    EBB_CUDA(c, cudaMemset(P->d_bar, 0, sizeof(unsigned int) * 2 * nlocal));
    for (int i = 0; i < nlocal; ++i) {
        h[i].part = P->d_part + (size_t)i * 4 * kCg1PartStride;
        h[i].bar = P->d_bar + 2 * i;
    }
    EBB_CUDA(c, cudaMemcpy(P->d_args, h.data(), sizeof(PeerRankArgs) * nlocal, cudaMemcpyHostToDevice));
    P->one = h[0];
    *group_out = (int32_t)(c->peer_groups.size() - 1);
    return EBB_OK;
}

ebb_status ebb_cg_peer_step(ebb_ctx ctx, int32_t group, int32_t iters, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c) return EBB_E_ARG;
    if (group < 0 || (size_t)group >= c->peer_groups.size() || !c->peer_groups[group])
        return fail(c, EBB_E_ARG, "peer_step: bad group %d", group);
    if (iters < 0) return fail(c, EBB_E_ARG, "negative iteration count");
    PeerGroup* P = (PeerGroup*)c->peer_groups[group];
    if (P->d_halo) return fail(c, EBB_E_ARG, "peer_step: group %d is a halo group", group);
    for (ebb_field f : P->fields)
        if (!get_field(c, f)) return fail(c, EBB_E_STATE, "peer_step: a field of group %d was freed", group);
    cudaStream_t s = (cudaStream_t)stream;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P->G * (unsigned)P->nlocal);
    cfg.blockDim = dim3(32 * (TMA_CONSUMERS + 1));
    cfg.dynamicSmemBytes = P->smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;   // every CTA of every local rank resident at once
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    KernelTimer kt(c, EBB_K_CG_SOLVE, s);
    const void* k = P->dt == EBB_F64 ? peer_kernel<double>(P->nlocal, P->saad) : peer_kernel<float>(P->nlocal, P->saad);
    unsigned long long* err = c->d_err;
    int it = (int)iters;
    double tol2 = P->tol2;
    const PeerRankArgs* recs = P->d_args;
    unsigned G = P->G;
    void* one_args[] = {(void*)&P->one, (void*)&err, (void*)&it, (void*)&tol2};
    void* multi_args[] = {(void*)&recs, (void*)&G, (void*)&err, (void*)&it, (void*)&tol2};
    EBB_CUDA(c, cudaLaunchKernelExC(&cfg, k, P->nlocal == 1 ? one_args : multi_args));
    return EBB_OK;
}

ebb_status ebb_peer_halo_bind(ebb_ctx ctx, int32_t nlocal, const ebb_peer_halo* descs, int32_t* group_out) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !descs || !group_out) return fail(c, EBB_E_ARG, "null argument");
    if (nlocal < 1 || nlocal > EBB_MAX_RANKS) return fail(c, EBB_E_ARG, "halo_bind: nlocal must be 1..%d", EBB_MAX_RANKS);
    std::vector<HaloRankArgs> h(nlocal);
    std::vector<ebb_field> used;
    for (int i = 0; i < nlocal; ++i) {
        const ebb_peer_halo* d = &descs[i];
        if (d->nranks < 1 || d->nranks > EBB_MAX_RANKS || d->rank < 0 || d->rank >= d->nranks ||
            d->nranks != descs[0].nranks)
            return fail(c, EBB_E_ARG, "halo_bind: rank %d: bad rank / nranks (%d / %d)", i, d->rank, d->nranks);
        for (int j = 0; j < i; ++j)
            if (descs[j].rank == d->rank) return fail(c, EBB_E_ARG, "halo_bind: rank %d bound twice", d->rank);
        Field* F = get_field(c, d->field);
        if (!F || F->dtype == EBB_KEY) return fail(c, EBB_E_TYPE, "halo_bind: bad or key field");
        const size_t es = dtype_size(F->dtype);
        if (es != 4 && es != 8) return fail(c, EBB_E_TYPE, "halo_bind: elements must be 4 or 8 bytes");
        if (d->mode != EBB_HALO_COPY && d->mode != EBB_HALO_ADD) return fail(c, EBB_E_ARG, "halo_bind: bad mode");
        if (d->mode == EBB_HALO_ADD && F->dtype != EBB_F64 && F->dtype != EBB_F32)
            return fail(c, EBB_E_TYPE, "halo_bind: EBB_HALO_ADD needs an F32 / F64 field");
        if (d->n_src > c->rels[F->rel].size) return fail(c, EBB_E_SIZE, "halo_bind: n_src exceeds the rows");
        Field* SO = get_field(c, d->send_off);
        Field* SD = get_field(c, d->send_dst);
        Field* MB = get_field(c, d->mbox);
        if (!SO || SO->dtype != EBB_U32 || SO->comps() != 1 || c->rels[SO->rel].size != d->n_src + 1)
            return fail(c, EBB_E_TYPE, "halo_bind: send_off must be a U32 field of n_src + 1 rows");
        if (!SD || SD->dtype != EBB_U32 || SD->comps() != 2)
            return fail(c, EBB_E_TYPE, "halo_bind: send_dst must be a U32 2x1 field");
        if (!MB || MB->dtype != EBB_F64 || MB->comps() != 1 || c->rels[MB->rel].size < EBB_PEER_MBOX_WORDS)
            return fail(c, EBB_E_TYPE, "halo_bind: mbox must be an F64 field of >= %d rows", EBB_PEER_MBOX_WORDS);
        for (int q = 0; q < d->nranks; ++q)
            if (q != d->rank && (!d->peer_field[q] || !d->peer_mbox[q] ||
                                 (F->layout == EBB_SOA && F->comps() > 1 && !d->peer_rows[q])))
                return fail(c, EBB_E_ARG, "halo_bind: rank %d: missing buffer address / rows of peer %d", d->rank, q);
        HaloRankArgs& a = h[i];
        memset(&a, 0, sizeof(a));
        a.src = F->ptr;
        a.n_src = d->n_src;
        a.n_rows = c->rels[F->rel].size;
        a.comps = F->comps();
        a.esize = (uint32_t)es;
        a.soa = F->layout == EBB_SOA && F->comps() > 1;
        a.add = d->mode == EBB_HALO_ADD;
        a.is_f64 = F->dtype == EBB_F64;
        a.send_off = (const uint32_t*)SO->ptr;
        a.send_dst = (const uint2*)SD->ptr;
        a.mbox = (unsigned long long*)MB->ptr;
        for (int q = 0; q < d->nranks; ++q) {
            a.peer_dst[q] = (void*)(uintptr_t)d->peer_field[q];
            a.peer_rows[q] = d->peer_rows[q];
            a.peer_mbox[q] = (unsigned long long*)(uintptr_t)d->peer_mbox[q];
        }
        a.rank = d->rank;
        a.nranks = d->nranks;
        for (ebb_field f : {d->field, d->send_off, d->send_dst, d->mbox}) used.push_back(f);
    }
    int nb = 0;
    EBB_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_peer_halo, 256, 0));
    unsigned G = (unsigned)c->num_sms;                 // one CTA per SM and rank: a light copy kernel
    if ((uint64_t)G * nlocal > (uint64_t)nb * c->num_sms) G = (unsigned)((uint64_t)nb * c->num_sms / nlocal);
    if (G < 1) return fail(c, EBB_E_SIZE, "halo_bind: %d ranks cannot all be resident", nlocal);
    PeerGroup* P = new PeerGroup();
    P->nlocal = nlocal;
    P->G = G;
    P->fields = used;
    P->noop = descs[0].nranks == 1;    // a one-rank job has no peer and no ghost row
    c->peer_groups.push_back(P);
    EBB_CUDA(c, cudaMalloc(&P->d_halo, sizeof(HaloRankArgs) * nlocal));
    EBB_CUDA(c, cudaMalloc(&P->d_bar, sizeof(unsigned int) * 2 * nlocal));
    EBB_CUDA(c, cudaMemset(P->d_bar, 0, sizeof(unsigned int) * 2 * nlocal));
    for (int i = 0; i < nlocal; ++i) h[i].bar = P->d_bar + 2 * i;
    EBB_CUDA(c, cudaMemcpy(P->d_halo, h.data(), sizeof(HaloRankArgs) * nlocal, cudaMemcpyHostToDevice));
    *group_out = (int32_t)(c->peer_groups.size() - 1);
    return EBB_OK;
}

ebb_status ebb_peer_halo_push(ebb_ctx ctx, int32_t group, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c) return EBB_E_ARG;
    if (group < 0 || (size_t)group >= c->peer_groups.size() || !c->peer_groups[group] ||
        !((PeerGroup*)c->peer_groups[group])->d_halo)
        return fail(c, EBB_E_ARG, "halo_push: bad halo group %d", group);
    PeerGroup* P = (PeerGroup*)c->peer_groups[group];
    for (ebb_field f : P->fields)
        if (!get_field(c, f)) return fail(c, EBB_E_STATE, "halo_push: a field of group %d was freed", group);
    if (P->noop) return EBB_OK;        // one rank: nothing to move, no launch
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P->G * (unsigned)P->nlocal);
    cfg.blockDim = dim3(256);
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const HaloRankArgs* recs = P->d_halo;
    unsigned G = P->G;
    unsigned long long* err = c->d_err;
    c->launches++;
    EBB_CUDA(c, cudaLaunchKernelEx(&cfg, k_peer_halo, recs, G, err));
    return EBB_OK;
}

}  // extern "C"
