// chunk_map.cu -- the CHUNK element map ("+=" strategy
// (i) without atomics and without redundant element work): every tet's
// element physics is computed exactly once.
//
// Per tet (P:941-946 Vega StVK, P:975-980 neo-Hookean): gather u[v[k]] through
// the key-field tets.v, element physics (element.cuh), and the
// field reductions f[v[i]] += f_i, K[e[i][j]] += K_ij plus energy +=
// W Psi:
//
//   tiles  tile k = the NT consecutive tets [k NT, (k+1) NT) (the tet order is
//          the renumbered SFC order, so a tile is a compact blob of the mesh).
//          Every canonical edge row (tail <= head; a self row carries its
//          vertex's force too) receives blocks from one or more tiles; its
//          OWNER is the last of them.  A tile sums, per touched row, the
//          blocks of its own tets ("segments", planned once per mesh); a
//          segment of a row owned by a later tile is a MESSAGE: the partial
//          sum goes to a 128-byte slot in global memory (L2), and the owner
//          adds its incoming messages, in tile order, to its own segment and
//          stores the row (and its transpose) exactly once.
//   kernel persistent CTAs (one resident wave) take tiles round-robin
//          (tile = blockIdx + j grid: lockstep rounds); per tile
//            phase 1   thread = tet: element physics -> compact state in smem
//            phase 2a  thread = outgoing segment chunk: sum, write the message;
//                      then one release-increment per receiver tile
//            phase 2b  wait until every sender tile has signalled;
//                      thread = owned segment chunk: sum + incoming messages
//                      (L2 loads), store the K row, its transpose, the force.
//          Messages only flow to LATER tiles and every CTA walks its tiles in
//          increasing order, so with all CTAs resident the lowest unfinished
//          tile never waits: no deadlock.
//   plan   built on the device (CUB radix sorts, scans; chunk_plan below).
// The sums are in plan order (own blocks in (tet, pair) order, then messages
// by sender tile): bitwise run-to-run deterministic.  The oracle computes the
// same quantities by the textbook F-form and a generic 4th-order tensor
// contraction (oracle/ebb_oracle.c); the two share no code.
#include <cub/cub.cuh>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "async_copy.cuh"
#include "ebb_internal.cuh"
#include "element.cuh"
#include "reduce.cuh"
#include "seg_common.cuh"

namespace ebb {
namespace {

constexpr uint32_t kNoTile = 0xFFFFFFFFu;
constexpr int kMsgBytes = 128;   // one message = one L2 line

// item = {meta, row, row2, w}
//   meta  begin[0:13) count[13:18) pos[18:21) last[21:24) kind[24] nmsg[25:32)
//         (begin = first entry of the chunk in the tile's entry list, count <= 31
//          entries, pos / last = chunk index / last chunk index of the segment,
//          kind 1 = self row + vertex force, nmsg = incoming messages <= 127)
//   row   owned: the K row (self row for kind 1); ~0 = padding
//   row2  owned: transpose row (kind 0) or the vertex (kind 1)
//   w     outgoing: the message slot; owned: the first incoming slot
__device__ __forceinline__ uint32_t it_begin(uint32_t m) { return m & 0x1FFFu; }
__device__ __forceinline__ uint32_t it_count(uint32_t m) { return (m >> 13) & 0x1Fu; }
__device__ __forceinline__ uint32_t it_pos(uint32_t m) { return (m >> 18) & 7u; }
__device__ __forceinline__ uint32_t it_last(uint32_t m) { return (m >> 21) & 7u; }
__device__ __forceinline__ uint32_t it_kind(uint32_t m) { return (m >> 24) & 1u; }
__device__ __forceinline__ uint32_t it_nmsg(uint32_t m) { return m >> 25; }

// Signals.  The sender's red.release (MEMBAR.ALL.GPU + RED) orders its CTA's
// message stores (made visible at CTA scope by the preceding bar.sync) before
// the first count; the further receivers' counts follow it in program order
// behind that MEMBAR (one per tile: a release per receiver serializes on the
// RED round trips).  The receiver spins with relaxed gpu-scope loads and reads the
// messages with L2 (.cg, STRONG.GPU) loads after a bar.sync: no acquire fence,
// because on sm_100a ld.acquire / fence.acq_rel add CCTL.IVALL (the whole L1
// invalidated -- the tile's cached gathers with it), measured at 2x the map time.
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// one chunk of a segment: the blocks (kind 0) or diagonal blocks + corner
// forces (kind 1) of its entries, summed in entry order
template <typename R, int MODEL, int NT>
__device__ __forceinline__ void chunk_walk(const R* __restrict__ st, const uint32_t* __restrict__ E, uint32_t meta,
                                           R a9[9]) {
    using G = SegState<MODEL>;
    const uint32_t e0 = it_begin(meta), e1 = e0 + it_count(meta);
    if (it_kind(meta) == 0) {
        uint32_t x = e0 < e1 ? E[e0] : 0u;
#pragma unroll 2
        for (uint32_t e = e0; e < e1; ++e) {
            const uint32_t nx = e + 1 < e1 ? E[e + 1] : 0u;
            seg_block<R, MODEL, NT>(st, x, a9);
            x = nx;
        }
    } else {
        uint32_t x = e0 < e1 ? E[e0] : 0u;
#pragma unroll 2
        for (uint32_t e = e0; e < e1; ++e) {
            const uint32_t nx = e + 1 < e1 ? E[e + 1] : 0u;
            seg_diag<R, MODEL, NT>(st, x, a9);
            const R* sf = st + G::F * NT + (x & 0x1FFFu);   // f_i at the offset of k_i
            a9[6] += sf[0];
            a9[7] += sf[NT];
            a9[8] += sf[2 * NT];
            x = nx;
        }
    }
}

// the chunks of a segment sit in consecutive lanes: shuffle tree into pos 0
template <typename R>
__device__ __forceinline__ void chunk_combine(uint32_t meta, R a9[9]) {
    const uint32_t pos = it_pos(meta), last = it_last(meta);
#pragma unroll
    for (uint32_t step = 1; step < 8; step <<= 1) {
        if (!__any_sync(0xFFFFFFFFu, last >= step)) break;
        const bool take = pos + step <= last;
#pragma unroll
        for (uint32_t q = 0; q < 9; ++q) {
            const R o = __shfl_down_sync(0xFFFFFFFFu, a9[q], step);
            if (take) a9[q] += o;
        }
    }
}

// an owned row's final sum: K row (+ its transpose), or the self row + the force
template <typename R>
__device__ __forceinline__ void chunk_store(uint32_t kind, uint32_t row, uint32_t row2, R a9[9], R* __restrict__ f,
                                            R* __restrict__ K, uint64_t ne, int accumulate) {
    if (kind == 1) {
        R* df = f + 3ull * row2;
#pragma unroll
        for (int a = 0; a < 3; ++a) df[a] = accumulate ? df[a] + a9[6 + a] : a9[6 + a];
        const R dd[6] = {a9[0], a9[1], a9[2], a9[3], a9[4], a9[5]};
        a9[0] = dd[0]; a9[1] = dd[1]; a9[2] = dd[2];
        a9[3] = dd[1]; a9[4] = dd[3]; a9[5] = dd[4];
        a9[6] = dd[2]; a9[7] = dd[4]; a9[8] = dd[5];
    }
    R* dst = K + row;
#pragma unroll
    for (int q = 0; q < 9; ++q, dst += ne) *dst = accumulate ? *dst + a9[q] : a9[q];
    if (kind == 0) {
        dst = K + row2;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int c = 0; c < 3; ++c, dst += ne) *dst = accumulate ? *dst + a9[3 * c + a] : a9[3 * c + a];
    }
}


// RED mode: the same destinations as chunk_store, added with red.global.add
// (the row was zeroed before the map: k_chunk_zero_shared)
template <typename R>
__device__ __forceinline__ void chunk_red(uint32_t kind, uint32_t row, uint32_t row2, R a9[9], R* __restrict__ f,
                                          R* __restrict__ K, uint64_t ne) {
    if (kind == 1) {
        R* df = f + 3ull * row2;
#pragma unroll
        for (int a = 0; a < 3; ++a) atomicAdd(df + a, a9[6 + a]);
        const R dd[6] = {a9[0], a9[1], a9[2], a9[3], a9[4], a9[5]};
        a9[0] = dd[0]; a9[1] = dd[1]; a9[2] = dd[2];
        a9[3] = dd[1]; a9[4] = dd[3]; a9[5] = dd[4];
        a9[6] = dd[2]; a9[7] = dd[4]; a9[8] = dd[5];
    }
    R* dst = K + row;
#pragma unroll
    for (int q = 0; q < 9; ++q, dst += ne) atomicAdd(dst, a9[q]);
    if (kind == 0) {
        dst = K + row2;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int c = 0; c < 3; ++c, dst += ne) atomicAdd(dst, a9[3 * c + a]);
    }
}

#ifdef CHUNK_PROF
__device__ unsigned long long g_chunk_prof[16];
#endif
template <typename R, int NT>
constexpr int chunk_min_blocks() { return NT <= 256 ? 2 : 1; }   // NT <= 128: no register cap

template <typename R, int MODEL, bool WANT_E, int NT, bool RED>
__global__ void __launch_bounds__(NT, chunk_min_blocks<R, NT>()) k_tet_map_chunk(
    uint32_t ntiles, const uint4* __restrict__ tdesc, const uint32_t* __restrict__ expect,
    const uint32_t* __restrict__ recv, uint32_t* __restrict__ cnt, uint32_t* __restrict__ ticket,
    const uint4* __restrict__ items, const uint32_t* __restrict__ ents, R* __restrict__ msg, uint64_t nt,
    const uint4* __restrict__ tv, const R* __restrict__ u, const R* __restrict__ Dminv, const R* __restrict__ Wt,
    const R* __restrict__ mu_t, const R* __restrict__ lam_t, R* __restrict__ f, R* __restrict__ K, uint64_t ne,
    int accumulate, double* __restrict__ tile_e, R* __restrict__ energy, unsigned long long* __restrict__ err) {
    using G = SegState<MODEL>;
    constexpr uint32_t ENT = 10 * NT;               // entries per tile (the last tile is padded)
    constexpr uint32_t MW = kMsgBytes / sizeof(R);  // words per message slot
    extern __shared__ __align__(16) unsigned char chunk_smem[];
    R* st = reinterpret_cast<R*>(chunk_smem);                                 // [SW][NT]
    uint32_t* ebuf = reinterpret_cast<uint32_t*>(st + (size_t)G::SW * NT);    // [2][ENT]
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ double e_w[NT / 32];     // per-warp energy of the current tile
    __shared__ bool am_last;
    const uint32_t tid = threadIdx.x, G0 = gridDim.x;
    // static round-robin schedule: this CTA's tiles are blockIdx + j G0, so all
    // CTAs sweep the tiles in lockstep rounds and a tile's senders (earlier
    // tiles, mostly a few back) run in the same or an earlier round.  Needs
    // every CTA resident (the grid is one occupancy wave): the lowest
    // unfinished tile is then always being processed and never waits.
    // (Dynamic claiming with a ticket counter was measured 8x slower: a sender
    // queued behind another CTA's tile stalls its receivers in convoys.)
    const uint32_t m = blockIdx.x < ntiles ? (ntiles - blockIdx.x + G0 - 1) / G0 : 0;
    auto tile_of = [&](uint32_t j) -> uint32_t { return j < m ? blockIdx.x + j * G0 : kNoTile; };
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto stage = [&](uint32_t tile, int b) {   // thread 0: the tile's entry list -> ebuf[b]
        mbar_arrive_expect_tx(&bar[b], ENT * 4u);
        bulk_g2s(ebuf + (size_t)b * ENT, ents + (size_t)tile * ENT, ENT * 4u, &bar[b]);
    };
    auto keys_of = [&](uint32_t tile) -> uint4 {
        if (tile == kNoTile) return make_uint4(0, 0, 0, 0);
        const uint64_t t = (uint64_t)tile * NT + tid;
        return t < nt ? __ldg(tv + t) : make_uint4(0, 0, 0, 0);
    };
    auto tet_of = [&](uint32_t tile) -> uint32_t {
        if (tile == kNoTile) return 0xFFFFFFFFu;
        const uint64_t t = (uint64_t)tile * NT + tid;
        return t < nt ? (uint32_t)t : 0xFFFFFFFFu;
    };
    // register software pipeline: inputs of the current tile, keys of the next
    uint32_t tc = tile_of(0);
    if (tid == 0 && tc != kNoTile) stage(tc, 0);
    SegIn<R> in;
    seg_load(tet_of(tc), keys_of(tc), nt, u, Dminv, Wt, mu_t, lam_t, in);
    uint4 v1 = keys_of(tile_of(1));
#ifdef CHUNK_PROF
    long long tp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tc0 = clock64();
#define CP_MARK(q)                      \
    do {                                \
        const long long tn_ = clock64(); \
        tp[q] += tn_ - tc0;             \
        tc0 = tn_;                      \
    } while (0)
#else
#define CP_MARK(q) \
    do {           \
    } while (0)
#endif
    for (uint32_t j = 0; j < m; ++j) {
        tc = tile_of(j);
        const uint32_t tn = tile_of(j + 1), tnn = tile_of(j + 2);
        // ---- phase 1: this thread's tet -> compact state
        const uint32_t t = tet_of(tc);
        double et = 0.0;
        if (t != 0xFFFFFFFFu) {
            TetState<R> ts;
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int c = 0; c < 3; ++c) ts.g[r + 1][c] = in.g[r][c];
#pragma unroll
            for (int c = 0; c < 3; ++c) ts.g[0][c] = -(ts.g[1][c] + ts.g[2][c] + ts.g[3][c]);
            ts.W = in.W;
            ts.mu = in.mu;
            ts.lam = in.lam;
            tet_physics<R, MODEL, true>(in.uu, ts);
            if (MODEL == EBB_NH && !(ts.J > R(0))) atomicAdd(&err[ERR_INVERTED], 1ull);
            if (WANT_E) et = (double)(ts.W * ts.psi);
            R fi[4][3];
            tet_forces(ts, fi);
            seg_put_state<R, MODEL, NT>(ts, fi, st + tid);
        }
        if (WANT_E) {   // the tile's energy: fixed shuffle tree + warp order (deterministic)
            et = warp_reduce<ROP_SUM>(et);
            if ((tid & 31) == 0) e_w[tid >> 5] = et;
        }
        // ---- advance the pipeline (these loads land during phase 2)
        seg_load(tet_of(tn), v1, nt, u, Dminv, Wt, mu_t, lam_t, in);
        v1 = keys_of(tnn);
        if (tid == 0 && tn != kNoTile) {
            fence_proxy_async_smem();
            stage(tn, (j + 1) & 1);
        }
        const uint4 d = __ldg(tdesc + tc);   // {item0, outgoing items, owned items, receiver list}
        const uint32_t r1 = __ldg(&tdesc[tc + 1].w);
        CP_MARK(0);
        __syncthreads();   // state complete
        if (WANT_E && tid == 0) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < NT / 32; ++w) s += e_w[w];
            tile_e[tc] = s;
        }
        mbar_wait(&bar[j & 1], (j >> 1) & 1);
        CP_MARK(1);
        const uint32_t* E = ebuf + (size_t)(j & 1) * ENT;
        // ---- phase 2a: outgoing segments -> messages
        for (uint32_t base = 0; base < d.y; base += NT) {
            const uint4 it = base + tid < d.y ? __ldg(items + d.x + base + tid) : make_uint4(0, 0xFFFFFFFFu, 0, 0);
            R a9[9];
#pragma unroll
            for (int q = 0; q < 9; ++q) a9[q] = R(0);
            chunk_walk<R, MODEL, NT>(st, E, it.x, a9);
            chunk_combine<R>(it.x, a9);
            if (it_pos(it.x) == 0 && it.y != 0xFFFFFFFFu) {
                if constexpr (RED) {
                    chunk_red<R>(it_kind(it.x), it.y, it.z, a9, f, K, ne);   // strategy (i): no message
                } else {
                    R* mm = msg + (size_t)it.w * MW;
#pragma unroll
                    for (int q = 0; q < 9; ++q) mm[q] = a9[q];
                }
            }
        }
        if constexpr (!RED) __syncthreads();   // every message of this tile written (CTA scope)
        CP_MARK(2);
        // ---- signal the receivers, wait for the senders
        if (!RED && tid == 0) {
            if (r1 > d.w) {
                red_release_add(cnt + __ldg(recv + d.w), 1u);   // MEMBAR.ALL.GPU once, then the RED
                for (uint32_t r = d.w + 1; r < r1; ++r) atomicAdd(cnt + __ldg(recv + r), 1u);
            }
            const uint32_t need = __ldg(expect + tc);
            if (need) {
                while (ld_relaxed(cnt + tc) < need) {
                }
                cnt[tc] = 0;   // every sender has signalled: reset for the next launch
            }
        }
        CP_MARK(3);
        if constexpr (!RED) __syncthreads();
        CP_MARK(4);
        // ---- phase 2b: owned segments + their incoming messages (L2 loads)
        for (uint32_t base = 0; base < d.z; base += NT) {
            const uint4 it =
                base + tid < d.z ? __ldg(items + d.x + d.y + base + tid) : make_uint4(0, 0xFFFFFFFFu, 0, 0);
            R a9[9];
#pragma unroll
            for (int q = 0; q < 9; ++q) a9[q] = R(0);
            chunk_walk<R, MODEL, NT>(st, E, it.x, a9);
            chunk_combine<R>(it.x, a9);
            if (it_pos(it.x) == 0 && it.y != 0xFFFFFFFFu) {
                const uint32_t nm = it_nmsg(it.x);
                if constexpr (RED) {
                    // a row other tiles also feed: added; a row only this tile feeds: stored
                    if (nm) chunk_red<R>(it_kind(it.x), it.y, it.z, a9, f, K, ne);
                    else chunk_store<R>(it_kind(it.x), it.y, it.z, a9, f, K, ne, accumulate);
                } else {
                    for (uint32_t k = 0; k < nm; ++k) {
                        const R* mm = msg + (size_t)(it.w + k) * MW;
#pragma unroll
                        for (int q = 0; q < 9; ++q) a9[q] += __ldcg(mm + q);
                    }
                    chunk_store<R>(it_kind(it.x), it.y, it.z, a9, f, K, ne, accumulate);
                }
            }
        }
        CP_MARK(5);
        __syncthreads();   // state and entry buffer free for reuse
        CP_MARK(6);
    }
#ifdef CHUNK_PROF
    if (tid == 0 || tid == NT - 1) {
        const int w = tid == 0 ? 0 : 1;
        for (int q = 0; q < 7; ++q) atomicAdd(&g_chunk_prof[8 * w + q], (unsigned long long)tp[q]);
        atomicAdd(&g_chunk_prof[8 * w + 7], 1ull);
    }
#endif
    if (!WANT_E) return;
    // the last CTA out sums the per-tile energies in tile order
    if (tid == 0) {
        __threadfence();
        const uint32_t k = atomicAdd(ticket + 1, 1u);
        am_last = k == gridDim.x - 1;
        if (am_last) ticket[1] = 0;
    }
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    double s = 0.0;
    for (uint32_t k = tid; k < ntiles; k += NT) s += __ldcg(tile_e + k);
    s = block_reduce<ROP_SUM>(s);
    if (tid == 0) *energy = (R)((double)*energy + s);
}

// rows and forces no tet contributes to (isolated vertices): zero unless accumulating
template <typename R>
__global__ void k_chunk_zero(const uint32_t* __restrict__ zrows, uint64_t nz, const uint32_t* __restrict__ zverts,
                             uint64_t nzv, R* __restrict__ K, uint64_t ne, R* __restrict__ f) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < nz)
        for (int q = 0; q < 9; ++q) K[q * ne + zrows[i]] = R(0);
    if (i < nzv)
        for (int a = 0; a < 3; ++a) f[3ull * zverts[i] + a] = R(0);
}

// RED mode: the rows more than one tile feeds (and their transposes / the
// vertex forces of self rows) start from zero -- every contribution is a RED
template <typename R>
__global__ void k_chunk_zero_shared(const uint32_t* __restrict__ srows, uint64_t n, const uint32_t* __restrict__ tval,
                                    R* __restrict__ K, uint64_t ne, R* __restrict__ f) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t r = srows[i], t = tval[2 * i], v = tval[2 * i + 1];
    for (int q = 0; q < 9; ++q) K[q * ne + r] = R(0);
    if (t != r)
        for (int q = 0; q < 9; ++q) K[q * ne + t] = R(0);
    else
        for (int a = 0; a < 3; ++a) f[3ull * v + a] = R(0);
}

// ------------------------------------------------------------------ plan (device)
// contribution (t, p): p < 6 the off-diagonal pair (pair_i, pair_j) -> the
// canonical row (lower vertex first), p >= 6 the diagonal / self row of corner p-6
__device__ __forceinline__ void contrib_row(const uint4 v, const uint32_t* __restrict__ e16, int p, uint32_t& row,
                                            uint32_t& bi, uint32_t& bj) {
    const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
    const int i = pair_i(p), j = pair_j(p);
    bi = vv[i] <= vv[j] ? i : j;
    bj = vv[i] <= vv[j] ? j : i;
    row = e16[4 * bi + bj];
}

__global__ void kp_owner(uint64_t nt, int NT, const uint4* __restrict__ tv, const uint32_t* __restrict__ te,
                         int* __restrict__ owner) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const uint4 v = tv[t];
    const int tile = (int)(t / NT);
    for (int p = 0; p < 10; ++p) {
        uint32_t r, bi, bj;
        contrib_row(v, te + 16 * t, p, r, bi, bj);
        atomicMax(owner + r, tile);
    }
}

// sort key = tile | class | row; class 0 outgoing self, 1 outgoing off-diagonal,
// 2 owned self, 3 owned off-diagonal (the phase order of the kernel)
__global__ void kp_keys(uint64_t nt, int NT, int rbits, const uint4* __restrict__ tv, const uint32_t* __restrict__ te,
                        const int* __restrict__ owner, uint64_t* __restrict__ key, uint32_t* __restrict__ val) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const uint4 v = tv[t];
    const uint64_t tile = t / NT;
    for (int p = 0; p < 10; ++p) {
        uint32_t r, bi, bj;
        contrib_row(v, te + 16 * t, p, r, bi, bj);
        const uint64_t cls = (owner[r] == (int)tile ? 2u : 0u) + (p < 6 ? 1u : 0u);
        key[10 * t + p] = (tile << (rbits + 2)) | (cls << rbits) | r;
        val[10 * t + p] = (uint32_t)(10 * t + p);
    }
}

// entry words in sorted order: oi | oj << 13 | p << 26 (oi, oj = the state word
// offsets of k_i, k_j of the tail-side / head-side corner); padding 0
__global__ void kp_entries(uint64_t nc, uint64_t ncap, int NT, const uint4* __restrict__ tv,
                           const uint32_t* __restrict__ val, uint32_t* __restrict__ ents) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= ncap) return;
    if (i >= nc) {
        ents[i] = 0;
        return;
    }
    const uint32_t c = val[i];
    const uint64_t t = c / 10;
    const int p = (int)(c % 10);
    const uint4 v = tv[t];
    const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
    const int a = pair_i(p), b = pair_j(p);
    const uint32_t bi = vv[a] <= vv[b] ? a : b, bj = vv[a] <= vv[b] ? b : a;
    const uint32_t lr = (uint32_t)(t % NT);
    ents[i] = (3 * bi * NT + lr) | ((3 * bj * NT + lr) << 13) | ((uint32_t)p << 26);
}

// per segment (unique key): tile, class, row; outgoing ones get a (row, tile)
// sort key for the slot order and count into nout[row]; per tile the segment count
__global__ void kp_segs(uint64_t ns, int rbits, const uint64_t* __restrict__ ukey, uint32_t* __restrict__ nout,
                        uint32_t* __restrict__ seg_per_tile, uint64_t* __restrict__ okey, uint32_t* __restrict__ oval,
                        uint32_t* __restrict__ nouts, uint64_t* __restrict__ pair) {
    const uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (s >= ns) return;
    const uint64_t k = ukey[s];
    const uint32_t row = (uint32_t)(k & ((1ull << rbits) - 1)), cls = (uint32_t)((k >> rbits) & 3u);
    const uint32_t tile = (uint32_t)(k >> (rbits + 2));
    atomicAdd(seg_per_tile + tile, 1u);
    if (cls < 2) {
        atomicAdd(nout + row, 1u);
        const uint32_t o = atomicAdd(nouts, 1u);
        okey[o] = ((uint64_t)row << 32) | tile;
        oval[o] = (uint32_t)s;
    }
    (void)pair;
}

// outgoing segment (sorted by (row, tile)) -> its message slot; the (sender,
// receiver) tile pair of each message
__global__ void kp_slots(uint64_t no, const uint64_t* __restrict__ okey_sorted, const uint32_t* __restrict__ oval_sorted,
                         const int* __restrict__ owner, uint32_t* __restrict__ slot_of_seg, uint64_t* __restrict__ pair) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= no) return;
    slot_of_seg[oval_sorted[i]] = (uint32_t)i;
    const uint64_t k = okey_sorted[i];
    const uint32_t row = (uint32_t)(k >> 32), tile = (uint32_t)k;
    pair[i] = ((uint64_t)tile << 32) | (uint32_t)owner[row];
}

__global__ void kp_pairs(uint64_t np, const uint64_t* __restrict__ upair, uint32_t* __restrict__ nrecv,
                         uint32_t* __restrict__ expect) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= np) return;
    atomicAdd(nrecv + (upair[i] >> 32), 1u);
    atomicAdd(expect + (uint32_t)upair[i], 1u);
}

__global__ void kp_recv(uint64_t np, const uint64_t* __restrict__ upair, uint32_t* __restrict__ recv) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= np) return;
    recv[i] = (uint32_t)upair[i];   // pairs sorted by (sender, receiver): CSR by sender
}

// Item layout of one tile (one thread per tile, sequential over its segments in
// key order).  L = entries per chunk (<= 31, <= 8 chunks a segment); chunks of
// a segment never straddle a warp; each of the 4 classes starts a warp.
// count pass (emit = false): per tile the padded outgoing / owned item counts
// and the chosen L; emit pass: the items.
struct SegView {
    const uint64_t* ukey;
    const uint32_t* ucnt;
    const uint64_t* sbeg;        // first contribution of each segment (global position)
    const uint32_t* seg_ptr;     // per tile: first segment
    const uint32_t* slot_of_seg; // outgoing segments
    const uint32_t* mstart;      // per row: first incoming slot
    const uint32_t* nout;        // per row: incoming messages
    const uint32_t* tval;        // per row: transpose row (off-diagonal) or ~0
    const uint32_t* rvert;       // per self row: the vertex
    uint32_t* bad;               // range error flags (1: segment too long, 2: too many messages)
    int rbits, NT;
};

__device__ uint32_t layout_tile(const SegView& S, uint32_t tile, uint32_t L, bool emit, uint4* out, uint32_t* nsec) {
    uint32_t n = 0, sec_out = 0;
    int prev_cls = -1;
    auto pad = [&]() {
        while (n % 32) {
            if (emit) out[n] = make_uint4(0, 0xFFFFFFFFu, 0, 0);
            ++n;
        }
    };
    const uint32_t s0 = S.seg_ptr[tile], s1 = S.seg_ptr[tile + 1];
    const uint64_t tile_e0 = (uint64_t)tile * 10 * S.NT;
    for (uint32_t s = s0; s < s1; ++s) {
        const uint64_t k = S.ukey[s];
        const uint32_t row = (uint32_t)(k & ((1ull << S.rbits) - 1));
        const int cls = (int)((k >> S.rbits) & 3u);
        if (cls != prev_cls) {
            pad();
            if (cls >= 2 && prev_cls < 2) sec_out = n;
            prev_cls = cls;
        }
        const uint32_t cnt = S.ucnt[s];
        const uint32_t nc = (cnt + L - 1) / L;
        if ((n % 32) + nc > 32) pad();
        uint32_t beg = (uint32_t)(S.sbeg[s] - tile_e0);
        const uint32_t kind = (cls & 1) ? 0u : 1u;
        const uint32_t nm = cls >= 2 ? S.nout[row] : 0u;
        const uint32_t row2 = kind ? S.rvert[row] : S.tval[row];
        for (uint32_t cc = 0; cc < nc; ++cc, ++n) {
            const uint32_t sz = cnt / nc + (cc < cnt % nc ? 1 : 0);
            if (emit) {
                uint4 it;
                if (cls < 2) it = make_uint4(0, row, row2, S.slot_of_seg[s]);   // row, row2: the RED mode
                else it = make_uint4(nm << 25, row, row2, S.mstart[row]);
                it.x |= beg | (sz << 13) | (cc << 18) | ((nc - 1) << 21) | (kind << 24);
                out[n] = it;
            }
            beg += sz;
        }
    }
    pad();
    if (prev_cls < 2) sec_out = n;   // no owned segments
    nsec[0] = sec_out;
    nsec[1] = n - sec_out;
    return n;
}

__global__ void kp_layout_count(SegView S, uint32_t ntiles, uint32_t* __restrict__ nitems, uint32_t* __restrict__ tileL,
                                uint32_t* __restrict__ nout_items) {
    const uint32_t tile = blockIdx.x * blockDim.x + threadIdx.x;
    if (tile >= ntiles) return;
    // longest segment and entry total of the tile
    uint32_t longest = 1, tot = 0;
    for (uint32_t s = S.seg_ptr[tile]; s < S.seg_ptr[tile + 1]; ++s) {
        longest = max(longest, S.ucnt[s]);
        tot += S.ucnt[s];
        const uint64_t k = S.ukey[s];
        if (((k >> S.rbits) & 3u) >= 2 && S.nout[(uint32_t)(k & ((1ull << S.rbits) - 1))] > 127) atomicOr(S.bad, 2u);
    }
    if (longest > 8 * 31) atomicOr(S.bad, 1u);
    // L: the smallest chunk (from the even share per thread) whose item list
    // fits the fewest passes of NT threads; at most 8 chunks per segment
    const uint32_t L0 = min(31u, max(max(2u, (tot + S.NT - 1) / S.NT), (longest + 7) / 8));
    uint32_t bestL = L0, bestc = 0xFFFFFFFFu, bo = 0, bn = 0;
    for (uint32_t L = L0; L <= min(31u, max(L0, 4 * L0)); ++L) {
        uint32_t sec[2];
        const uint32_t n = layout_tile(S, tile, L, false, nullptr, sec);
        const uint32_t passes = (sec[0] + S.NT - 1) / S.NT + (sec[1] + S.NT - 1) / S.NT;
        const uint32_t cost = passes * min(L, longest);
        if (cost < bestc) {
            bestc = cost;
            bestL = L;
            bo = sec[0];
            bn = n;
        }
        if (L >= longest) break;
    }
    tileL[tile] = bestL;
    nitems[tile] = bn;
    nout_items[tile] = bo;
}

__global__ void kp_layout_emit(SegView S, uint32_t ntiles, const uint32_t* __restrict__ tileL,
                               const uint32_t* __restrict__ item0, uint4* __restrict__ items) {
    const uint32_t tile = blockIdx.x * blockDim.x + threadIdx.x;
    if (tile >= ntiles) return;
    uint32_t sec[2];
    layout_tile(S, tile, tileL[tile], true, items + item0[tile], sec);
}

__global__ void kp_tdesc(uint32_t ntiles, const uint32_t* __restrict__ item0, const uint32_t* __restrict__ nitems,
                         const uint32_t* __restrict__ nout_items, const uint32_t* __restrict__ recv0,
                         uint4* __restrict__ tdesc) {
    const uint32_t tile = blockIdx.x * blockDim.x + threadIdx.x;
    if (tile > ntiles) return;
    if (tile == ntiles) {
        tdesc[tile] = make_uint4(item0[tile], 0, 0, recv0[tile]);
        return;
    }
    tdesc[tile] = make_uint4(item0[tile], nout_items[tile], nitems[tile] - nout_items[tile], recv0[tile]);
}

// per row: transpose row (off-diagonal; binary search in the head's group) or
// the vertex of a self row; rows without contributions -> zero list
__global__ void kp_rowinfo(uint64_t nv, const uint32_t* __restrict__ index, const uint32_t* __restrict__ head,
                           const int* __restrict__ owner, uint32_t* __restrict__ tval, uint32_t* __restrict__ rvert,
                           uint32_t* __restrict__ zrows, uint32_t* __restrict__ nz, uint32_t* __restrict__ zverts,
                           uint32_t* __restrict__ nzv) {
    const uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (v >= nv) return;
    for (uint32_t r = index[v]; r < index[v + 1]; ++r) {
        const uint32_t h = head[r];
        rvert[r] = (uint32_t)v;
        if (h == v) {
            tval[r] = r;
            if (owner[r] < 0) zverts[atomicAdd(nzv, 1u)] = (uint32_t)v;
        } else {
            uint32_t lo = index[h], hi = index[h + 1];
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (head[mid] < v) lo = mid + 1;
                else hi = mid;
            }
            tval[r] = lo;
        }
        // a transposed row (head < tail) is written with its canonical row
        if (owner[h >= v ? r : tval[r]] < 0) zrows[atomicAdd(nz, 1u)] = r;
    }
}

// rows with incoming messages (fed by more than one tile): (row) and (transpose or self, vertex)
__global__ void kp_shared_rows(uint64_t ne, const uint32_t* __restrict__ nout, const uint32_t* __restrict__ tval,
                               const uint32_t* __restrict__ rvert, uint32_t* __restrict__ srows,
                               uint32_t* __restrict__ sinfo, uint32_t* __restrict__ ns) {
    const uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (r >= ne || nout[r] == 0) return;
    const uint32_t k = atomicAdd(ns, 1u);
    srows[k] = (uint32_t)r;
    sinfo[2 * k] = tval[r];
    sinfo[2 * k + 1] = rvert[r];
}

int bits_for(uint64_t n) {
    int b = 1;
    while ((1ull << b) < n) ++b;
    return b;
}

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() { cudaFree(p); }
    cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes + 16); }
    template <typename T>
    T* as() const { return (T*)p; }
};

}  // namespace

void ChunkPlan::release() {
    cudaFree(tdesc); cudaFree(expect); cudaFree(recv); cudaFree(cnt); cudaFree(ticket);
    cudaFree(items); cudaFree(ents); cudaFree(msg); cudaFree(zrows); cudaFree(zverts); cudaFree(tile_e);
    cudaFree(srows);
    tdesc = nullptr; items = nullptr; tile_e = nullptr;
    expect = recv = cnt = ticket = ents = zrows = zverts = srows = nullptr;
    msg = nullptr;
}

ebb_status build_chunk_plan(Ctx* c, ebb_field vf, ebb_field ef, int NT, ChunkPlan** out) {
    for (ChunkPlan* P : c->chunkplans)
        if (P->v == vf && P->e == ef && P->nt_tile == NT) {
            *out = P;
            return EBB_OK;
        }
    const auto t_start = std::chrono::steady_clock::now();
    Field* V = get_field(c, vf);
    Field* Ef = get_field(c, ef);
    Relation& ER = c->rels[Ef->key_target];
    if (ER.grouped_by == EBB_NONE || ER.index == EBB_NONE)
        return fail(c, EBB_E_STATE, "chunk map: the edge relation must be grouped by tail");
    ebb_field hf = EBB_NONE;
    for (ebb_field fh : ER.fields)
        if (c->fields[fh].alive && c->fields[fh].name == "head") hf = fh;
    if (hf == EBB_NONE) return fail(c, EBB_E_STATE, "chunk map: edge relation has no 'head' key-field");
    const uint64_t nt = c->rels[V->rel].size, nv = c->rels[V->key_target].size, ne = ER.size;
    if (nt * 10 >= (1ull << 32)) return fail(c, EBB_E_RANGE, "chunk map: more than 429M tets");
    const uint32_t ntiles = (uint32_t)((nt + NT - 1) / NT);
    const int rbits = bits_for(ne + 1), tbits = bits_for(ntiles + 1);
    const uint64_t nc = nt * 10, ncap = (uint64_t)ntiles * 10 * NT;
    const uint4* tv = (const uint4*)V->ptr;
    const uint32_t* te = (const uint32_t*)Ef->ptr;
    const uint32_t* index = (const uint32_t*)c->fields[ER.index].ptr;
    const uint32_t* head = (const uint32_t*)c->fields[hf].ptr;
    cudaStream_t s = 0;
    const unsigned B = 256;
    ChunkPlan* P = new ChunkPlan();
    P->v = vf;
    P->e = ef;
    P->nt_tile = NT;
    P->ntiles = ntiles;
    auto bail = [&](ebb_status st) {
        P->release();
        delete P;
        return st;
    };
#define CP_CUDA(call)                                                           \
    do {                                                                        \
        cudaError_t _e = (call);                                                \
        if (_e != cudaSuccess) return bail(::ebb::cuda_fail(c, _e, #call));     \
    } while (0)
    // 1. owner tile of every row (-1: no contribution)
    DevBuf owner;
    CP_CUDA(owner.alloc(ne * 4));
    CP_CUDA(cudaMemsetAsync(owner.p, 0xFF, ne * 4, s));
    if (nt) kp_owner<<<grid_for(nt, B), B, 0, s>>>(nt, NT, tv, te, owner.as<int>());
    // 2. contributions sorted by (tile, class, row), stable in (tet, pair)
    DevBuf key, key2, val, val2, tmp;
    CP_CUDA(key.alloc(nc * 8));
    CP_CUDA(key2.alloc(nc * 8));
    CP_CUDA(val.alloc(nc * 4));
    CP_CUDA(val2.alloc(nc * 4));
    if (nt) kp_keys<<<grid_for(nt, B), B, 0, s>>>(nt, NT, rbits, tv, te, owner.as<int>(), key.as<uint64_t>(),
                                                  val.as<uint32_t>());
    size_t tb = 0;
    const int kbits = rbits + 2 + tbits;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, key.as<uint64_t>(), key2.as<uint64_t>(), val.as<uint32_t>(),
                                    val2.as<uint32_t>(), (int64_t)nc, 0, kbits, s);
    size_t tb_rle = 0, tb_scan = 0;
    cub::DeviceRunLengthEncode::Encode(nullptr, tb_rle, key2.as<uint64_t>(), key.as<uint64_t>(), val.as<uint32_t>(),
                                       (uint32_t*)nullptr, (int64_t)nc, s);
    cub::DeviceScan::ExclusiveSum(nullptr, tb_scan, (uint32_t*)nullptr, (uint64_t*)nullptr, (int64_t)nc, s);
    CP_CUDA(tmp.alloc(std::max(tb, std::max(tb_rle, tb_scan))));
    CP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.as<uint64_t>(), key2.as<uint64_t>(), val.as<uint32_t>(),
                                            val2.as<uint32_t>(), (int64_t)nc, 0, kbits, s));
    // entries (sorted order = per tile contiguous, 10 NT per tile)
    CP_CUDA(cudaMalloc(&P->ents, ncap * 4 + 16));
    if (ncap) kp_entries<<<grid_for(ncap, B), B, 0, s>>>(nc, ncap, NT, tv, val2.as<uint32_t>(), P->ents);
    // 3. segments = runs of equal keys (reuse key / val as the unique keys / counts)
    DevBuf nseg_d;
    CP_CUDA(nseg_d.alloc(8));
    CP_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.p, tb_rle, key2.as<uint64_t>(), key.as<uint64_t>(),
                                               val.as<uint32_t>(), nseg_d.as<uint32_t>(), (int64_t)nc, s));
    uint32_t ns = 0;
    CP_CUDA(cudaMemcpyAsync(&ns, nseg_d.p, 4, cudaMemcpyDeviceToHost, s));
    CP_CUDA(cudaStreamSynchronize(s));
    const uint64_t* ukey = key.as<uint64_t>();
    const uint32_t* ucnt = val.as<uint32_t>();
    DevBuf sbeg;
    CP_CUDA(sbeg.alloc((uint64_t)ns * 8));
    CP_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb_scan, ucnt, sbeg.as<uint64_t>(), (int64_t)ns, s));
    // 4. per-segment bookkeeping: outgoing segments, incoming counts per row
    DevBuf nout, seg_per_tile, okey, okey2, oval, oval2, nouts;
    CP_CUDA(nout.alloc((ne + 1) * 4));
    CP_CUDA(seg_per_tile.alloc((ntiles + 1) * 4));
    CP_CUDA(okey.alloc((uint64_t)ns * 8));
    CP_CUDA(okey2.alloc((uint64_t)ns * 8));
    CP_CUDA(oval.alloc((uint64_t)ns * 4));
    CP_CUDA(oval2.alloc((uint64_t)ns * 4));
    CP_CUDA(nouts.alloc(4));
    CP_CUDA(cudaMemsetAsync(nout.p, 0, (ne + 1) * 4, s));
    CP_CUDA(cudaMemsetAsync(seg_per_tile.p, 0, (ntiles + 1) * 4, s));
    CP_CUDA(cudaMemsetAsync(nouts.p, 0, 4, s));
    if (ns) kp_segs<<<grid_for(ns, B), B, 0, s>>>(ns, rbits, ukey, nout.as<uint32_t>(), seg_per_tile.as<uint32_t>(),
                                                  okey.as<uint64_t>(), oval.as<uint32_t>(), nouts.as<uint32_t>(),
                                                  nullptr);
    uint32_t no = 0;
    CP_CUDA(cudaMemcpyAsync(&no, nouts.p, 4, cudaMemcpyDeviceToHost, s));
    CP_CUDA(cudaStreamSynchronize(s));
    // slots of outgoing segments in (row, tile) order
    size_t tb2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb2, okey.as<uint64_t>(), okey2.as<uint64_t>(), oval.as<uint32_t>(),
                                    oval2.as<uint32_t>(), (int64_t)no, 0, 32 + rbits, s);
    DevBuf tmp2, slot_of_seg, pair, pair2, upair, npair_d;
    CP_CUDA(tmp2.alloc(tb2));
    CP_CUDA(slot_of_seg.alloc((uint64_t)ns * 4));
    CP_CUDA(pair.alloc((uint64_t)no * 8));
    CP_CUDA(pair2.alloc((uint64_t)no * 8));
    CP_CUDA(upair.alloc((uint64_t)no * 8));
    CP_CUDA(npair_d.alloc(8));
    if (no) {
        CP_CUDA(cub::DeviceRadixSort::SortPairs(tmp2.p, tb2, okey.as<uint64_t>(), okey2.as<uint64_t>(),
                                                oval.as<uint32_t>(), oval2.as<uint32_t>(), (int64_t)no, 0, 32 + rbits,
                                                s));
        kp_slots<<<grid_for(no, B), B, 0, s>>>(no, okey2.as<uint64_t>(), oval2.as<uint32_t>(), owner.as<int>(),
                                               slot_of_seg.as<uint32_t>(), pair.as<uint64_t>());
    }
    // per row: first incoming slot (exclusive scan of nout over rows)
    DevBuf mstart, seg_ptr;
    CP_CUDA(mstart.alloc((ne + 1) * 4));
    CP_CUDA(seg_ptr.alloc((ntiles + 1) * 4));
    size_t tb3 = 0, tb4 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb3, nout.as<uint32_t>(), mstart.as<uint32_t>(), (int64_t)(ne + 1), s);
    cub::DeviceScan::ExclusiveSum(nullptr, tb4, seg_per_tile.as<uint32_t>(), seg_ptr.as<uint32_t>(),
                                  (int64_t)(ntiles + 1), s);
    DevBuf tmp3;
    CP_CUDA(tmp3.alloc(std::max(tb3, tb4)));
    CP_CUDA(cub::DeviceScan::ExclusiveSum(tmp3.p, tb3, nout.as<uint32_t>(), mstart.as<uint32_t>(), (int64_t)(ne + 1),
                                          s));
    CP_CUDA(cub::DeviceScan::ExclusiveSum(tmp3.p, tb4, seg_per_tile.as<uint32_t>(), seg_ptr.as<uint32_t>(),
                                          (int64_t)(ntiles + 1), s));
    // 5. (sender, receiver) tile pairs: unique, CSR by sender; expected counts
    uint32_t np = 0;
    DevBuf nrecv, recv0;
    CP_CUDA(nrecv.alloc((ntiles + 1) * 4));
    CP_CUDA(recv0.alloc((ntiles + 1) * 4));
    CP_CUDA(cudaMalloc(&P->expect, (ntiles + 1) * 4));
    CP_CUDA(cudaMemsetAsync(nrecv.p, 0, (ntiles + 1) * 4, s));
    CP_CUDA(cudaMemsetAsync(P->expect, 0, (ntiles + 1) * 4, s));
    if (no) {
        size_t tb5 = 0, tb6 = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tb5, pair.as<uint64_t>(), pair2.as<uint64_t>(), (int64_t)no, 0,
                                       32 + tbits, s);
        cub::DeviceSelect::Unique(nullptr, tb6, pair2.as<uint64_t>(), upair.as<uint64_t>(), npair_d.as<uint32_t>(),
                                  (int64_t)no, s);
        DevBuf tmp5;
        CP_CUDA(tmp5.alloc(std::max(tb5, tb6)));
        CP_CUDA(cub::DeviceRadixSort::SortKeys(tmp5.p, tb5, pair.as<uint64_t>(), pair2.as<uint64_t>(), (int64_t)no, 0,
                                               32 + tbits, s));
        CP_CUDA(cub::DeviceSelect::Unique(tmp5.p, tb6, pair2.as<uint64_t>(), upair.as<uint64_t>(),
                                          npair_d.as<uint32_t>(), (int64_t)no, s));
        CP_CUDA(cudaMemcpyAsync(&np, npair_d.p, 4, cudaMemcpyDeviceToHost, s));
        CP_CUDA(cudaStreamSynchronize(s));
        kp_pairs<<<grid_for(np, B), B, 0, s>>>(np, upair.as<uint64_t>(), nrecv.as<uint32_t>(), P->expect);
    }
    CP_CUDA(cudaMalloc(&P->recv, (uint64_t)np * 4 + 16));
    if (np) kp_recv<<<grid_for(np, B), B, 0, s>>>(np, upair.as<uint64_t>(), P->recv);
    {
        size_t tb7 = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb7, nrecv.as<uint32_t>(), recv0.as<uint32_t>(), (int64_t)(ntiles + 1),
                                      s);
        DevBuf tmp7;
        CP_CUDA(tmp7.alloc(tb7));
        CP_CUDA(cub::DeviceScan::ExclusiveSum(tmp7.p, tb7, nrecv.as<uint32_t>(), recv0.as<uint32_t>(),
                                              (int64_t)(ntiles + 1), s));
    }
    // 6. row info (transposes, self-row vertices, zero lists)
    DevBuf tval, rvert, zcnt;
    CP_CUDA(tval.alloc(ne * 4));
    CP_CUDA(rvert.alloc(ne * 4));
    CP_CUDA(zcnt.alloc(12));
    CP_CUDA(cudaMalloc(&P->zrows, ne * 4 + 16));
    CP_CUDA(cudaMalloc(&P->zverts, nv * 4 + 16));
    CP_CUDA(cudaMemsetAsync(zcnt.p, 0, 12, s));
    if (nv) kp_rowinfo<<<grid_for(nv, B), B, 0, s>>>(nv, index, head, owner.as<int>(), tval.as<uint32_t>(),
                                                     rvert.as<uint32_t>(), P->zrows, zcnt.as<uint32_t>(), P->zverts,
                                                     zcnt.as<uint32_t>() + 1);
    // 6b. rows fed by several tiles (the RED mode zeroes them first): the row
    // list, then (transpose or self, vertex) per entry, in one allocation
    DevBuf nsr;
    CP_CUDA(nsr.alloc(4));
    CP_CUDA(cudaMemsetAsync(nsr.p, 0, 4, s));
    CP_CUDA(cudaMalloc(&P->srows, ne * 12 + 16));
    if (ne) kp_shared_rows<<<grid_for(ne, B), B, 0, s>>>(ne, nout.as<uint32_t>(), tval.as<uint32_t>(),
                                                         rvert.as<uint32_t>(), P->srows, P->srows + ne,
                                                         nsr.as<uint32_t>());
    // 7. item layout per tile
    SegView S;
    S.ukey = ukey;
    S.ucnt = ucnt;
    S.sbeg = sbeg.as<uint64_t>();
    S.seg_ptr = seg_ptr.as<uint32_t>();
    S.slot_of_seg = slot_of_seg.as<uint32_t>();
    S.mstart = mstart.as<uint32_t>();
    S.nout = nout.as<uint32_t>();
    S.tval = tval.as<uint32_t>();
    S.rvert = rvert.as<uint32_t>();
    S.rbits = rbits;
    S.NT = NT;
    S.bad = zcnt.as<uint32_t>() + 2;
    DevBuf nitems, tileL, nout_items, item0;
    CP_CUDA(nitems.alloc((ntiles + 1) * 4));
    CP_CUDA(tileL.alloc((ntiles + 1) * 4));
    CP_CUDA(nout_items.alloc((ntiles + 1) * 4));
    CP_CUDA(item0.alloc((ntiles + 1) * 4));
    CP_CUDA(cudaMemsetAsync(nitems.p, 0, (ntiles + 1) * 4, s));
    if (ntiles) kp_layout_count<<<grid_for(ntiles, 64), 64, 0, s>>>(S, ntiles, nitems.as<uint32_t>(),
                                                                    tileL.as<uint32_t>(), nout_items.as<uint32_t>());
    {
        size_t tb8 = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb8, nitems.as<uint32_t>(), item0.as<uint32_t>(), (int64_t)(ntiles + 1),
                                      s);
        DevBuf tmp8;
        CP_CUDA(tmp8.alloc(tb8));
        CP_CUDA(cub::DeviceScan::ExclusiveSum(tmp8.p, tb8, nitems.as<uint32_t>(), item0.as<uint32_t>(),
                                              (int64_t)(ntiles + 1), s));
    }
    uint32_t nit = 0, zc[3] = {0, 0, 0}, nsr_h = 0;
    CP_CUDA(cudaMemcpyAsync(&nsr_h, nsr.p, 4, cudaMemcpyDeviceToHost, s));
    CP_CUDA(cudaMemcpyAsync(&nit, item0.as<uint32_t>() + ntiles, 4, cudaMemcpyDeviceToHost, s));
    CP_CUDA(cudaMemcpyAsync(zc, zcnt.p, 12, cudaMemcpyDeviceToHost, s));
    CP_CUDA(cudaStreamSynchronize(s));
    if (zc[2] & 1u) return bail(fail(c, EBB_E_RANGE, "chunk map: a row gets > 248 blocks from one tile"));
    if (zc[2] & 2u) return bail(fail(c, EBB_E_RANGE, "chunk map: a row gets blocks from > 128 tiles"));
    CP_CUDA(cudaMalloc(&P->items, (uint64_t)nit * 16 + 16));
    if (ntiles) kp_layout_emit<<<grid_for(ntiles, 64), 64, 0, s>>>(S, ntiles, tileL.as<uint32_t>(),
                                                                   item0.as<uint32_t>(), P->items);
    CP_CUDA(cudaMalloc(&P->tdesc, (uint64_t)(ntiles + 1) * 16));
    kp_tdesc<<<grid_for(ntiles + 1, B), B, 0, s>>>(ntiles, item0.as<uint32_t>(), nitems.as<uint32_t>(),
                                                   nout_items.as<uint32_t>(), recv0.as<uint32_t>(), P->tdesc);
    // 8. message slots, arrival counters, ticket
    CP_CUDA(cudaMalloc(&P->msg, (uint64_t)no * kMsgBytes + kMsgBytes));
    CP_CUDA(cudaMalloc(&P->cnt, (ntiles + 1) * 4));
    CP_CUDA(cudaMemsetAsync(P->cnt, 0, (ntiles + 1) * 4, s));
    CP_CUDA(cudaMalloc(&P->ticket, 16));
    CP_CUDA(cudaMalloc(&P->tile_e, (uint64_t)(ntiles + 1) * 8));
    CP_CUDA(cudaMemsetAsync(P->ticket, 0, 16, s));
    CP_CUDA(cudaStreamSynchronize(s));
    CP_CUDA(cudaGetLastError());
#undef CP_CUDA
    P->nseg = ns;
    P->nmsg = no;
    P->npair = np;
    P->nitems = nit;
    P->nzrows = zc[0];
    P->nzverts = zc[1];
    P->nsrows = nsr_h;
    P->build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    c->chunkplans.push_back(P);
    *out = P;
    return EBB_OK;
}

namespace {

template <typename R, int MODEL, int NT, bool RED>
ebb_status launch_chunk_t(Ctx* c, const ChunkPlan& P, bool want_e, int accumulate, uint64_t nt, const Field* V,
                          const Field* U, const Field* D, const Field* W, const Field* MU, const Field* LA,
                          const Field* Fo, const Field* Ko, uint64_t ne, const Field* En, cudaStream_t s) {
    const size_t smem = (size_t)SegState<MODEL>::SW * NT * sizeof(R) + 2ull * 10 * NT * 4;
    if (smem > 227 * 1024)
        return fail(c, EBB_E_RANGE, "chunk map: %zu B of shared memory needed (> 227 KB)", smem);
    KernelTimer kt(c, EBB_K_TET_MAP, s);   // the whole map: the zero passes included
    if (!accumulate && (P.nzrows || P.nzverts)) {
        const uint64_t n = std::max(P.nzrows, P.nzverts);
        k_chunk_zero<R><<<grid_for(n, 256), 256, 0, s>>>(P.zrows, P.nzrows, P.zverts, P.nzverts, (R*)Ko->ptr, ne,
                                                          (R*)Fo->ptr);
        EBB_CUDA(c, cudaGetLastError());
        c->launches++;
    }
    if (RED && !accumulate && P.nsrows) {
        // the srows allocation holds the rows (ne entries) then (tval, vertex) pairs
        k_chunk_zero_shared<R><<<grid_for(P.nsrows, 256), 256, 0, s>>>(P.srows, P.nsrows, P.srows + ne, (R*)Ko->ptr,
                                                                       ne, (R*)Fo->ptr);
        EBB_CUDA(c, cudaGetLastError());
        c->launches++;
    }
    if (P.ntiles == 0) return EBB_OK;
    auto kern = want_e ? k_tet_map_chunk<R, MODEL, true, NT, RED> : k_tet_map_chunk<R, MODEL, false, NT, RED>;
    static thread_local size_t configured_dev[kMaxDevices][2] = {};
    size_t* const configured = configured_dev[c->device % kMaxDevices];
    if (smem > configured[want_e]) {
        EBB_CUDA(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured[want_e] = smem;
    }
    unsigned grid = occ_grid(c, kern, NT, smem, (uint64_t)P.ntiles * NT);
    const char* eg = getenv("EBB_CHUNK_GRID");   // test knob: fewer CTAs
    if (eg && atoi(eg) > 0 && (unsigned)atoi(eg) < grid) grid = (unsigned)atoi(eg);
    kern<<<grid, NT, smem, s>>>(P.ntiles, P.tdesc, P.expect, P.recv, P.cnt, P.ticket, P.items, P.ents, (R*)P.msg, nt,
                                (const uint4*)V->ptr, (const R*)U->ptr, (const R*)D->ptr, (const R*)W->ptr,
                                (const R*)MU->ptr, (const R*)LA->ptr, (R*)Fo->ptr, (R*)Ko->ptr, ne, accumulate,
                                P.tile_e, En ? (R*)En->ptr : nullptr, c->d_err);
    EBB_CUDA(c, cudaGetLastError());
#ifdef CHUNK_PROF
    {
        unsigned long long h[16];
        cudaDeviceSynchronize();
        cudaMemcpyFromSymbol(h, g_chunk_prof, sizeof(h));
        const unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(g_chunk_prof, z, sizeof(z));
        for (int w = 0; w < 2; ++w) {
            double tot = 0;
            for (int q = 0; q < 7; ++q) tot += (double)h[8 * w + q];
            fprintf(stderr, "CHUNK_PROF %s: p1 %.1f%% bar+ent %.1f%% 2a+bar %.1f%% signal+wait %.1f%% bar %.1f%% 2c+2b %.1f%% bar %.1f%% (ctas %llu, Mcyc/cta %.3f)\n",
                    w ? "last" : "t0", 100 * h[8 * w] / tot, 100 * h[8 * w + 1] / tot, 100 * h[8 * w + 2] / tot,
                    100 * h[8 * w + 3] / tot, 100 * h[8 * w + 4] / tot, 100 * h[8 * w + 5] / tot,
                    100 * h[8 * w + 6] / tot, h[8 * w + 7], tot / h[8 * w + 7] / 1e6);
        }
    }
#endif
    return EBB_OK;
}

}  // namespace

// tets per tile = threads per CTA (the compact state must fit in shared memory
// next to two entry buffers)
int chunk_threads(ebb_dtype dt, int model) {
    const char* e = getenv("EBB_CHUNK_NT");
    const int ev = e ? atoi(e) : 0;
    int v = (dt == EBB_F64 && model == EBB_STVK) ? 384 : 256;
    if (ev == 128 || ev == 256 || ev == 384 || ev == 512) v = ev;
    if (dt == EBB_F64 && model == EBB_STVK && v > 384) v = 384;
    return v;
}

ebb_status chunk_plan_probe(Ctx* c, ebb_field vf, ebb_field ef, ebb_dtype dt, int model) {
    ChunkPlan* P;
    return build_chunk_plan(c, vf, ef, chunk_threads(dt, model), &P);
}

ebb_status chunk_map_launch(Ctx* c, ebb_field vf, ebb_field ef, int model, bool want_e, int accumulate, uint64_t nt,
                            const Field* V, const Field* U, const Field* D, const Field* W, const Field* MU,
                            const Field* LA, const Field* Fo, const Field* Ko, uint64_t ne, const Field* En,
                            cudaStream_t s, bool red) {
    const ebb_dtype dt = U->dtype;
    const int NT = chunk_threads(dt, model);
    ChunkPlan* P;
    EBB_TRY(build_chunk_plan(c, vf, ef, NT, &P));
#define EBB_CARGS c, *P, want_e, accumulate, nt, V, U, D, W, MU, LA, Fo, Ko, ne, En, s
#define EBB_CDISPATCH2(R, MODEL, RD)                                        \
    do {                                                                    \
        if (NT == 128) return launch_chunk_t<R, MODEL, 128, RD>(EBB_CARGS); \
        if (NT == 256) return launch_chunk_t<R, MODEL, 256, RD>(EBB_CARGS); \
        if (NT == 384) return launch_chunk_t<R, MODEL, 384, RD>(EBB_CARGS); \
        if constexpr (!(sizeof(R) == 8 && MODEL == EBB_STVK))               \
            return launch_chunk_t<R, MODEL, 512, RD>(EBB_CARGS);            \
        return fail(c, EBB_E_ARG, "chunk map: bad thread count %d", NT);   \
    } while (0)
#define EBB_CDISPATCH(R, MODEL)                  \
    do {                                         \
        if (red) EBB_CDISPATCH2(R, MODEL, true); \
        EBB_CDISPATCH2(R, MODEL, false);         \
    } while (0)
    if (dt == EBB_F64) {
        if (model == EBB_NH) EBB_CDISPATCH(double, EBB_NH);
        EBB_CDISPATCH(double, EBB_STVK);
    }
    if (model == EBB_NH) EBB_CDISPATCH(float, EBB_NH);
    EBB_CDISPATCH(float, EBB_STVK);
#undef EBB_CDISPATCH
#undef EBB_CDISPATCH2
#undef EBB_CARGS
}

}  // namespace ebb

extern "C" ebb_status ebb_map_chunk_stats(ebb_ctx ctx, ebb_field v, ebb_field e, double out[8]) {
    using namespace ebb;
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !out) return EBB_E_ARG;
    for (int k = 0; k < 8; ++k) out[k] = 0;
    Field* V = get_field(c, v);
    if (!V) return fail(c, EBB_E_ARG, "map_chunk_stats: bad field handle");
    const double nt = (double)c->rels[V->rel].size;
    for (ChunkPlan* P : c->chunkplans)
        if (P->v == v && P->e == e) {
            out[0] = P->ntiles;
            out[1] = P->nt_tile;
            out[2] = (double)P->nseg;
            out[3] = (double)P->nmsg;
            out[4] = (double)P->nitems;
            out[5] = P->build_ms;
            const double bytes = 40.0 * P->ntiles * P->nt_tile + 16.0 * P->nitems + 16.0 * (P->ntiles + 1) +
                                 (double)kMsgBytes * P->nmsg + 4.0 * P->npair + 8.0 * (P->ntiles + 1) +
                                 4.0 * (P->nzrows + P->nzverts) + 12.0 * (P->ntiles + 1);
            out[6] = nt > 0 ? bytes / nt : 0;
            out[7] = (double)P->nzrows;
        }
    return EBB_OK;
}
