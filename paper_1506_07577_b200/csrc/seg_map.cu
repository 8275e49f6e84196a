// seg_map.cu -- the SEGMENTED element map ("+=" strategy
// (iii): per-tet compact stiffness state, then a per-edge-row segmented sum of
// the K_ij rebuilt from the states of the row's contributing (tet, i, j)).
//
// Per tet (P:941-946 Vega StVK, P:975-980 neo-Hookean): gather u[v[k]] through
// the key-field tets.v, element physics (element.cuh: displacement
// form + closed rank-1 stiffness), and the field reductions f[v[i]] += f_i,
// K[e[i][j]] += K_ij plus energy += W Psi -- without atomics:
//
//   plan (host, once per mesh)  vertex tiles = runs of consecutive SFC-ordered
//        vertices grown until the tets touching them ("instances") reach NT;
//        a tile owns the canonical rows (tail <= head) of its vertices and
//        their forces.  Per owned row the list of (instance, i, j) blocks that
//        add into it; a self row's list is exactly its vertex's (instance,
//        corner) list, so the same walk also sums the vertex's force.
//   kernel (persistent CTA of NT threads, one tile per pass)
//        phase 1  thread = instance: element physics, compact state -> smem
//                 (NH: k_i = F^-T g_i, W mu m_ij, W c1, W lam, f_i;
//                  StVK: h_i = F g_i, W s_ij, W mu m_ij, F F^T, W mu, W lam, f_i);
//                 then the loads of the next tile's instance inputs are issued
//                 (they land during phase 2: a register software pipeline)
//        phase 2  thread = owned row: walk its entries (staged in smem by a
//                 bulk async copy issued one tile ahead), rebuild each 3x3
//                 block from the state, sum in registers, store the row and its
//                 transpose once (self rows: the symmetric 6 + the force).
// Every K row and f row is written exactly once (plain stores, no zero-fill),
// in a fixed order: bitwise run-to-run deterministic.  The oracle computes the
// same quantities by the textbook F-form and a generic 4th-order tensor
// contraction (oracle/ebb_oracle.c); the two share no code.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "async_copy.cuh"
#include "ebb_internal.cuh"
#include "element.cuh"
#include "reduce.cuh"
#include "seg_common.cuh"

namespace ebb {
namespace {

// CTAs per SM at NT = 256: two CTAs overlap one's barrier tail with the
// other's work; fp32 state leaves room for a third (fp64 would spill) -- measured
#ifndef SEG_F32_MINB
#define SEG_F32_MINB 3
#endif
// inputs of the next tile's instance held in registers across phase 2: fp64
// (StVK 12 % faster with it, NH neutral); fp32 loads them at phase-1 start
// (2-4 % faster: 72 instead of 80 registers) -- measured
#ifndef SEG_UNROLL
#define SEG_UNROLL 2    // phase-2 entry walk unroll (measured)
#endif
constexpr int kSegUnroll = SEG_UNROLL;
#ifndef SEG_PIPE_INPUTS
#define SEG_PIPE_INPUTS (sizeof(R) == 8)
#endif
template <typename R, int NT>
constexpr int seg_min_blocks() { return NT <= 128 ? (sizeof(R) == 4 ? 6 : 4) : NT <= 256 ? (sizeof(R) == 4 ? SEG_F32_MINB : 2) : 1; }
#ifdef SEG_PROF
__device__ unsigned long long g_seg_prof[16];
#endif
template <typename R, int MODEL, bool WANT_E, int NT>
__global__ void __launch_bounds__(NT, seg_min_blocks<R, NT>()) k_tet_map_seg(
    uint32_t ntiles, uint32_t run, const uint4* __restrict__ tdesc, const uint2* __restrict__ inst,
    const uint4* __restrict__ items, const uint32_t* __restrict__ ents, uint32_t max_ent, uint64_t nt,
    const uint4* __restrict__ tv, const R* __restrict__ u, const R* __restrict__ Dminv, const R* __restrict__ Wt,
    const R* __restrict__ mu_t, const R* __restrict__ lam_t, R* __restrict__ f, R* __restrict__ K, uint64_t ne,
    int accumulate, double* __restrict__ partials, unsigned int* __restrict__ counter, R* __restrict__ energy,
    unsigned long long* __restrict__ err) {
    using G = SegState<MODEL>;
    extern __shared__ __align__(16) unsigned char seg_smem[];
    R* st = reinterpret_cast<R*>(seg_smem);                                // [SW][NT]
    uint32_t* ebuf = reinterpret_cast<uint32_t*>(st + (size_t)G::SW * NT);  // [2][max_ent]
    __shared__ __align__(16) uint4 dring[64][2];   // descriptors {v0, inst0, item0, ent0} of local tile j
                                                   // and of its successor (= its ends), slot j & 63
    __shared__ __align__(8) uint64_t bar[2];       // entry buffers 0/1
    const uint32_t tid = threadIdx.x, G0 = gridDim.x;
    // this CTA's tiles: the runs (of `run` consecutive tiles) blockIdx.x + r G0
    // -- all CTAs sweep the SFC order together, so the tets and rows shared by
    // neighbouring runs meet in L2; inside a run the state of the tets shared
    // by consecutive tiles stays in shared memory (the plan keeps their slots)
    const uint32_t nruns = (ntiles + run - 1) / run;
    const uint32_t myruns = blockIdx.x < nruns ? (nruns - blockIdx.x + G0 - 1) / G0 : 0;
    const uint32_t lastrun = myruns ? blockIdx.x + (myruns - 1) * G0 : 0;
    const uint32_t m = myruns == 0 ? 0
                     : (myruns - 1) * run + (lastrun == nruns - 1 ? ntiles - lastrun * run : run);
    auto tile_of = [&](uint32_t j) -> uint32_t { return (blockIdx.x + (j / run) * G0) * run + j % run; };
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    // descriptor ring: warp 0 copies (cp.async, no registers held) 32 tiles
    // ahead; the copies complete (wait_group) 16 tiles before their first use
    auto ring_fill = [&](uint32_t j) {   // warp 0, lane l: local tile j + l
        const uint32_t jj = j + (tid & 31);
        if (jj < m) {
            const uint32_t t = tile_of(jj);
            const uint32_t d = smem_addr(&dring[jj & 63][0]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(tdesc + t) : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + 16), "l"(tdesc + t + 1) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (tid < 32) {
        ring_fill(0);
        ring_fill(32);
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    auto D = [&](uint32_t j) -> uint4 { return dring[j & 63][0]; };
    auto Dn = [&](uint32_t j) -> uint4 { return dring[j & 63][1]; };
    auto stage = [&](uint32_t j, int b) {   // thread 0: bulk copy of tile j's entry lists
        const uint32_t e0 = D(j).w, bytes = (Dn(j).w - e0) * 4u;
        mbar_arrive_expect_tx(&bar[b], bytes);
        if (bytes) bulk_g2s(ebuf + (size_t)b * max_ent, ents + e0, bytes, &bar[b]);
    };
    // the tile's NEW instances (tet, state slot | energy-owner << 16); carried
    // ones are already in shared memory
    auto inst_of = [&](uint32_t j) -> uint2 {
        if (j >= m) return make_uint2(0xFFFFFFFFu, 0);
        const uint32_t i0 = D(j).y, n = Dn(j).y - i0;
        return tid < n ? __ldg(inst + i0 + tid) : make_uint2(0xFFFFFFFFu, 0);
    };
    auto verts_of = [&](uint2 t) -> uint4 { return t.x == 0xFFFFFFFFu ? make_uint4(0, 0, 0, 0) : __ldg(tv + t.x); };

    // first pass of a tile's phase-2 items, loaded one tile ahead
    const uint4 no_item = make_uint4(0, 0xFFFFFFFFu, 0xFFFFFFFFu, 0);
    uint32_t it0_n = 0, nit_n = 0;
    uint4 item_n = no_item;
    auto item_head = [&](uint32_t j) {
        it0_n = 0;
        nit_n = 0;
        item_n = no_item;
        if (j >= m) return;
        it0_n = D(j).z;
        nit_n = Dn(j).z - it0_n;
        if (tid < nit_n) item_n = __ldg(items + it0_n + tid);
    };
    if (tid == 0 && m > 0) stage(0, 0);
    item_head(0);
    // software pipeline: inputs of this tile, keys of the next, tet id of the one after
    uint2 tc = inst_of(0);
    uint4 vc = verts_of(tc);
    SegIn<R> in;
    if constexpr (SEG_PIPE_INPUTS) seg_load(tc.x, vc, nt, u, Dminv, Wt, mu_t, lam_t, in);
    uint2 t1 = inst_of(1);
    uint4 v1 = verts_of(t1);
    uint2 t2 = inst_of(2);
    __shared__ double e_sm[NT];   // per-thread energy partial (kept out of the register budget)
    e_sm[tid] = 0.0;
#ifdef SEG_PROF
    // per-CTA wall-clock split (thread 0 and a lane of the last warp): phase 1,
    // barrier 1 + entry wait, phase 2, barrier 2
    long long tp[4] = {0, 0, 0, 0};
    long long tc0 = clock64();
#define SEG_MARK(q)                          \
    do {                                     \
        const long long tn = clock64();      \
        tp[q] += tn - tc0;                   \
        tc0 = tn;                            \
    } while (0)
#else
#define SEG_MARK(q) \
    do {            \
    } while (0)
#endif
    for (uint32_t j = 0; j < m; ++j) {
        const uint32_t k = j;
        // descriptor ring: copy [j + 32, j + 64) at j = 32 r, complete at j = 32 r + 16
        if (tid < 32) {
            if ((j & 31) == 0 && j > 0) ring_fill(j + 32);
            if ((j & 31) == 16) asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        // ---- phase 1: this thread's instance -> compact state
        if constexpr (!SEG_PIPE_INPUTS) seg_load(tc.x, vc, nt, u, Dminv, Wt, mu_t, lam_t, in);
        if (tc.x != 0xFFFFFFFFu) {
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
            const bool owner = (tc.y >> 16) & 1u;   // counted once: in its min vertex's run, first sighting
            if (MODEL == EBB_NH && owner && !(ts.J > R(0))) atomicAdd(&err[ERR_INVERTED], 1ull);
            if (WANT_E && owner) e_sm[tid] += (double)(ts.W * ts.psi);
            R fi[4][3];
            tet_forces(ts, fi);
            R* sr = st + (tc.y & 0xFFFFu);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    sr[(G::KV + 3 * i + a) * NT] = ts.kv[i][a];
                    sr[(G::F + 3 * i + a) * NT] = fi[i][a];
                }
#pragma unroll
            for (int p = 0; p < 10; ++p) {
                const int i = pair_i(p), j = pair_j(p);
                const R mij = ts.g[i][0] * ts.g[j][0] + ts.g[i][1] * ts.g[j][1] + ts.g[i][2] * ts.g[j][2];
                if constexpr (MODEL == EBB_NH) {
                    sr[(SegState<EBB_NH>::CM + p) * NT] = ts.W * ts.mu * mij;
                } else {
                    R Sg[3];
#pragma unroll
                    for (int a = 0; a < 3; ++a)
                        Sg[a] = ts.S[a][0] * ts.g[i][0] + ts.S[a][1] * ts.g[i][1] + ts.S[a][2] * ts.g[i][2];
                    sr[(SegState<EBB_STVK>::WS + p) * NT] =
                        ts.W * (Sg[0] * ts.g[j][0] + Sg[1] * ts.g[j][1] + Sg[2] * ts.g[j][2]);
                    sr[(SegState<EBB_STVK>::WM + p) * NT] = ts.W * ts.mu * mij;
                }
            }
            if constexpr (MODEL == EBB_NH) {
                sr[SegState<EBB_NH>::C1 * NT] = ts.W * ts.c1;
                sr[SegState<EBB_NH>::CL * NT] = ts.W * ts.lam;
            } else {
                constexpr int B = SegState<EBB_STVK>::B;
                sr[(B + 0) * NT] = ts.B[0][0];
                sr[(B + 1) * NT] = ts.B[0][1];
                sr[(B + 2) * NT] = ts.B[0][2];
                sr[(B + 3) * NT] = ts.B[1][1];
                sr[(B + 4) * NT] = ts.B[1][2];
                sr[(B + 5) * NT] = ts.B[2][2];
                sr[SegState<EBB_STVK>::CH * NT] = ts.W * ts.mu;
                sr[SegState<EBB_STVK>::CL * NT] = ts.W * ts.lam;
            }
        }
        // ---- advance the pipeline: these loads land during phase 2
        tc = t1;
        vc = v1;
        if constexpr (SEG_PIPE_INPUTS) seg_load(tc.x, vc, nt, u, Dminv, Wt, mu_t, lam_t, in);
        t1 = t2;
        v1 = verts_of(t1);
        t2 = inst_of(j + 3);
        if (tid == 0 && j + 1 < m) {
            fence_proxy_async_smem();
            stage(j + 1, (k + 1) & 1);
        }
        // phase-2 work list of this tile (its first pass was loaded one tile ahead)
        const uint32_t it0 = it0_n, nit = nit_n;
        uint4 item = item_n;
        item_head(j + 1);
        SEG_MARK(0);
        __syncthreads();   // state complete
        const int b = k & 1;
        mbar_wait(&bar[b], (k >> 1) & 1);
        SEG_MARK(1);
        const uint32_t* E = ebuf + (size_t)b * max_ent;
        // ---- phase 2: items = chunks of one row's list (self rows also sum the
        // vertex's force: their entries are exactly its (instance, corner) pairs);
        // the chunks of a list sit in consecutive lanes and are combined by a
        // shuffle tree (items are padded to whole warps: the loop is warp-uniform)
        for (uint32_t base = 0; base < nit; base += NT) {
            if (base) item = base + tid < nit ? __ldg(items + it0 + base + tid) : no_item;
            const uint32_t meta = item.x;
            const uint32_t e0 = meta & 0xFFFFu, e1 = e0 + ((meta >> 16) & 0x7Fu);
            const uint32_t pos = (meta >> 23) & 7u, last = (meta >> 26) & 7u, kind = (meta >> 29) & 3u;
            R a9[9];
#pragma unroll
            for (int q = 0; q < 9; ++q) a9[q] = R(0);
            // entry e + 1 is loaded while block e is rebuilt (the state loads
            // of a block depend only on its own entry)
            if (kind == 0) {
                uint32_t x = e0 < e1 ? E[e0] : 0u;
#pragma unroll kSegUnroll
                for (uint32_t e = e0; e < e1; ++e) {
                    const uint32_t nx = e + 1 < e1 ? E[e + 1] : 0u;
                    seg_block<R, MODEL, NT>(st, x, a9);
                    x = nx;
                }
            } else {
                // self row + the vertex's force: the same (instance, corner) list
                uint32_t x = e0 < e1 ? E[e0] : 0u;
#pragma unroll kSegUnroll
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
            // combine the chunks of a list (9 values: a block, or 6 + a force)
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
            if (pos == 0 && item.y != 0xFFFFFFFFu) {
                if (kind == 1) {
                    R* df = f + 3ull * item.z;
#pragma unroll
                    for (int a = 0; a < 3; ++a) df[a] = accumulate ? df[a] + a9[6 + a] : a9[6 + a];
                    // symmetric self block: expand 00 01 02 11 12 22
                    const R d[6] = {a9[0], a9[1], a9[2], a9[3], a9[4], a9[5]};
                    a9[0] = d[0]; a9[1] = d[1]; a9[2] = d[2];
                    a9[3] = d[1]; a9[4] = d[3]; a9[5] = d[4];
                    a9[6] = d[2]; a9[7] = d[4]; a9[8] = d[5];
                }
#ifdef SEG_NO_KSTORE   // measurement-only build: the cost of the scattered K row stores
                if (a9[0] == R(12345.678)) K[item.y] = a9[1];
#elif defined(SEG_KAOS_PROBE)   // measurement-only build: K rows element-major (72 contiguous bytes)
                {
                    R* dst = K + 9ull * item.y;
#pragma unroll
                    for (int q = 0; q < 9; ++q) dst[q] = a9[q];
                    if (kind == 0) {
                        dst = K + 9ull * item.z;
#pragma unroll
                        for (int a = 0; a < 3; ++a)
#pragma unroll
                            for (int c = 0; c < 3; ++c) dst[3 * a + c] = a9[3 * c + a];
                    }
                }
#else
                R* dst = K + item.y;
#pragma unroll
                for (int q = 0; q < 9; ++q, dst += ne) *dst = accumulate ? *dst + a9[q] : a9[q];
#ifdef SEG_NO_KSTORE_T   // measurement-only build: the transposed-row stores alone skipped
                if (kind == 0 && a9[0] == R(12345.678)) K[item.z] = a9[1];
#else
                if (kind == 0) {
                    dst = K + item.z;
#pragma unroll
                    for (int a = 0; a < 3; ++a)
#pragma unroll
                        for (int c = 0; c < 3; ++c, dst += ne) *dst = accumulate ? *dst + a9[3 * c + a] : a9[3 * c + a];
                }
#endif
#endif
            }
        }
        SEG_MARK(2);
        __syncthreads();   // state and entry buffer b free for reuse
        SEG_MARK(3);
    }
#ifdef SEG_PROF
    if (tid == 0 || tid == NT - 1) {
        const int w = tid == 0 ? 0 : 1;
        for (int q = 0; q < 4; ++q) atomicAdd((unsigned long long*)&g_seg_prof[8 * w + q], (unsigned long long)tp[q]);
        atomicAdd((unsigned long long*)&g_seg_prof[8 * w + 4], 1ull);
    }
#endif
    if (WANT_E) {
        double tot;
        if (block_sum_last_done(e_sm[tid], partials, counter, &tot)) *energy = (R)((double)*energy + tot);
    }
}

// ------------------------------------------------------------------ plan (host)
uint32_t lower_bound_u32(const uint32_t* a, uint32_t lo, uint32_t hi, uint32_t x) {
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <typename T>
ebb_status upload(Ctx* c, const std::vector<T>& h, T** d) {
    EBB_CUDA(c, cudaMalloc((void**)d, h.size() * sizeof(T) + 16));
    if (!h.empty()) EBB_CUDA(c, cudaMemcpy(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    return EBB_OK;
}

// Phase 2 walks, in lockstep, entry e of 32 lists (one per lane); each entry's
// shared-memory loads all hit bank pair (lr mod 16) of the state (fp64, SoA,
// NT a multiple of 16), so two lanes of a half-warp on the same pair with
// different lr serialize.  The order of a chunk's entries is free (the sum is
// still in a fixed, plan-given order): greedily give every lane, step by
// step, its remaining entry whose bank pair is least used by its half-warp.
void bank_schedule(uint4* it, size_t nit, uint32_t* ent, int ni) {
    std::vector<uint32_t> tmp;
    for (size_t w0 = 0; w0 + 32 <= nit; w0 += 32) {
        uint32_t steps = 0;
        for (int l = 0; l < 32; ++l) steps = std::max(steps, (it[w0 + l].x >> 16) & 0x7Fu);
        if (steps < 2) continue;
        std::vector<uint8_t> used(steps * 2 * 16, 0);
        for (int l = 0; l < 32; ++l) {
            const uint32_t meta = it[w0 + l].x, beg = meta & 0xFFFFu, sz = (meta >> 16) & 0x7Fu;
            if (sz < 2) {
                if (sz == 1) {
                    const uint32_t lr = (ent[beg] & 0x1FFFu) % (uint32_t)ni;
                    used[(0 * 2 + (l >> 4)) * 16 + (lr & 15)]++;
                }
                continue;
            }
            tmp.assign(ent + beg, ent + beg + sz);
            std::vector<char> taken(sz, 0);
            for (uint32_t e = 0; e < sz; ++e) {
                uint32_t best = 0, bc = 0xFFFFFFFFu;
                for (uint32_t k = 0; k < sz; ++k) {
                    if (taken[k]) continue;
                    const uint32_t lr = (tmp[k] & 0x1FFFu) % (uint32_t)ni;
                    const uint32_t cnt = used[(e * 2 + (l >> 4)) * 16 + (lr & 15)];
                    if (cnt < bc) {
                        bc = cnt;
                        best = k;
                    }
                }
                taken[best] = 1;
                ent[beg + e] = tmp[best];
                used[(e * 2 + (l >> 4)) * 16 + (((tmp[best] & 0x1FFFu) % (uint32_t)ni) & 15)]++;
            }
        }
    }
}

// One tile's plan (instances, phase-2 items, entry lists) appended to o.
// Independent of every other tile once the tile boundaries are fixed.
struct TileOut {
    std::vector<uint2> inst;
    std::vector<uint4> items;
    std::vector<uint32_t> ents;
    std::vector<uint32_t> n_inst, n_items, n_ents;   // per tile of this worker
    uint32_t max_ent = 0, max_items = 0;
    int err = 0;                                    // 1: > 65535 entries, 2: a list > 8 x 127
    uint32_t err_tile = 0;
    size_t err_len = 0;
};

struct PlanMesh {
    const uint32_t *tv, *index, *head, *vt_ptr, *vt, *rself, *tile_v, *tile_of_v;
    int ni;
    bool no_bank_sched, len_order;
};

void plan_tile(const PlanMesh& M, uint32_t T, TileOut& o) {
    const int ni = M.ni;
    const uint32_t a = M.tile_v[T], b = M.tile_v[T + 1];
    // instances: tets touching [a, b), ascending; state slot = position
    std::vector<uint32_t> tinst;
    for (uint32_t v = a; v < b; ++v)
        for (uint32_t q = M.vt_ptr[v]; q < M.vt_ptr[v + 1]; ++q) tinst.push_back(M.vt[q]);
    std::sort(tinst.begin(), tinst.end());
    tinst.erase(std::unique(tinst.begin(), tinst.end()), tinst.end());
    const uint32_t ninst = (uint32_t)tinst.size();
    for (uint32_t l = 0; l < ninst; ++l) {
        const uint32_t t = tinst[l];
        const uint32_t* vv = &M.tv[4ull * t];
        const uint32_t vmin = std::min(std::min(vv[0], vv[1]), std::min(vv[2], vv[3]));
        // the energy (and the inverted-element count) of a tet goes with its min vertex's tile
        const bool own = M.tile_of_v[vmin] == T;
        o.inst.push_back(make_uint2(t, l | (own ? 1u << 16 : 0u)));
    }
    // canonical slots of the tile in row order
    const uint32_t nvl = b - a;
    std::vector<uint32_t> sbase(nvl + 1, 0);
    for (uint32_t v = a; v < b; ++v) sbase[v - a + 1] = sbase[v - a] + (M.index[v + 1] - M.rself[v]);
    const uint32_t ns = sbase[nvl];
    std::vector<std::vector<uint32_t>> lists(ns);   // a self slot's list doubles as its vertex's force list
    for (uint32_t l = 0; l < ninst; ++l) {
        const uint32_t* vv = &M.tv[4ull * tinst[l]];
        for (int p = 0; p < 10; ++p) {
            const int i = pair_i(p), j = pair_j(p);
            const uint32_t lo = std::min(vv[i], vv[j]), hi = std::max(vv[i], vv[j]);
            if (lo < a || lo >= b) continue;
            const uint32_t r = lower_bound_u32(M.head, M.rself[lo], M.index[lo + 1], hi);
            const uint32_t sl = sbase[lo - a] + (r - M.rself[lo]);
            // block K_ij lands on row (v_i, v_j): transposed (K_ji) when v_i > v_j
            const uint32_t bi = vv[i] <= vv[j] ? i : j, bj = vv[i] <= vv[j] ? j : i;
            lists[sl].push_back((3 * bi * (uint32_t)ni + l) | ((3 * bj * (uint32_t)ni + l) << 13) | ((uint32_t)p << 26));
        }
    }
    // rows of the slots
    std::vector<uint32_t> srow(ns), strow(ns);
    for (uint32_t lv = 0; lv < nvl; ++lv)
        for (uint32_t sl = sbase[lv]; sl < sbase[lv + 1]; ++sl) {
            const uint32_t tail = a + lv, r = M.rself[tail] + (sl - sbase[lv]), hd = M.head[r];
            srow[sl] = r;
            strow[sl] = hd == tail ? r : lower_bound_u32(M.head, M.index[hd], M.index[hd + 1], tail);
        }
    // work lists in kind order: self rows + forces (1), off-diagonal rows (0) in row order
    // (a warp's stores of one K plane land on neighbouring rows: measured -7 % vs
    // descending list length, which EBB_SEG_LENORDER selects)
    std::vector<uint32_t> order;
    for (uint32_t lv = 0; lv < nvl; ++lv) order.push_back(sbase[lv]);
    const size_t n_self = order.size();
    for (uint32_t lv = 0; lv < nvl; ++lv)
        for (uint32_t sl = sbase[lv] + 1; sl < sbase[lv + 1]; ++sl) order.push_back(sl);
    if (M.len_order)
        std::stable_sort(order.begin() + n_self, order.end(),
                         [&](uint32_t x, uint32_t y) { return lists[x].size() > lists[y].size(); });
    auto kind_of = [&](size_t qi) -> uint32_t { return qi < n_self ? 1u : 0u; };
    const size_t e_base = o.ents.size();
    std::vector<uint32_t> lbeg(ns, 0);
    size_t tot = 0, longest = 0;
    for (uint32_t q : order) {
        lbeg[q] = (uint32_t)(o.ents.size() - e_base);
        o.ents.insert(o.ents.end(), lists[q].begin(), lists[q].end());
        tot += lists[q].size();
        longest = std::max(longest, lists[q].size());
    }
    while ((o.ents.size() - e_base) % 4) o.ents.push_back(0);
    const uint32_t nent = (uint32_t)(o.ents.size() - e_base);
    if (nent >= 65536 && !o.err) {
        o.err = 1;
        o.err_tile = T;
        o.err_len = nent;
    }
    // chunk cap L: the smallest (from the even share per thread) whose
    // warp-padded item list fits one pass of the CTA; at most 8 chunks a
    // list, the chunks of a list never straddle a warp, kinds start a warp
    const size_t it_base = o.items.size();
    auto layout = [&](size_t L, bool emit) {
        size_t n = 0;
        auto pad = [&]() {
            while (n % 32) {
                if (emit) o.items.push_back(make_uint4(0, 0xFFFFFFFFu, 0xFFFFFFFFu, 0));
                ++n;
            }
        };
        for (size_t qi = 0; qi < order.size(); ++qi) {
            if (qi > 0 && kind_of(qi) != kind_of(qi - 1)) pad();
            const uint32_t q = order[qi], kind = kind_of(qi);
            const uint32_t cnt = (uint32_t)lists[q].size();
            const uint32_t nc = cnt == 0 ? 1 : (uint32_t)((cnt + L - 1) / L);
            if ((n % 32) + nc > 32) pad();
            uint32_t beg = lbeg[q];
            for (uint32_t cc = 0; cc < nc; ++cc, ++n) {
                const uint32_t sz = cnt / nc + (cc < cnt % nc ? 1 : 0);
                if (emit) {
                    const uint32_t meta = beg | (sz << 16) | (cc << 23) | ((nc - 1) << 26) | (kind << 29);
                    // self rows: z = the vertex (its force); off-diagonal: z = the transpose row
                    o.items.push_back(kind == 1 ? make_uint4(meta, srow[q], a + (uint32_t)qi, 0)
                                                : make_uint4(meta, srow[q], strow[q], 0));
                }
                beg += sz;
            }
        }
        pad();
        return n;
    };
    // (a tile whose lists cannot fit one pass -- more rows than threads --
    // runs several passes: L stops growing at 4x the even share)
    const size_t L0 = std::max<size_t>({(size_t)2, (tot + ni - 1) / ni, (longest + 7) / 8});
    const size_t Lcap = std::max<size_t>(L0, std::min<size_t>(127, 4 * L0));
    size_t L = L0;
    while (L < Lcap && L < longest && layout(L, false) > (size_t)ni) ++L;
    if (L > 127 && !o.err) {
        o.err = 2;
        o.err_tile = T;
        o.err_len = longest;
    }
    if (L <= 127) layout(L, true);
    if (!M.no_bank_sched && L <= 127)
        bank_schedule(o.items.data() + it_base, o.items.size() - it_base, o.ents.data() + e_base, ni);
    o.max_ent = std::max(o.max_ent, nent);
    o.max_items = std::max(o.max_items, (uint32_t)(o.items.size() - it_base));
    o.n_inst.push_back(ninst);
    o.n_items.push_back((uint32_t)(o.items.size() - it_base));
    o.n_ents.push_back(nent);
}

ebb_status build_seg_plan(Ctx* c, ebb_field vf, ebb_field ef, int ni, SegPlan** out) {
    for (SegPlan* P : c->segplans)
        if (P->v == vf && P->e == ef && P->ni == ni) {
            *out = P;
            return EBB_OK;
        }
    const auto t_start = std::chrono::steady_clock::now();
    Field* V = get_field(c, vf);
    Field* E = get_field(c, ef);
    Relation& ER = c->rels[E->key_target];
    if (ER.grouped_by == EBB_NONE || ER.index == EBB_NONE)
        return fail(c, EBB_E_STATE, "segmented map: the edge relation must be grouped by tail");
    ebb_field hf = EBB_NONE;
    for (ebb_field fh : ER.fields)
        if (c->fields[fh].alive && c->fields[fh].name == "head") hf = fh;
    if (hf == EBB_NONE) return fail(c, EBB_E_STATE, "segmented map: edge relation has no 'head' key-field");
    const uint64_t nt = c->rels[V->rel].size, nv = c->rels[V->key_target].size, ne = ER.size;
    // on the device unless the host builder is asked for (EBB_SEG_PLAN=host, or
    // the EBB_SEG_LENORDER measurement ordering, which only the host has)
    const char* pe = getenv("EBB_SEG_PLAN");
    if (!(pe && std::string(pe) == "host") && !getenv("EBB_SEG_LENORDER")) {
        SegPlan* P = new SegPlan();
        P->v = vf;
        P->e = ef;
        P->ni = ni;
        const ebb_status st = build_seg_plan_device(c, (const uint32_t*)V->ptr, nt,
                                                    (const uint32_t*)c->fields[ER.index].ptr,
                                                    (const uint32_t*)c->fields[hf].ptr, nv, ni, P);
        if (st != EBB_OK) {
            P->release();
            delete P;
            return st;
        }
        c->segplans.push_back(P);
        *out = P;
        return EBB_OK;
    }
    std::vector<uint32_t> tv(nt * 4), index(nv + 1), head(ne);
    EBB_CUDA(c, cudaMemcpy(tv.data(), V->ptr, nt * 16, cudaMemcpyDeviceToHost));
    EBB_CUDA(c, cudaMemcpy(index.data(), c->fields[ER.index].ptr, (nv + 1) * 4, cudaMemcpyDeviceToHost));
    EBB_CUDA(c, cudaMemcpy(head.data(), c->fields[hf].ptr, ne * 4, cudaMemcpyDeviceToHost));
    // vertex -> incident tets (ascending tet id)
    std::vector<uint32_t> vt_ptr(nv + 1, 0), vt(nt * 4);
    for (uint64_t i = 0; i < nt * 4; ++i) vt_ptr[tv[i] + 1]++;
    for (uint64_t v = 0; v < nv; ++v) vt_ptr[v + 1] += vt_ptr[v];
    {
        std::vector<uint32_t> cur(vt_ptr.begin(), vt_ptr.end() - 1);
        for (uint64_t i = 0; i < nt * 4; ++i) vt[cur[tv[i]]++] = (uint32_t)(i >> 2);
    }
    // self row of every vertex (canonical rows of v = [self, index[v+1]))
    std::vector<uint32_t> rself(nv);
    for (uint64_t v = 0; v < nv; ++v) {
        rself[v] = lower_bound_u32(head.data(), index[v], index[v + 1], (uint32_t)v);
        if (rself[v] >= index[v + 1] || head[rself[v]] != v)
            return fail(c, EBB_E_STATE, "segmented map: vertex %llu has no self-loop edge row", (unsigned long long)v);
    }
    // greedy tiles: grow until the next vertex would push the instances past ni
    std::vector<uint32_t> tile_v{0};
    {
        std::vector<int64_t> stamp(nt, -1);
        int64_t tile = 0;
        uint32_t ci = 0, cv = 0;
        for (uint64_t v = 0; v < nv; ++v) {
            const uint32_t deg = vt_ptr[v + 1] - vt_ptr[v];
            if (deg > (uint32_t)ni)
                return fail(c, EBB_E_RANGE, "segmented map: vertex %llu touches %u tets (> %d per tile)",
                            (unsigned long long)v, deg, ni);
            uint32_t nw = 0;
            for (uint32_t q = vt_ptr[v]; q < vt_ptr[v + 1]; ++q) nw += stamp[vt[q]] != tile;
            // a tile never crosses a block of kSegBlock vertices (the device builder's unit)
            if (cv > 0 && (ci + nw > (uint32_t)ni || cv >= 4096 || v % kSegBlock == 0)) {
                tile_v.push_back((uint32_t)v);
                ++tile;
                ci = 0;
                cv = 0;
                nw = deg;
            }
            for (uint32_t q = vt_ptr[v]; q < vt_ptr[v + 1]; ++q) stamp[vt[q]] = tile;
            ci += nw;
            ++cv;
        }
        if (nv > 0) tile_v.push_back((uint32_t)nv);
    }
    const uint32_t ntiles = (uint32_t)tile_v.size() - 1;
    std::vector<uint32_t> tile_of_v(nv);
    for (uint32_t T = 0; T < ntiles; ++T)
        for (uint32_t v = tile_v[T]; v < tile_v[T + 1]; ++v) tile_of_v[v] = T;
    // per-tile plans, in parallel over contiguous tile ranges (host threads)
    PlanMesh M{tv.data(), index.data(), head.data(), vt_ptr.data(), vt.data(), rself.data(), tile_v.data(),
               tile_of_v.data(), ni, getenv("EBB_SEG_NO_BANK_SCHED") != nullptr, getenv("EBB_SEG_LENORDER") != nullptr};
    unsigned nth = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    if (ntiles < 64 * nth) nth = std::max(1u, ntiles / 64);
    std::vector<TileOut> outs(nth);
    {
        std::vector<std::thread> pool;
        for (unsigned w = 0; w < nth; ++w)
            pool.emplace_back([&, w]() {
                const uint32_t t0 = (uint32_t)((uint64_t)ntiles * w / nth), t1 = (uint32_t)((uint64_t)ntiles * (w + 1) / nth);
                for (uint32_t T = t0; T < t1; ++T) plan_tile(M, T, outs[w]);
            });
        for (auto& th : pool) th.join();
    }
    for (const TileOut& o : outs) {
        if (o.err == 1) return fail(c, EBB_E_RANGE, "segmented map: tile %u has %zu entries (> 65535)", o.err_tile, o.err_len);
        if (o.err == 2) return fail(c, EBB_E_RANGE, "segmented map: a list of %zu entries (> 8 x 127)", o.err_len);
    }
    // concatenate (tile order = worker order)
    std::vector<uint4> tdesc;
    tdesc.reserve(ntiles + 1);
    std::vector<uint2> inst;
    std::vector<uint4> items;
    std::vector<uint32_t> ents;
    size_t ni_tot = 0, nit_tot = 0, ne_tot = 0;
    for (const TileOut& o : outs) {
        ni_tot += o.inst.size();
        nit_tot += o.items.size();
        ne_tot += o.ents.size();
    }
    inst.reserve(ni_tot);
    items.reserve(nit_tot);
    ents.reserve(ne_tot);
    uint32_t max_ent = 0, max_items = 0, T = 0;
    for (const TileOut& o : outs) {
        size_t ii = 0, it = 0, ie = 0;
        for (size_t k = 0; k < o.n_inst.size(); ++k, ++T) {
            tdesc.push_back(make_uint4(tile_v[T], (uint32_t)(inst.size() + ii), (uint32_t)(items.size() + it),
                                       (uint32_t)(ents.size() + ie)));
            ii += o.n_inst[k];
            it += o.n_items[k];
            ie += o.n_ents[k];
        }
        inst.insert(inst.end(), o.inst.begin(), o.inst.end());
        items.insert(items.end(), o.items.begin(), o.items.end());
        ents.insert(ents.end(), o.ents.begin(), o.ents.end());
        max_ent = std::max(max_ent, o.max_ent);
        max_items = std::max(max_items, o.max_items);
    }
    tdesc.push_back(make_uint4(tile_v[ntiles], (uint32_t)inst.size(), (uint32_t)items.size(), (uint32_t)ents.size()));
    SegPlan* P = new SegPlan();
    P->v = vf;
    P->e = ef;
    P->ni = ni;
    P->ntiles = ntiles;
    P->max_ent = max_ent;
    P->max_items = max_items;
    P->ninst = inst.size();
    P->run = 1;
    P->nslots = 0;
    P->nent = ents.size();
    P->nitems = items.size();
    P->host_threads = nth;
    ebb_status s = EBB_OK;
    if (s == EBB_OK) s = upload(c, tdesc, &P->tdesc);
    if (s == EBB_OK) s = upload(c, inst, &P->inst);
    if (s == EBB_OK) s = upload(c, items, &P->items);
    if (s == EBB_OK) s = upload(c, ents, &P->ents);
    if (s != EBB_OK) {
        P->release();
        delete P;
        return s;
    }
    P->host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    c->segplans.push_back(P);
    *out = P;
    return EBB_OK;
}

template <typename R, int MODEL, int NT>
ebb_status launch_seg_t(Ctx* c, const SegPlan& P, bool want_e, int accumulate, uint64_t nt, const Field* V,
                        const Field* U, const Field* D, const Field* W, const Field* MU, const Field* LA,
                        const Field* Fo, const Field* Ko, uint64_t ne, const Field* En, cudaStream_t s) {
    const size_t smem = (size_t)SegState<MODEL>::SW * NT * sizeof(R) + 2ull * P.max_ent * 4;
    if (smem > 227 * 1024)
        return fail(c, EBB_E_RANGE, "segmented map: %zu B of shared memory needed (> 227 KB)", smem);
    auto kern = want_e ? k_tet_map_seg<R, MODEL, true, NT> : k_tet_map_seg<R, MODEL, false, NT>;
    static thread_local size_t configured_dev[kMaxDevices][2] = {};
    size_t* const configured = configured_dev[c->device % kMaxDevices];   // attribute set once (graph-capture safe)
    if (smem > configured[want_e]) {
        EBB_CUDA(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured[want_e] = smem;
    }
    unsigned grid = occ_grid(c, kern, NT, smem, (uint64_t)P.ntiles * NT);
    const char* eg = getenv("EBB_SEG_GRID");   // test knob: fewer CTAs = longer tile runs per CTA
    if (eg && atoi(eg) > 0 && (unsigned)atoi(eg) < grid) grid = (unsigned)atoi(eg);
    KernelTimer kt(c, EBB_K_TET_MAP, s);
    kern<<<grid, NT, smem, s>>>(P.ntiles, P.run, P.tdesc, P.inst, P.items, P.ents, P.max_ent, nt, (const uint4*)V->ptr,
                                (const R*)U->ptr, (const R*)D->ptr, (const R*)W->ptr, (const R*)MU->ptr,
                                (const R*)LA->ptr, (R*)Fo->ptr, (R*)Ko->ptr, ne, accumulate, c->d_partials,
                                c->d_counter + 0, En ? (R*)En->ptr : nullptr, c->d_err);
    EBB_CUDA(c, cudaGetLastError());
#ifdef SEG_PROF
    {
        unsigned long long h[16];
        cudaDeviceSynchronize();
        cudaMemcpyFromSymbol(h, g_seg_prof, sizeof(h));
        const unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(g_seg_prof, z, sizeof(z));
        for (int w = 0; w < 2; ++w) {
            const double tot = (double)(h[8 * w] + h[8 * w + 1] + h[8 * w + 2] + h[8 * w + 3]);
            fprintf(stderr, "SEG_PROF %s: phase1 %.1f%% bar1+wait %.1f%% phase2 %.1f%% bar2 %.1f%% (ctas %llu, Mcycles/cta %.2f)\n",
                    w ? "last thread" : "thread 0", 100 * h[8 * w] / tot, 100 * h[8 * w + 1] / tot,
                    100 * h[8 * w + 2] / tot, 100 * h[8 * w + 3] / tot, h[8 * w + 4], tot / h[8 * w + 4] / 1e6);
        }
    }
#endif
    return EBB_OK;
}

}  // namespace

// threads per CTA = instance cap per tile: the compact state must fit in
// shared memory next to two entry buffers (fp64 StVK state is 52 words)
int seg_threads(ebb_dtype dt, int model, uint64_t nt) {
    const char* e = getenv("EBB_SEG_NT");
    if (e && (atoi(e) == 128 || atoi(e) == 256 || atoi(e) == 384 || atoi(e) == 512)) {
        const int v = atoi(e);
        return (dt == EBB_F64 && model == EBB_STVK && v > 384) ? 384 : v;
    }
    // measured: fp64 StVK 384; fp64 NH 512 from 2e6 tets
    // (7-12 % faster from 3e6 tets, equal at 1e6, 5 % slower at 3e5); fp32
    // StVK 512 from 4e6 tets (11 % faster at 1e7, 1-2 % slower at <= 1e6);
    // otherwise 256
    if (dt == EBB_F64 && model == EBB_STVK) return 384;
    if (dt == EBB_F64 && model == EBB_NH && nt >= 2000000) return 512;
    if (dt == EBB_F32 && model == EBB_STVK && nt >= 4000000) return 512;
    return 256;
}

ebb_status seg_plan_probe(Ctx* c, ebb_field vf, ebb_field ef, ebb_dtype dt, int model) {
    SegPlan* P;
    return build_seg_plan(c, vf, ef, seg_threads(dt, model, c->rels[get_field(c, vf)->rel].size), &P);
}

ebb_status seg_map_launch(Ctx* c, ebb_field vf, ebb_field ef, int model, bool want_e, int accumulate, uint64_t nt,
                          const Field* V, const Field* U, const Field* D, const Field* W, const Field* MU,
                          const Field* LA, const Field* Fo, const Field* Ko, uint64_t ne, const Field* En,
                          cudaStream_t s) {
    const ebb_dtype dt = U->dtype;
    const int NT = seg_threads(dt, model, nt);
    SegPlan* P;
    EBB_TRY(build_seg_plan(c, vf, ef, NT, &P));
#define EBB_SARGS c, *P, want_e, accumulate, nt, V, U, D, W, MU, LA, Fo, Ko, ne, En, s
#define EBB_SDISPATCH(R, MODEL)                                               \
    do {                                                                      \
        if (NT == 128) return launch_seg_t<R, MODEL, 128>(EBB_SARGS);         \
        if (NT == 256) return launch_seg_t<R, MODEL, 256>(EBB_SARGS);         \
        if (NT == 384) return launch_seg_t<R, MODEL, 384>(EBB_SARGS);         \
        if constexpr (!(sizeof(R) == 8 && MODEL == EBB_STVK))                 \
            return launch_seg_t<R, MODEL, 512>(EBB_SARGS);                    \
        return fail(c, EBB_E_ARG, "segmented map: bad thread count %d", NT); \
    } while (0)
    if (dt == EBB_F64) {
        if (model == EBB_NH) EBB_SDISPATCH(double, EBB_NH);
        EBB_SDISPATCH(double, EBB_STVK);
    }
    if (model == EBB_NH) EBB_SDISPATCH(float, EBB_NH);
    EBB_SDISPATCH(float, EBB_STVK);
#undef EBB_SDISPATCH
#undef EBB_SARGS
}

}  // namespace ebb

extern "C" ebb_status ebb_map_plan_stats(ebb_ctx ctx, ebb_field v, ebb_field e, double out[8]) {
    using namespace ebb;
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !out) return EBB_E_ARG;
    for (int k = 0; k < 8; ++k) out[k] = 0;
    Field* V = get_field(c, v);
    if (!V) return fail(c, EBB_E_ARG, "map_plan_stats: bad field handle");
    const double nt = (double)c->rels[V->rel].size;
    for (SegPlan* P : c->segplans)
        if (P->v == v && P->e == e) {
            out[0] = P->ntiles;
            out[1] = (double)P->ninst;
            out[2] = nt > 0 ? (double)P->ninst / nt : 0;
            out[3] = (double)P->nent;
            out[4] = (double)P->nitems;
            out[5] = P->ni;
            out[6] = P->host_ms;
            out[7] = P->max_ent;
        }
    return EBB_OK;
}
