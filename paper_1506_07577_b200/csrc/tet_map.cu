// tet_map.cu -- the element map over the tets relation.
//
// Per tet (P:941-946 Vega StVK, P:975-980 neo-Hookean "specialized"): gather
// u[v[k]] through the key-field tets.v, element physics
// (element.cuh: displacement form + closed rank-1 stiffness), and the
// reductions f[v[i]] += f_i, K[e[i][j]] += K_ij (field `+=`) and
// energy += W Psi (global `+=`, fused two-pass).
//
// The entry point and three of the five scatter strategies (SURVEY §8(a)
// "the += strategies", chosen by measurement -- DESIGN.md §5.2):
//   ATOMIC  one thread per tet, red.global.add per value (the paper's field
//           reductions with native fp64 RED instead of Kepler CAS);
//   TILED   owner-computes vertex tiles: a CTA owns the canonical edge rows
//           (tail <= head) and the forces of a tile of consecutive vertices,
//           recomputes every tet touching the tile, accumulates in shared
//           memory and writes each K row and f row exactly once with plain
//           stores (row (b,a) as the transpose of canonical (a,b)).  No global
//           atomics, no zero-fill of K.
//   GATHER  the same tiles, warp-specialized producer/consumer rounds.
// SEGMENTED (the default, seg_map.cu) and COLOR (color_map.cu) live in their
// own files.
// The oracle computes the same quantities by the textbook F-form and a generic
// 4th-order tensor contraction (oracle/ebb_oracle.c); the two share no code.
#include <cub/cub.cuh>

#include <cstdlib>

#include "ebb_internal.cuh"
#include "element.cuh"
#include "reduce.cuh"

using namespace ebb;

namespace {

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

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

// ---------------------------------------------------------------- plan build
// pair order: off-diagonal (0,1) (0,2) (0,3) (1,2) (1,3) (2,3), diagonal (0,0)..(3,3)
__constant__ int8_t kPairI[10] = {0, 0, 0, 1, 1, 2, 0, 1, 2, 3};
__constant__ int8_t kPairJ[10] = {1, 2, 3, 2, 3, 3, 0, 1, 2, 3};

__global__ void k_canon_flag(uint64_t ne, const uint32_t* __restrict__ tail, const uint32_t* __restrict__ head,
                             uint32_t* __restrict__ flag) {
    uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (r < ne) flag[r] = head[r] >= tail[r] ? 1u : 0u;
}

__device__ __forceinline__ uint32_t find_row_d(const uint32_t* __restrict__ index, const uint32_t* __restrict__ head,
                                               uint32_t a, uint32_t b) {
    uint32_t lo = index[a], hi = index[a + 1];
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (head[mid] < b) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void k_canon_lists(uint64_t ne, const uint32_t* __restrict__ tail, const uint32_t* __restrict__ head,
                              const uint32_t* __restrict__ index, const uint32_t* __restrict__ gci,
                              uint32_t* __restrict__ crow, uint32_t* __restrict__ ctrow) {
    uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (r >= ne) return;
    uint32_t a = tail[r], b = head[r];
    if (b < a) return;
    uint32_t g = gci[r];
    crow[g] = (uint32_t)r;
    ctrow[g] = (a == b) ? (uint32_t)r : find_row_d(index, head, b, a);
}

__global__ void k_tile_cptr(uint32_t ntiles, int nvt, uint64_t nv, const uint32_t* __restrict__ index,
                            const uint32_t* __restrict__ gci, uint64_t ne, uint32_t ncanon, uint32_t* __restrict__ cptr) {
    uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t > ntiles) return;
    uint64_t v = t * (uint64_t)nvt;
    if (v > nv) v = nv;
    uint32_t r = index[v];
    cptr[t] = (r >= ne) ? ncanon : gci[r];
}

// contributions per canonical row (every tet adds one block per pair)
__global__ void k_canon_counts(uint64_t nt, const uint32_t* __restrict__ tv, const uint32_t* __restrict__ te,
                               const uint32_t* __restrict__ gci, uint32_t* __restrict__ cnt) {
    uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    uint32_t v[4];
    for (int k = 0; k < 4; ++k) v[k] = tv[4 * t + k];
    for (int p = 0; p < 10; ++p) {
        const int a = kPairI[p], b = kPairJ[p];
        const uint32_t r = (v[a] <= v[b]) ? te[16 * t + 4 * a + b] : te[16 * t + 4 * b + a];
        atomicAdd(&cnt[gci[r]], 1u);
    }
}

__device__ __forceinline__ uint32_t range_of(const uint32_t* __restrict__ ptr, uint32_t n, uint64_t i) {
    uint32_t lo = 0, hi = n;   // last k with ptr[k] <= i
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (ptr[mid] <= i) lo = mid;
        else hi = mid;
    }
    return lo;
}

// sort key of a canonical slot: its tile, then descending contribution count
__global__ void k_slot_keys(uint64_t ncanon, uint32_t ntiles, const uint32_t* __restrict__ tile_cptr,
                            const uint32_t* __restrict__ cnt, uint64_t* __restrict__ key, uint32_t* __restrict__ val) {
    uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (g >= ncanon) return;
    key[g] = ((uint64_t)range_of(tile_cptr, ntiles, g) << 32) | (0xFFFFFFFFu - cnt[g]);
    val[g] = (uint32_t)g;
}

__global__ void k_slot_newpos(uint64_t ncanon, const uint32_t* __restrict__ order, uint32_t* __restrict__ newpos,
                              const uint32_t* __restrict__ crow, const uint32_t* __restrict__ ctrow,
                              uint32_t* __restrict__ crow2, uint32_t* __restrict__ ctrow2) {
    uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= ncanon) return;
    const uint32_t g = order[k];
    newpos[g] = (uint32_t)k;
    crow2[k] = crow[g];
    ctrow2[k] = ctrow[g];
}

__global__ void k_remap_gci(uint64_t ne, const uint32_t* __restrict__ flag, const uint32_t* __restrict__ newpos,
                            uint32_t* __restrict__ gci) {
    uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (r < ne && flag[r]) gci[r] = newpos[gci[r]];
}

__global__ void k_inst_keys(uint64_t nt, const uint32_t* __restrict__ tv, int nvt, uint64_t* __restrict__ keys) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= nt * 4) return;
    uint64_t t = i >> 2;
    keys[i] = ((uint64_t)(tv[i] / (uint32_t)nvt) << 32) | t;
}

__global__ void k_inst_ptr(const uint64_t* __restrict__ keys, uint64_t n, uint32_t* __restrict__ ptr, uint32_t ntiles) {
    uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (s > ntiles) return;
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if ((keys[mid] >> 32) < s) lo = mid + 1;
        else hi = mid;
    }
    ptr[s] = (uint32_t)lo;
}

// record words: w0 tet | w1..w5 slot[10] (u16) | w6 local vertex of corner k (u8) | w7 flags
// flags bit p (p < 6): block of pair p is stored transposed; bit 8: energy owner
__global__ void k_inst_records(uint64_t ninst, const uint64_t* __restrict__ keys, const uint32_t* __restrict__ tv,
                               const uint32_t* __restrict__ te, const uint32_t* __restrict__ gci,
                               const uint32_t* __restrict__ cptr, int nvt, const uint32_t* __restrict__ inst_ptr,
                               const uint32_t* __restrict__ rec_ptr, int round, uint32_t* __restrict__ recs) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= ninst) return;
    const uint32_t tile = (uint32_t)(keys[i] >> 32);
    const uint64_t t0 = inst_ptr[tile], nloc = inst_ptr[tile + 1] - t0;
    uint64_t out;
    if (round == 0) {
        // Tiled: a pseudo-random order (k -> k * 1000003 mod n, a bijection
        // since the prime exceeds n): SFC-adjacent tets share rows, and
        // processing them concurrently makes every thread of a CTA CAS the same
        // shared-memory words; scattered, a row's ~24 contributors rarely coincide.
        out = t0 + ((i - t0) * 1000003ull) % nloc;
    } else {
        // Gather: the (SFC-sorted) instances dealt round-robin over the tile's
        // rounds, so every row receives an even share of its contributions in
        // each round and the owner threads of a warp stay converged.
        const uint64_t k = i - t0, nr = (nloc + round - 1) / round;
        out = rec_ptr[tile] + (k % nr) * (uint64_t)round + k / nr;
    }
    const uint64_t t = keys[i] & 0xFFFFFFFFull;
    uint32_t v[4];
    for (int k = 0; k < 4; ++k) v[k] = tv[4 * t + k];
    uint32_t w[8] = {(uint32_t)t, 0, 0, 0, 0, 0, 0, 0};
    uint32_t flags = 0;
    for (int p = 0; p < 10; ++p) {
        int a = kPairI[p], b = kPairJ[p];
        uint32_t lo = v[a] < v[b] ? v[a] : v[b];
        uint32_t slot = 0xFFFFu;
        if (lo / (uint32_t)nvt == tile) {
            // canonical row (min, max); block K_ab is stored transposed when v_a > v_b
            uint32_t r = (v[a] <= v[b]) ? te[16 * t + 4 * a + b] : te[16 * t + 4 * b + a];
            slot = gci[r] - cptr[tile];
            if (p < 6 && v[a] > v[b]) flags |= 1u << p;
        }
        w[1 + p / 2] |= slot << (16 * (p & 1));
    }
    uint32_t vmin = v[0];
    for (int k = 0; k < 4; ++k) {
        uint32_t lv = (v[k] / (uint32_t)nvt == tile) ? (v[k] - tile * (uint32_t)nvt) : 0xFFu;
        w[6] |= lv << (8 * k);
        vmin = v[k] < vmin ? v[k] : vmin;
    }
    if (vmin / (uint32_t)nvt == tile) flags |= 1u << 8;
    w[7] = flags;
    for (int k = 0; k < 8; ++k) recs[8 * out + k] = w[k];
}

// gather plans: once the contribution lists exist, a record only needs
// (t, v0..v3, flags) -- the vertex ids ride along so the producer's loads of
// u / Dminv / W are one dependent step from the record
__global__ void k_gather_records(uint64_t nrec, const uint32_t* __restrict__ tv, uint32_t* __restrict__ recs) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= nrec) return;
    uint32_t* w = recs + 8 * i;
    const uint32_t t = w[0];
    if (t == 0xFFFFFFFFu) return;
    for (int k = 0; k < 4; ++k) w[1 + k] = tv[4ull * t + k];
}

__global__ void k_round_counts(uint32_t ntiles, const uint32_t* __restrict__ inst_ptr, int round,
                               uint32_t* __restrict__ cnt) {
    uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > ntiles) return;
    cnt[t] = t == ntiles ? 0u : (inst_ptr[t + 1] - inst_ptr[t] + round - 1) / round * round;
}

__global__ void k_max_diff(const uint32_t* __restrict__ ptr, uint32_t n, unsigned int* out) {
    uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < n) atomicMax(out, ptr[s + 1] - ptr[s]);
}

// ---- gather-strategy contribution lists
__global__ void k_tile_ent_max(uint32_t ntiles, int nvt, uint64_t nv, const uint32_t* __restrict__ tile_cptr,
                               const uint32_t* __restrict__ slot_ptr, const uint32_t* __restrict__ fv_ptr,
                               unsigned int* out) {
    uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntiles) return;
    atomicMax(out, slot_ptr[tile_cptr[t + 1]] - slot_ptr[tile_cptr[t]]);
    const uint64_t v0 = (uint64_t)t * nvt, v1 = v0 + nvt < nv ? v0 + nvt : nv;
    atomicMax(out + 1, fv_ptr[v1] - fv_ptr[v0]);
}

__device__ __forceinline__ uint32_t tile_of(const uint32_t* __restrict__ inst_ptr, uint32_t ntiles, uint64_t i) {
    uint32_t lo = 0, hi = ntiles;   // last tile with inst_ptr[tile] <= i
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (inst_ptr[mid] <= i) lo = mid;
        else hi = mid;
    }
    return lo;
}

__global__ void k_entry_counts(uint64_t ninst, const uint32_t* __restrict__ recs, uint32_t* __restrict__ npair,
                               uint32_t* __restrict__ ncorner) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= ninst) return;
    const uint32_t* w = recs + 8 * i;
    uint32_t a = 0, b = 0;
    for (int p = 0; p < 10; ++p) a += ((w[1 + p / 2] >> (16 * (p & 1))) & 0xFFFFu) != 0xFFFFu;
    for (int k = 0; k < 4; ++k) b += ((w[6] >> (8 * k)) & 0xFFu) != 0xFFu;
    npair[i] = a;
    ncorner[i] = b;
}

__global__ void k_entry_emit(uint64_t ninst, const uint32_t* __restrict__ recs, const uint32_t* __restrict__ inst_ptr,
                             uint32_t ntiles, const uint32_t* __restrict__ cptr, int nvt,
                             const uint32_t* __restrict__ poff, const uint32_t* __restrict__ coff,
                             uint32_t* __restrict__ pkey, uint32_t* __restrict__ pval, uint32_t* __restrict__ ckey,
                             uint32_t* __restrict__ cval) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= ninst) return;
    const uint32_t* w = recs + 8 * i;
    const uint32_t tile = tile_of(inst_ptr, ntiles, i);
    const uint32_t li = (uint32_t)(i - inst_ptr[tile]);
    uint32_t o = poff[i];
    for (int p = 0; p < 10; ++p) {
        const uint32_t slot = (w[1 + p / 2] >> (16 * (p & 1))) & 0xFFFFu;
        if (slot == 0xFFFFu) continue;
        // (i, j) of the block as stored in the canonical row: a transposed
        // contribution K_ij^T = K_ji is the same closed form with i, j swapped
        const bool tr = p < 6 && ((w[7] >> p) & 1u);
        const uint32_t bi = (uint32_t)(tr ? kPairJ[p] : kPairI[p]), bj = (uint32_t)(tr ? kPairI[p] : kPairJ[p]);
        pkey[o] = cptr[tile] + slot;
        pval[o] = (li << 8) | (bi << 6) | (bj << 4) | (uint32_t)p;
        ++o;
    }
    o = coff[i];
    for (int k = 0; k < 4; ++k) {
        const uint32_t lv = (w[6] >> (8 * k)) & 0xFFu;
        if (lv == 0xFFu) continue;
        ckey[o] = tile * (uint32_t)nvt + lv;
        cval[o] = (li << 2) | (uint32_t)k;
        ++o;
    }
}

__global__ void k_lower_bound_u32(const uint32_t* __restrict__ sorted, uint64_t n, uint32_t* __restrict__ ptr,
                                  uint64_t nkeys) {
    uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (s > nkeys) return;
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if (sorted[mid] < s) lo = mid + 1;
        else hi = mid;
    }
    ptr[s] = (uint32_t)lo;
}

// sort (key, value) pairs by key and build key -> [ptr[k], ptr[k+1]) offsets
ebb_status sort_entries(Ctx* c, uint32_t* key, uint32_t* val, uint64_t n, uint64_t nkeys, uint32_t** ptr_out,
                        uint32_t** ent_out) {
    DevBuf k2, tmp;
    int bits = 1;
    while (bits < 32 && (1ull << bits) <= nkeys) ++bits;
    EBB_CUDA(c, cudaMalloc(&k2.p, n * 4 + 16));
    EBB_CUDA(c, cudaMalloc(ent_out, n * 4 + 16));
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, key, (uint32_t*)k2.p, val, *ent_out, (int)n, 0, bits);
    EBB_CUDA(c, cudaMalloc(&tmp.p, tb));
    EBB_CUDA(c, cub::DeviceRadixSort::SortPairs(tmp.p, tb, key, (uint32_t*)k2.p, val, *ent_out, (int)n, 0, bits));
    EBB_CUDA(c, cudaMalloc(ptr_out, (nkeys + 1) * 4));
    k_lower_bound_u32<<<grid_for(nkeys + 1, 256), 256>>>((const uint32_t*)k2.p, n, *ptr_out, nkeys);
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status build_gather_lists(Ctx* c, MapPlan& P, uint64_t nv) {
    const uint64_t ni = P.ninst;
    DevBuf npair, ncorner, poff, coff, tmp, pkey, pval, ckey, cval, mx;
    EBB_CUDA(c, cudaMalloc(&npair.p, ni * 4 + 16));
    EBB_CUDA(c, cudaMalloc(&ncorner.p, ni * 4 + 16));
    EBB_CUDA(c, cudaMalloc(&poff.p, ni * 4 + 16));
    EBB_CUDA(c, cudaMalloc(&coff.p, ni * 4 + 16));
    k_entry_counts<<<grid_for(ni, 256), 256>>>(ni, (const uint32_t*)P.recs, (uint32_t*)npair.p, (uint32_t*)ncorner.p);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, (const uint32_t*)npair.p, (uint32_t*)poff.p, (int)ni);
    EBB_CUDA(c, cudaMalloc(&tmp.p, tb));
    EBB_CUDA(c, cub::DeviceScan::ExclusiveSum(tmp.p, tb, (const uint32_t*)npair.p, (uint32_t*)poff.p, (int)ni));
    EBB_CUDA(c, cub::DeviceScan::ExclusiveSum(tmp.p, tb, (const uint32_t*)ncorner.p, (uint32_t*)coff.p, (int)ni));
    uint32_t lp, lc, op, oc;
    EBB_CUDA(c, cudaMemcpy(&lp, (uint32_t*)npair.p + ni - 1, 4, cudaMemcpyDeviceToHost));
    EBB_CUDA(c, cudaMemcpy(&lc, (uint32_t*)ncorner.p + ni - 1, 4, cudaMemcpyDeviceToHost));
    EBB_CUDA(c, cudaMemcpy(&op, (uint32_t*)poff.p + ni - 1, 4, cudaMemcpyDeviceToHost));
    EBB_CUDA(c, cudaMemcpy(&oc, (uint32_t*)coff.p + ni - 1, 4, cudaMemcpyDeviceToHost));
    const uint64_t np = (uint64_t)op + lp, nc = (uint64_t)oc + lc;
    EBB_CUDA(c, cudaMalloc(&pkey.p, np * 4 + 16));
    EBB_CUDA(c, cudaMalloc(&pval.p, np * 4 + 16));
    EBB_CUDA(c, cudaMalloc(&ckey.p, nc * 4 + 16));
    EBB_CUDA(c, cudaMalloc(&cval.p, nc * 4 + 16));
    k_entry_emit<<<grid_for(ni, 256), 256>>>(ni, (const uint32_t*)P.recs, P.inst_ptr, P.ntiles, P.tile_cptr, P.nvt,
                                             (const uint32_t*)poff.p, (const uint32_t*)coff.p, (uint32_t*)pkey.p,
                                             (uint32_t*)pval.p, (uint32_t*)ckey.p, (uint32_t*)cval.p);
    EBB_CUDA(c, cudaGetLastError());
    EBB_TRY(sort_entries(c, (uint32_t*)pkey.p, (uint32_t*)pval.p, np, P.ncanon, &P.slot_ptr, &P.slot_ent));
    EBB_TRY(sort_entries(c, (uint32_t*)ckey.p, (uint32_t*)cval.p, nc, nv, &P.fv_ptr, &P.fv_ent));
    EBB_CUDA(c, cudaMalloc(&mx.p, 4));
    EBB_CUDA(c, cudaMemset(mx.p, 0, 4));
    k_max_diff<<<grid_for(P.ntiles, 256), 256>>>(P.inst_ptr, P.ntiles, (unsigned int*)mx.p);
    EBB_CUDA(c, cudaMemcpy(&P.max_inst, mx.p, 4, cudaMemcpyDeviceToHost));
    DevBuf mx2;
    EBB_CUDA(c, cudaMalloc(&mx2.p, 8));
    EBB_CUDA(c, cudaMemset(mx2.p, 0, 8));
    k_tile_ent_max<<<grid_for(P.ntiles, 256), 256>>>(P.ntiles, P.nvt, nv, P.tile_cptr, P.slot_ptr, P.fv_ptr,
                                                     (unsigned int*)mx2.p);
    uint32_t m2[2];
    EBB_CUDA(c, cudaMemcpy(m2, mx2.p, 8, cudaMemcpyDeviceToHost));
    P.max_sent = m2[0];
    P.max_fent = m2[1];
    return EBB_OK;
}

ebb_status build_plan(Ctx* c, ebb_field vf, ebb_field ef, int nvt, int round, MapPlan** out) {
    for (auto& P : c->plans)
        if (P.v == vf && P.e == ef && P.nvt == nvt && P.round == round) {
            *out = &P;
            return EBB_OK;
        }
    Field* V = get_field(c, vf);
    Field* E = get_field(c, ef);
    ebb_rel edges = E->key_target;
    Relation& ER = c->rels[edges];
    if (ER.grouped_by == EBB_NONE || ER.index == EBB_NONE)
        return fail(c, EBB_E_STATE, "tiled map: the edge relation must be grouped by tail");
    ebb_field hf = EBB_NONE;
    for (ebb_field f : ER.fields)
        if (c->fields[f].alive && c->fields[f].name == "head") hf = f;
    if (hf == EBB_NONE) return fail(c, EBB_E_STATE, "tiled map: edge relation has no 'head' key-field");
    const uint32_t* tail = (const uint32_t*)c->fields[ER.grouped_by].ptr;
    const uint32_t* head = (const uint32_t*)c->fields[hf].ptr;
    const uint32_t* index = (const uint32_t*)c->fields[ER.index].ptr;
    const uint64_t nt = c->rels[V->rel].size, nv = c->rels[V->key_target].size, ne = ER.size;
    MapPlan P;
    P.v = vf;
    P.e = ef;
    P.nvt = nvt;
    P.round = round;
    P.ntiles = (uint32_t)((nv + nvt - 1) / nvt);
    DevBuf flag, gci, tmp, keys, keys2, uk, nsel, mx, tmp2;
    EBB_CUDA(c, cudaMalloc(&flag.p, ne * 4));
    EBB_CUDA(c, cudaMalloc(&gci.p, ne * 4));
    k_canon_flag<<<grid_for(ne, 256), 256>>>(ne, tail, head, (uint32_t*)flag.p);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, (const uint32_t*)flag.p, (uint32_t*)gci.p, (int)ne);
    EBB_CUDA(c, cudaMalloc(&tmp.p, tb));
    EBB_CUDA(c, cub::DeviceScan::ExclusiveSum(tmp.p, tb, (const uint32_t*)flag.p, (uint32_t*)gci.p, (int)ne));
    uint32_t last_g = 0, last_f = 0;
    EBB_CUDA(c, cudaMemcpy(&last_g, (uint32_t*)gci.p + ne - 1, 4, cudaMemcpyDeviceToHost));
    EBB_CUDA(c, cudaMemcpy(&last_f, (uint32_t*)flag.p + ne - 1, 4, cudaMemcpyDeviceToHost));
    P.ncanon = (uint64_t)last_g + last_f;
    EBB_CUDA(c, cudaMalloc(&P.crow, P.ncanon * 4));
    EBB_CUDA(c, cudaMalloc(&P.ctrow, P.ncanon * 4));
    k_canon_lists<<<grid_for(ne, 256), 256>>>(ne, tail, head, index, (const uint32_t*)gci.p, P.crow, P.ctrow);
    EBB_CUDA(c, cudaMalloc(&P.tile_cptr, (P.ntiles + 1) * 4));
    k_tile_cptr<<<grid_for(P.ntiles + 1, 256), 256>>>(P.ntiles, nvt, nv, index, (const uint32_t*)gci.p, ne,
                                                      (uint32_t)P.ncanon, P.tile_cptr);
    {
        // number each tile's canonical slots by descending contribution count:
        // the gather map deals slots to its owner threads in this order, so
        // the lanes of a warp walk lists of similar length
        const uint64_t nc = P.ncanon;
        DevBuf cnt, sk, sk2, sv, sv2, npos, cr2, ctr2, stmp;
        EBB_CUDA(c, cudaMalloc(&cnt.p, nc * 4 + 16));
        EBB_CUDA(c, cudaMemset(cnt.p, 0, nc * 4 + 16));
        k_canon_counts<<<grid_for(nt, 256), 256>>>(nt, (const uint32_t*)V->ptr, (const uint32_t*)E->ptr,
                                                   (const uint32_t*)gci.p, (uint32_t*)cnt.p);
        EBB_CUDA(c, cudaMalloc(&sk.p, nc * 8 + 16));
        EBB_CUDA(c, cudaMalloc(&sk2.p, nc * 8 + 16));
        EBB_CUDA(c, cudaMalloc(&sv.p, nc * 4 + 16));
        EBB_CUDA(c, cudaMalloc(&sv2.p, nc * 4 + 16));
        k_slot_keys<<<grid_for(nc, 256), 256>>>(nc, P.ntiles, P.tile_cptr, (const uint32_t*)cnt.p, (uint64_t*)sk.p,
                                                (uint32_t*)sv.p);
        int tb3 = 1;
        while (tb3 < 32 && (1ull << tb3) <= P.ntiles) ++tb3;
        size_t tbs = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tbs, (const uint64_t*)sk.p, (uint64_t*)sk2.p, (const uint32_t*)sv.p,
                                        (uint32_t*)sv2.p, (int)nc, 0, 32 + tb3);
        EBB_CUDA(c, cudaMalloc(&stmp.p, tbs));
        EBB_CUDA(c, cub::DeviceRadixSort::SortPairs(stmp.p, tbs, (const uint64_t*)sk.p, (uint64_t*)sk2.p,
                                                    (const uint32_t*)sv.p, (uint32_t*)sv2.p, (int)nc, 0, 32 + tb3));
        EBB_CUDA(c, cudaMalloc(&npos.p, nc * 4 + 16));
        EBB_CUDA(c, cudaMalloc(&cr2.p, nc * 4));
        EBB_CUDA(c, cudaMalloc(&ctr2.p, nc * 4));
        k_slot_newpos<<<grid_for(nc, 256), 256>>>(nc, (const uint32_t*)sv2.p, (uint32_t*)npos.p, P.crow, P.ctrow,
                                                  (uint32_t*)cr2.p, (uint32_t*)ctr2.p);
        k_remap_gci<<<grid_for(ne, 256), 256>>>(ne, (const uint32_t*)flag.p, (const uint32_t*)npos.p,
                                                (uint32_t*)gci.p);
        EBB_CUDA(c, cudaGetLastError());
        std::swap(P.crow, *(uint32_t**)&cr2.p);
        std::swap(P.ctrow, *(uint32_t**)&ctr2.p);
    }
    // instances: unique (tile, tet) over the 4 corners of every tet
    const uint64_t nk = nt * 4;
    EBB_CUDA(c, cudaMalloc(&keys.p, nk * 8));
    EBB_CUDA(c, cudaMalloc(&keys2.p, nk * 8));
    EBB_CUDA(c, cudaMalloc(&uk.p, nk * 8));
    EBB_CUDA(c, cudaMalloc(&nsel.p, 8));
    k_inst_keys<<<grid_for(nk, 256), 256>>>(nt, (const uint32_t*)V->ptr, nvt, (uint64_t*)keys.p);
    int tbits = 1;
    while (tbits < 32 && (1ull << tbits) <= P.ntiles) ++tbits;
    size_t tb1 = 0, tb2 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb1, (const uint64_t*)keys.p, (uint64_t*)keys2.p, (int)nk, 0, 32 + tbits);
    cub::DeviceSelect::Unique(nullptr, tb2, (const uint64_t*)keys2.p, (uint64_t*)uk.p, (int*)nsel.p, (int)nk);
    EBB_CUDA(c, cudaMalloc(&tmp2.p, tb1 > tb2 ? tb1 : tb2));
    EBB_CUDA(c, cub::DeviceRadixSort::SortKeys(tmp2.p, tb1, (const uint64_t*)keys.p, (uint64_t*)keys2.p, (int)nk, 0,
                                               32 + tbits));
    EBB_CUDA(c, cub::DeviceSelect::Unique(tmp2.p, tb2, (const uint64_t*)keys2.p, (uint64_t*)uk.p, (int*)nsel.p, (int)nk));
    int ni = 0;
    EBB_CUDA(c, cudaMemcpy(&ni, nsel.p, 4, cudaMemcpyDeviceToHost));
    P.ninst = (uint64_t)ni;
    EBB_CUDA(c, cudaMalloc(&P.inst_ptr, (P.ntiles + 1) * 4));
    k_inst_ptr<<<grid_for(P.ntiles + 1, 256), 256>>>((const uint64_t*)uk.p, P.ninst, P.inst_ptr, P.ntiles);
    uint32_t* rec_ptr = nullptr;
    uint64_t nrec = P.ninst;
    if (round > 0) {
        // gather: every tile padded to whole rounds; holes carry t = ~0
        DevBuf cnt, stmp;
        EBB_CUDA(c, cudaMalloc(&cnt.p, (P.ntiles + 1) * 4));
        EBB_CUDA(c, cudaMalloc(&rec_ptr, (P.ntiles + 1) * 4));
        k_round_counts<<<grid_for(P.ntiles + 1, 256), 256>>>(P.ntiles, P.inst_ptr, round, (uint32_t*)cnt.p);
        size_t tbs = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tbs, (const uint32_t*)cnt.p, rec_ptr, (int)(P.ntiles + 1));
        EBB_CUDA(c, cudaMalloc(&stmp.p, tbs));
        EBB_CUDA(c, cub::DeviceScan::ExclusiveSum(stmp.p, tbs, (const uint32_t*)cnt.p, rec_ptr, (int)(P.ntiles + 1)));
        uint32_t tot = 0;
        EBB_CUDA(c, cudaMemcpy(&tot, rec_ptr + P.ntiles, 4, cudaMemcpyDeviceToHost));
        nrec = tot;
    }
    EBB_CUDA(c, cudaMalloc(&P.recs, nrec * 32));
    if (round > 0) EBB_CUDA(c, cudaMemset(P.recs, 0xFF, nrec * 32));
    k_inst_records<<<grid_for(P.ninst, 256), 256>>>(P.ninst, (const uint64_t*)uk.p, (const uint32_t*)V->ptr,
                                                    (const uint32_t*)E->ptr, (const uint32_t*)gci.p, P.tile_cptr, nvt,
                                                    P.inst_ptr, rec_ptr, round, (uint32_t*)P.recs);
    if (round > 0) {
        EBB_CUDA(c, cudaDeviceSynchronize());
        cudaFree(P.inst_ptr);
        P.inst_ptr = rec_ptr;
        P.ninst = nrec;
    }
    EBB_CUDA(c, cudaMalloc(&mx.p, 4));
    EBB_CUDA(c, cudaMemset(mx.p, 0, 4));
    k_max_diff<<<grid_for(P.ntiles, 256), 256>>>(P.tile_cptr, P.ntiles, (unsigned int*)mx.p);
    EBB_CUDA(c, cudaGetLastError());
    EBB_CUDA(c, cudaMemcpy(&P.max_slots, mx.p, 4, cudaMemcpyDeviceToHost));
    if (P.max_slots >= 0xFFFFu) {
        P.release();
        return fail(c, EBB_E_RANGE, "tiled map: %u canonical rows in one tile (> 65534)", P.max_slots);
    }
    {
        ebb_status st = build_gather_lists(c, P, nv);
        if (st != EBB_OK) {
            P.release();
            return st;
        }
        if (round > 0) {
            k_gather_records<<<grid_for(P.ninst, 256), 256>>>(P.ninst, (const uint32_t*)V->ptr, (uint32_t*)P.recs);
            EBB_CUDA(c, cudaGetLastError());
        }
    }
    c->plans.push_back(P);
    *out = &c->plans.back();
    return EBB_OK;
}

// ---------------------------------------------------------------- TILED
template <typename R, int MODEL, bool WANT_E>
__global__ void __launch_bounds__(256) k_tet_map_tiled(
    uint32_t ntiles, int nvt, uint64_t nv, uint64_t nt, const uint32_t* __restrict__ inst_ptr,
    const uint4* __restrict__ recs, const uint32_t* __restrict__ tile_cptr, const uint32_t* __restrict__ crow,
    const uint32_t* __restrict__ ctrow, uint32_t max_slots, const uint4* __restrict__ tv, const R* __restrict__ u,
    const R* __restrict__ Dminv, const R* __restrict__ Wt, const R* __restrict__ mu_t, const R* __restrict__ lam_t,
    R* __restrict__ f, R* __restrict__ K, uint64_t ne, int accumulate, double* __restrict__ partials,
    unsigned int* __restrict__ counter, R* __restrict__ energy, unsigned long long* __restrict__ err) {
    extern __shared__ __align__(16) unsigned char tile_smem[];
    R* acc = reinterpret_cast<R*>(tile_smem);   // [max_slots][9]
    R* facc = acc + (size_t)max_slots * 9;       // [nvt][3]
    double e_acc = 0.0;
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint32_t c0 = tile_cptr[tile], ns = tile_cptr[tile + 1] - c0;
        const uint64_t v0 = (uint64_t)tile * nvt;
        const uint32_t nvl = (uint32_t)((v0 + nvt <= nv) ? nvt : nv - v0);
        for (uint32_t k = threadIdx.x; k < ns * 9; k += blockDim.x) acc[k] = R(0);
        for (uint32_t k = threadIdx.x; k < nvl * 3; k += blockDim.x) facc[k] = R(0);
        __syncthreads();
        const uint32_t i1 = inst_ptr[tile + 1];
        for (uint32_t i = inst_ptr[tile] + threadIdx.x; i < i1; i += blockDim.x) {
            const uint4 ra = recs[2ull * i], rb = recs[2ull * i + 1];
            const uint64_t t = ra.x;
            uint32_t v[4];
            R uu[4][3];
            TetState<R> st;
            load_tet(t, nt, tv, u, Dminv, Wt, mu_t, lam_t, v, uu, st);
            tet_physics<R, MODEL, true>(uu, st);
            const uint32_t flags = rb.w;
            if (MODEL == EBB_NH && (flags & 0x100u) && !(st.J > R(0))) atomicAdd(&err[ERR_INVERTED], 1ull);
            if (WANT_E && (flags & 0x100u)) e_acc += (double)(st.W * st.psi);
            R fi[4][3];
            tet_forces(st, fi);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t lv = (rb.z >> (8 * k)) & 0xFFu;
                if (lv != 0xFFu)
#pragma unroll
                    for (int a = 0; a < 3; ++a) atomicAdd(&facc[3 * lv + a], fi[k][a]);
            }
            const uint32_t sw[5] = {ra.y, ra.z, ra.w, rb.x, rb.y};
#pragma unroll
            for (int p = 0; p < 10; ++p) {
                const uint32_t slot = (sw[p / 2] >> (16 * (p & 1))) & 0xFFFFu;
                if (slot == 0xFFFFu) continue;
                const int bi = p < 6 ? (p < 3 ? 0 : (p < 5 ? 1 : 2)) : p - 6;
                const int bj = p < 6 ? (p < 3 ? p + 1 : (p < 5 ? p - 1 : 3)) : p - 6;
                R Kb[3][3];
                tet_block<R, MODEL>(st, bi, bj, Kb);
                R* as = acc + 9 * slot;
                if (p >= 6) {
                    // symmetric diagonal block: upper triangle only, mirrored at the flush
                    atomicAdd(as + 0, Kb[0][0]);
                    atomicAdd(as + 1, Kb[0][1]);
                    atomicAdd(as + 2, Kb[0][2]);
                    atomicAdd(as + 4, Kb[1][1]);
                    atomicAdd(as + 5, Kb[1][2]);
                    atomicAdd(as + 8, Kb[2][2]);
                } else if ((flags >> p) & 1u) {
#pragma unroll
                    for (int a = 0; a < 3; ++a)
#pragma unroll
                        for (int b = 0; b < 3; ++b) atomicAdd(as + 3 * a + b, Kb[b][a]);
                } else {
#pragma unroll
                    for (int a = 0; a < 3; ++a)
#pragma unroll
                        for (int b = 0; b < 3; ++b) atomicAdd(as + 3 * a + b, Kb[a][b]);
                }
            }
        }
        __syncthreads();
        // flush: canonical row (a,b) and its transpose (b,a), each written once
        for (uint32_t s = threadIdx.x; s < ns; s += blockDim.x) {
            const uint32_t r = crow[c0 + s], rt = ctrow[c0 + s];
            const R* as = acc + 9 * s;
            R blk[9];
#pragma unroll
            for (int c = 0; c < 9; ++c) blk[c] = as[c];
            if (rt == r) {
                blk[3] = blk[1];
                blk[6] = blk[2];
                blk[7] = blk[5];
            }
#pragma unroll
            for (int c = 0; c < 9; ++c) {
                R* dst = K + (uint64_t)c * ne + r;
                *dst = accumulate ? *dst + blk[c] : blk[c];
            }
            if (rt != r) {
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int b = 0; b < 3; ++b) {
                        R* dst = K + (uint64_t)(3 * a + b) * ne + rt;
                        *dst = accumulate ? *dst + blk[3 * b + a] : blk[3 * b + a];
                    }
            }
        }
        for (uint32_t k = threadIdx.x; k < nvl * 3; k += blockDim.x) {
            R* dst = f + 3 * v0 + k;
            *dst = accumulate ? *dst + facc[k] : facc[k];
        }
        __syncthreads();
    }
    if (WANT_E) {
        double tot;
        if (block_sum_last_done(e_acc, partials, counter, &tot)) *energy = (R)((double)*energy + tot);
    }
}


// ---------------------------------------------------------------- GATHER
// Atomic-free owner-computes map, entirely on chip.  Per tile (persistent CTA
// loop), the tile's instances are processed in rounds of ROUND (= blockDim):
//  phase 1  one thread per instance: element physics, then a compact state
//           row stored column-wise in shared memory (NH: k_i = F^-T g_i,
//           W mu m_ij per pair, W c1, W lam, f_i;  StVK: h_i = F g_i, W s_ij,
//           W mu m_ij per pair, F F^T, W mu, W lam, f_i);
//  phase 2  one owner thread per canonical row walks that row's contribution
//           list from its cursor up to the end of the round (lists are sorted
//           by instance), rebuilds each 3x3 block from the state (closed
//           rank-1 forms) and adds it to the row's shared accumulator with a
//           plain read-modify-write (the owner is the only writer).  One owner
//           thread per tile vertex does the same for the forces.
// After the last round every row and its transpose are written once.
// Deterministic (fixed list order, no atomics); shared traffic per instance
// is ~SW stores + ~10 row reads instead of ~90 atomic read-modify-writes.
template <int MODEL>
struct GState;
template <>
struct GState<EBB_NH> {   // [kv 12][cm 10][W c1][W lam][f 12]
    static constexpr int KV = 0, CM = 12, C1 = 22, CL = 23, F = 24, SW = 36;
};
template <>
struct GState<EBB_STVK> { // [kv 12][ws 10][wm 10][B 6][W mu][W lam][f 12]
    static constexpr int KV = 0, WS = 12, WM = 22, B = 32, CH = 38, CL = 39, F = 40, SW = 52;
};

// instances per round (= producer threads; consumers fill the CTA to 512):
// the double-buffered state of StVK in fp64 only fits at 128 (+128 consumers)
int gather_round(ebb_dtype dt, int model) {
    if (dt == EBB_F64 && model == EBB_STVK) return 128;
    const char* e = getenv("EBB_GATHER_NR");
    const int v = e ? atoi(e) : 0;
    if (v == 128 || v == 192 || v == 256) return v;
    return (dt == EBB_F64 && model == EBB_NH) ? 192 : 256;   // measured
}

// Adds one stored block (entry = (li << 8) | (i << 6) | (j << 4) | pair) to
// acc:  K_ij = W [ mu m_ij I + c1 k_j k_i^T + lam k_i k_j^T ]  (NH),
//       K_ij = W [ s_ij I + mu (m_ij F F^T + h_j h_i^T) + lam h_i h_j^T ]  (StVK).
template <typename R, int MODEL, int NR>
__device__ __forceinline__ void gather_block(const R* __restrict__ st, uint32_t ent, uint32_t r0, R acc[9]) {
    using G = GState<MODEL>;
    const uint32_t lr = (ent >> 8) - r0, i = (ent >> 6) & 3u, j = (ent >> 4) & 3u, p = ent & 15u;
    const R* si = st + (G::KV + 3 * i) * NR + lr;
    const R* sj = st + (G::KV + 3 * j) * NR + lr;
    const R ki[3] = {si[0], si[NR], si[2 * NR]};
    const R kj[3] = {sj[0], sj[NR], sj[2 * NR]};
    R ca, cb, cc, cd = R(0), Bm[6];
    if (MODEL == EBB_NH) {
        ca = st[(GState<EBB_NH>::CM + p) * NR + lr];
        cb = st[GState<EBB_NH>::C1 * NR + lr];
        cc = st[GState<EBB_NH>::CL * NR + lr];
    } else {
        using S = GState<EBB_STVK>;
        ca = st[(S::WS + p) * NR + lr];
        cb = st[S::CH * NR + lr];
        cc = st[S::CL * NR + lr];
        cd = st[(S::WM + p) * NR + lr];
#pragma unroll
        for (int k = 0; k < 6; ++k) Bm[k] = st[(S::B + k) * NR + lr];
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            R val = cb * kj[a] * ki[b] + cc * ki[a] * kj[b];
            if (a == b) val += ca;
            if (MODEL != EBB_NH) {
                constexpr int bidx[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
                val += cd * Bm[bidx[a][b]];
            }
            acc[3 * a + b] += val;
        }
}

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Warp-specialized: NR producer threads compute the element state of round g
// (NR instances) into buffer g&1 while NC consumer threads walk the rows for
// round g-1.  Named barriers 1,2 = "buffer b full", 3,4 = "buffer b empty",
// 5 = consumers only.
template <typename R, int MODEL, bool WANT_E, int NR, int NC>
__global__ void __launch_bounds__(NR + NC, 1) k_tet_map_gather(
    uint32_t ntiles, int nvt, uint64_t nv, uint64_t nt, const uint32_t* __restrict__ inst_ptr,
    const uint4* __restrict__ recs, const uint32_t* __restrict__ tile_cptr, const uint32_t* __restrict__ crow,
    const uint32_t* __restrict__ ctrow, const uint32_t* __restrict__ slot_ptr, const uint32_t* __restrict__ slot_ent,
    const uint32_t* __restrict__ fv_ptr, const uint32_t* __restrict__ fv_ent, uint32_t max_slots,
    uint32_t max_sent, const uint4* __restrict__ tv, const R* __restrict__ u, const R* __restrict__ Dminv,
    const R* __restrict__ Wt, const R* __restrict__ mu_t, const R* __restrict__ lam_t, R* __restrict__ f,
    R* __restrict__ K, uint64_t ne, int accumulate, double* __restrict__ partials, unsigned int* __restrict__ counter,
    R* __restrict__ energy, unsigned long long* __restrict__ err) {
    using G = GState<MODEL>;
    constexpr int NT = NR + NC;
    extern __shared__ __align__(16) unsigned char tile_smem[];
    R* stb = reinterpret_cast<R*>(tile_smem);              // [2][SW][NR]
    R* acc = stb + 2 * (size_t)G::SW * NR;                  // [max_slots][9]
    R* facc = acc + (size_t)max_slots * 9;                  // [nvt][3]
    uint32_t* cur = reinterpret_cast<uint32_t*>(facc + (size_t)nvt * 3);   // [max_slots]
    uint32_t* cend = cur + max_slots;                                         // [max_slots]
    uint32_t* fcur = cend + max_slots;                                        // [nvt]
    uint32_t* fend = fcur + nvt;                                              // [nvt]
    uint32_t* sent = fend + nvt;                                              // [max_sent]
    uint32_t* fent = sent + max_sent;                                         // [max_fent]
    double e_acc = 0.0;
    const bool producer = threadIdx.x < NR;
    const uint32_t tid = producer ? threadIdx.x : threadIdx.x - NR;
    uint32_t g = 0;   // global round counter of this CTA
    if (producer) {
        for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const uint32_t i0 = inst_ptr[tile], ni = inst_ptr[tile + 1] - i0;
            for (uint32_t r0 = 0; r0 < ni; r0 += NR, ++g) {
                const int b = g & 1;
                const uint32_t li = r0 + tid;
                const uint4 ra = li < ni ? recs[2ull * (i0 + li)] : make_uint4(~0u, 0, 0, 0);
                const bool live = ra.x != 0xFFFFFFFFu;   // padded rounds: holes carry t = ~0
                uint4 rb = make_uint4(0, 0, 0, 0);
                R uu[4][3];
                TetState<R> ts;
                if (live) {
                    // record = (t, v0..v3, flags): all input loads issue now and
                    // land while the producer waits for its buffer
                    rb = recs[2ull * (i0 + li) + 1];
                    const uint64_t t = ra.x;
                    const uint32_t v[4] = {ra.y, ra.z, ra.w, rb.x};
#pragma unroll
                    for (int k = 0; k < 4; ++k)
#pragma unroll
                        for (int a = 0; a < 3; ++a) uu[k][a] = u[3ull * v[k] + a];
#pragma unroll
                    for (int r = 0; r < 3; ++r)
#pragma unroll
                        for (int c = 0; c < 3; ++c) ts.g[r + 1][c] = Dminv[(uint64_t)(3 * r + c) * nt + t];
                    ts.W = Wt[t];
                    ts.mu = mu_t[t];
                    ts.lam = lam_t[t];
                }
                if (g >= 2) named_sync(3 + b, NT);   // consumers released buffer b
                if (live) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) ts.g[0][c] = -(ts.g[1][c] + ts.g[2][c] + ts.g[3][c]);
                    tet_physics<R, MODEL, true>(uu, ts);
                    const uint32_t flags = rb.w;
                    if (MODEL == EBB_NH && (flags & 0x100u) && !(ts.J > R(0))) atomicAdd(&err[ERR_INVERTED], 1ull);
                    if (WANT_E && (flags & 0x100u)) e_acc += (double)(ts.W * ts.psi);
                    R fi[4][3];
                    tet_forces(ts, fi);
                    R* sr = stb + (size_t)b * G::SW * NR + tid;
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            sr[(G::KV + 3 * i + a) * NR] = ts.kv[i][a];
                            sr[(G::F + 3 * i + a) * NR] = fi[i][a];
                        }
#pragma unroll
                    for (int p = 0; p < 10; ++p) {
                        const int i = p < 6 ? (p < 3 ? 0 : (p < 5 ? 1 : 2)) : p - 6;
                        const int j = p < 6 ? (p < 3 ? p + 1 : (p < 5 ? p - 1 : 3)) : p - 6;
                        const R mij = ts.g[i][0] * ts.g[j][0] + ts.g[i][1] * ts.g[j][1] + ts.g[i][2] * ts.g[j][2];
                        if (MODEL == EBB_NH) {
                            sr[(GState<EBB_NH>::CM + p) * NR] = ts.W * ts.mu * mij;
                        } else {
                            R Sg[3];
#pragma unroll
                            for (int a = 0; a < 3; ++a)
                                Sg[a] = ts.S[a][0] * ts.g[i][0] + ts.S[a][1] * ts.g[i][1] + ts.S[a][2] * ts.g[i][2];
                            sr[(GState<EBB_STVK>::WS + p) * NR] =
                                ts.W * (Sg[0] * ts.g[j][0] + Sg[1] * ts.g[j][1] + Sg[2] * ts.g[j][2]);
                            sr[(GState<EBB_STVK>::WM + p) * NR] = ts.W * ts.mu * mij;
                        }
                    }
                    if (MODEL == EBB_NH) {
                        sr[GState<EBB_NH>::C1 * NR] = ts.W * ts.c1;
                        sr[GState<EBB_NH>::CL * NR] = ts.W * ts.lam;
                    } else {
                        constexpr int B = GState<EBB_STVK>::B;
                        sr[(B + 0) * NR] = ts.B[0][0];
                        sr[(B + 1) * NR] = ts.B[0][1];
                        sr[(B + 2) * NR] = ts.B[0][2];
                        sr[(B + 3) * NR] = ts.B[1][1];
                        sr[(B + 4) * NR] = ts.B[1][2];
                        sr[(B + 5) * NR] = ts.B[2][2];
                        sr[GState<EBB_STVK>::CH * NR] = ts.W * ts.mu;
                        sr[GState<EBB_STVK>::CL * NR] = ts.W * ts.lam;
                    }
                }
                named_arrive(1 + b, NT);   // buffer b full
            }
        }
        // drain: match the consumers' releases of the last two rounds
        if (g >= 2) named_sync(3 + (g & 1), NT);
        if (g >= 1) named_sync(3 + ((g + 1) & 1), NT);
    } else {
        for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const uint32_t ni = inst_ptr[tile + 1] - inst_ptr[tile];
            const uint32_t c0 = tile_cptr[tile], ns = tile_cptr[tile + 1] - c0;
            const uint64_t v0 = (uint64_t)tile * nvt;
            const uint32_t nvl = (uint32_t)((v0 + nvt <= nv) ? nvt : nv - v0);
            // stage the tile's contribution lists in shared memory (all
            // consumers are past the previous tile's walks first)
            const uint32_t eb = slot_ptr[c0], ee = slot_ptr[c0 + ns];
            const uint32_t fb = fv_ptr[v0], fe = fv_ptr[v0 + nvl];
            named_sync(5, NC);
            for (uint32_t k = tid; k < ee - eb; k += NC) sent[k] = __ldg(slot_ent + eb + k);
            for (uint32_t k = tid; k < fe - fb; k += NC) fent[k] = __ldg(fv_ent + fb + k);
            // every row / vertex is owned by one consumer thread
            for (uint32_t s = tid; s < ns; s += NC) {
                cur[s] = slot_ptr[c0 + s] - eb;
                cend[s] = slot_ptr[c0 + s + 1] - eb;
#pragma unroll
                for (int k = 0; k < 9; ++k) acc[9 * s + k] = R(0);
            }
            for (uint32_t lv = tid; lv < nvl; lv += NC) {
                fcur[lv] = fv_ptr[v0 + lv] - fb;
                fend[lv] = fv_ptr[v0 + lv + 1] - fb;
                facc[3 * lv] = facc[3 * lv + 1] = facc[3 * lv + 2] = R(0);
            }
            named_sync(5, NC);
            for (uint32_t r0 = 0; r0 < ni; r0 += NR, ++g) {
                const int b = g & 1;
                named_sync(1 + b, NT);   // wait: buffer b full
                const R* st = stb + (size_t)b * G::SW * NR;
                const uint32_t rend = r0 + NR;   // instances of this round: li in [r0, rend)
                // slots are numbered by descending list length; deal them
                // snake-wise (k even: tid, k odd: NC-1-tid) for balance
                for (uint32_t k = 0; k * NC < ns; ++k) {
                    const uint32_t s = k * NC + ((k & 1) ? NC - 1 - tid : tid);
                    if (s >= ns) continue;
                    const uint32_t e1 = cend[s];
                    uint32_t e = cur[s];
                    R a9[9];
#pragma unroll
                    for (int q = 0; q < 9; ++q) a9[q] = R(0);
                    for (; e < e1; ++e) {
                        const uint32_t en = sent[e];
                        if ((en >> 8) >= rend) break;
                        gather_block<R, MODEL, NR>(st, en, r0, a9);
                    }
                    cur[s] = e;
#pragma unroll
                    for (int q = 0; q < 9; ++q) acc[9 * s + q] += a9[q];
                }
                for (uint32_t lv = NC - 1 - tid; lv < nvl; lv += NC) {
                    const uint32_t e1 = fend[lv];
                    uint32_t e = fcur[lv];
                    R f0 = 0, f1 = 0, f2 = 0;
                    for (; e < e1; ++e) {
                        const uint32_t en = fent[e];
                        if ((en >> 2) >= rend) break;
                        const uint32_t lr = (en >> 2) - r0, k = en & 3u;
                        f0 += st[(G::F + 3 * k + 0) * NR + lr];
                        f1 += st[(G::F + 3 * k + 1) * NR + lr];
                        f2 += st[(G::F + 3 * k + 2) * NR + lr];
                    }
                    fcur[lv] = e;
                    facc[3 * lv] += f0;
                    facc[3 * lv + 1] += f1;
                    facc[3 * lv + 2] += f2;
                }
                named_arrive(3 + b, NT);   // buffer b empty
            }
            // flush: every canonical row and its transpose, then the forces
            // (rows were accumulated by their dealt owners: consumer barrier)
            named_sync(5, NC);
            for (uint32_t s = tid; s < ns; s += NC) {
                const uint32_t gs = c0 + s;
                const uint32_t r = crow[gs], rt = ctrow[gs];
                const R* a9 = acc + 9 * s;
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    R* dst = K + (uint64_t)k * ne + r;
                    *dst = accumulate ? *dst + a9[k] : a9[k];
                }
                if (rt != r) {
#pragma unroll
                    for (int a = 0; a < 3; ++a)
#pragma unroll
                        for (int bb = 0; bb < 3; ++bb) {
                            R* dst = K + (uint64_t)(3 * a + bb) * ne + rt;
                            *dst = accumulate ? *dst + a9[3 * bb + a] : a9[3 * bb + a];
                        }
                }
            }
            for (uint32_t lv = tid; lv < nvl; lv += NC) {
                R* dst = f + 3 * (v0 + lv);
#pragma unroll
                for (int a = 0; a < 3; ++a) dst[a] = accumulate ? dst[a] + facc[3 * lv + a] : facc[3 * lv + a];
            }
        }
    }
    if (WANT_E) {
        double tot;
        if (block_sum_last_done(e_acc, partials, counter, &tot)) *energy = (R)((double)*energy + tot);
    }
}

template <typename R, int MODEL>
size_t gather_smem(const MapPlan& P) {
    return 2 * (size_t)GState<MODEL>::SW * P.round * sizeof(R) + ((size_t)P.max_slots * 9 + (size_t)P.nvt * 3) * sizeof(R) +
           2 * ((size_t)P.max_slots + P.nvt) * 4 + ((size_t)P.max_sent + P.max_fent) * 4;
}

template <typename R, int MODEL, int NR, int NC>
ebb_status launch_gather_split(Ctx* c, const MapPlan& P, bool want_e, int accumulate, uint64_t nt, uint64_t nv,
                               const Field* V, const Field* U, const Field* D, const Field* W, const Field* MU,
                               const Field* LA, const Field* Fo, const Field* Ko, uint64_t ne, const Field* En,
                               cudaStream_t s) {
    const size_t smem = gather_smem<R, MODEL>(P);
    auto kern = want_e ? k_tet_map_gather<R, MODEL, true, NR, NC> : k_tet_map_gather<R, MODEL, false, NR, NC>;
    static thread_local size_t configured_dev[kMaxDevices][2] = {};
    size_t* const configured = configured_dev[c->device % kMaxDevices];   // attribute set once (graph-capture safe)
    if (smem > configured[want_e]) {
        EBB_CUDA(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured[want_e] = smem;
    }
    unsigned grid = occ_grid(c, kern, NR + NC, smem, (uint64_t)P.ntiles * (NR + NC));
    KernelTimer kt(c, EBB_K_TET_MAP, s);
    kern<<<grid, NR + NC, smem, s>>>(P.ntiles, P.nvt, nv, nt, P.inst_ptr, P.recs, P.tile_cptr, P.crow, P.ctrow,
                                     P.slot_ptr, P.slot_ent, P.fv_ptr, P.fv_ent, P.max_slots, P.max_sent,
                                     (const uint4*)V->ptr, (const R*)U->ptr, (const R*)D->ptr, (const R*)W->ptr,
                                     (const R*)MU->ptr, (const R*)LA->ptr, (R*)Fo->ptr, (R*)Ko->ptr, ne, accumulate,
                                     c->d_partials, c->d_counter + 0, En ? (R*)En->ptr : nullptr, c->d_err);
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

template <typename R, int MODEL>
ebb_status launch_gather(Ctx* c, const MapPlan& P, bool want_e, int accumulate, uint64_t nt, uint64_t nv,
                         const Field* V, const Field* U, const Field* D, const Field* W, const Field* MU,
                         const Field* LA, const Field* Fo, const Field* Ko, uint64_t ne, const Field* En,
                         cudaStream_t s) {
#define EBB_GARGS c, P, want_e, accumulate, nt, nv, V, U, D, W, MU, LA, Fo, Ko, ne, En, s
    if constexpr (MODEL == EBB_STVK && sizeof(R) == 8) {   // state only fits at 128 instances per round
        return launch_gather_split<R, MODEL, 128, 384>(EBB_GARGS);
    } else {
        if (P.round == 128) return launch_gather_split<R, MODEL, 128, 384>(EBB_GARGS);
        if (P.round == 192) return launch_gather_split<R, MODEL, 192, 320>(EBB_GARGS);
        return launch_gather_split<R, MODEL, 256, 256>(EBB_GARGS);
    }
#undef EBB_GARGS
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

template <typename R, int MODEL>
ebb_status launch_tiled(Ctx* c, const MapPlan& P, bool want_e, int accumulate, uint64_t nt, uint64_t nv,
                        const Field* V, const Field* U, const Field* D, const Field* W, const Field* MU,
                        const Field* LA, const Field* Fo, const Field* Ko, uint64_t ne, const Field* En,
                        cudaStream_t s) {
    const int block = 256;
    const size_t smem = ((size_t)P.max_slots * 9 + (size_t)P.nvt * 3) * sizeof(R);
    auto kern = want_e ? k_tet_map_tiled<R, MODEL, true> : k_tet_map_tiled<R, MODEL, false>;
    static thread_local size_t configured_dev[kMaxDevices][2] = {};
    size_t* const configured = configured_dev[c->device % kMaxDevices];   // attribute set once (graph-capture safe)
    if (smem > configured[want_e]) {
        EBB_CUDA(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured[want_e] = smem;
    }
    unsigned grid = occ_grid(c, kern, block, smem, (uint64_t)P.ntiles * block);
    KernelTimer kt(c, EBB_K_TET_MAP, s);
    kern<<<grid, block, smem, s>>>(P.ntiles, P.nvt, nv, nt, P.inst_ptr, P.recs, P.tile_cptr, P.crow, P.ctrow,
                                   P.max_slots, (const uint4*)V->ptr, (const R*)U->ptr, (const R*)D->ptr,
                                   (const R*)W->ptr, (const R*)MU->ptr, (const R*)LA->ptr, (R*)Fo->ptr, (R*)Ko->ptr,
                                   ne, accumulate, c->d_partials, c->d_counter + 0, En ? (R*)En->ptr : nullptr,
                                   c->d_err);
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

int tile_env() {
    const char* e = getenv("EBB_TILE_VERTS");
    return (e && atoi(e) > 0 && atoi(e) <= 255) ? atoi(e) : 0;
}

int tile_vertices(ebb_dtype dt) {
    if (tile_env()) return tile_env();
    return dt == EBB_F64 ? 128 : 192;
}

size_t gather_smem_for(const MapPlan& P, ebb_dtype dt, int model) {
    if (dt == EBB_F64) return model == EBB_NH ? gather_smem<double, EBB_NH>(P) : gather_smem<double, EBB_STVK>(P);
    return model == EBB_NH ? gather_smem<float, EBB_NH>(P) : gather_smem<float, EBB_STVK>(P);
}

// gather: the largest tile (from a per-type start) whose double-buffered
// element state, row accumulators and staged lists fit in shared memory
ebb_status gather_plan(Ctx* c, ebb_field vf, ebb_field ef, ebb_dtype dt, int model, MapPlan** out) {
    const size_t limit = 227 * 1024;
    int nvt = tile_env();
    const bool forced = nvt != 0;
    if (!forced) nvt = dt == EBB_F64 ? (model == EBB_NH ? 64 : 96) : (model == EBB_NH ? 160 : 128);
    for (;;) {
        MapPlan* P;
        EBB_TRY(build_plan(c, vf, ef, nvt, gather_round(dt, model), &P));
        const size_t need = gather_smem_for(*P, dt, model);
        if (need <= limit) {
            *out = P;
            return EBB_OK;
        }
        if (forced || nvt <= 4)
            return fail(c, EBB_E_RANGE, "gather map: a %d-vertex tile needs %zu B of shared memory", nvt, need);
        for (size_t k = 0; k < c->plans.size(); ++k)   // drop the unusable plan
            if (&c->plans[k] == P) {
                c->plans[k].release();
                c->plans.erase(c->plans.begin() + k);
                break;
            }
        nvt = nvt * 3 / 4;
    }
}

}  // namespace

extern "C" ebb_status ebb_map_tet_forces(ebb_ctx ctx, const ebb_tet_map_desc* d, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !d) return fail(c, EBB_E_ARG, "null argument");
    if (d->model != EBB_STVK && d->model != EBB_NH) return fail(c, EBB_E_ARG, "unknown model %d", d->model);
    if (d->scatter < EBB_SCATTER_AUTO || d->scatter > EBB_SCATTER_CHUNK)
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
    if (Ko && strat == EBB_SCATTER_CHUNK) {
        // every K row and f row is written exactly once: zero_outputs means overwrite
        if (d->zero_outputs && En) EBB_CUDA(c, cudaMemsetAsync(En->ptr, 0, dtype_size(dt), s));
        return chunk_map_launch(c, d->v, d->e, d->model, En != nullptr, d->zero_outputs ? 0 : 1, nt, V, U, D, W, MU,
                                LA, Fo, Ko, ne, En, s);
    }
    if (Ko && strat == EBB_SCATTER_SEGMENTED) {
        // every K row and f row is written exactly once: zero_outputs means overwrite
        if (d->zero_outputs && En) EBB_CUDA(c, cudaMemsetAsync(En->ptr, 0, dtype_size(dt), s));
        return seg_map_launch(c, d->v, d->e, d->model, En != nullptr, d->zero_outputs ? 0 : 1, nt, V, U, D, W, MU, LA,
                              Fo, Ko, ne, En, s);
    }
    const bool tiled = Ko && (strat == EBB_SCATTER_TILED || strat == EBB_SCATTER_GATHER);
    if (tiled) {
        // every K row and f row is written exactly once: zero_outputs means overwrite
        const bool gather = strat == EBB_SCATTER_GATHER;
        MapPlan* P;
        if (gather) EBB_TRY(gather_plan(c, d->v, d->e, dt, d->model, &P));
        else EBB_TRY(build_plan(c, d->v, d->e, tile_vertices(dt), 0, &P));
        V = get_field(c, d->v); U = get_field(c, d->u); D = get_field(c, d->Dminv); W = get_field(c, d->W);
        MU = get_field(c, d->mu); LA = get_field(c, d->lam); Fo = get_field(c, d->f); Ko = get_field(c, d->K);
        En = d->energy == EBB_NONE ? nullptr : get_field(c, d->energy);
        if (d->zero_outputs && En) EBB_CUDA(c, cudaMemsetAsync(En->ptr, 0, dtype_size(dt), s));
        int accum = d->zero_outputs ? 0 : 1;
        bool we = En != nullptr;
        if (gather) {
            if (dt == EBB_F64) {
                if (d->model == EBB_NH)
                    return launch_gather<double, EBB_NH>(c, *P, we, accum, nt, nv, V, U, D, W, MU, LA, Fo, Ko, ne, En, s);
                return launch_gather<double, EBB_STVK>(c, *P, we, accum, nt, nv, V, U, D, W, MU, LA, Fo, Ko, ne, En, s);
            }
            if (d->model == EBB_NH)
                return launch_gather<float, EBB_NH>(c, *P, we, accum, nt, nv, V, U, D, W, MU, LA, Fo, Ko, ne, En, s);
            return launch_gather<float, EBB_STVK>(c, *P, we, accum, nt, nv, V, U, D, W, MU, LA, Fo, Ko, ne, En, s);
        }
        if (dt == EBB_F64) {
            if (d->model == EBB_NH)
                return launch_tiled<double, EBB_NH>(c, *P, we, accum, nt, nv, V, U, D, W, MU, LA, Fo, Ko, ne, En, s);
            return launch_tiled<double, EBB_STVK>(c, *P, we, accum, nt, nv, V, U, D, W, MU, LA, Fo, Ko, ne, En, s);
        }
        if (d->model == EBB_NH)
            return launch_tiled<float, EBB_NH>(c, *P, we, accum, nt, nv, V, U, D, W, MU, LA, Fo, Ko, ne, En, s);
        return launch_tiled<float, EBB_STVK>(c, *P, we, accum, nt, nv, V, U, D, W, MU, LA, Fo, Ko, ne, En, s);
    }
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
