// seg_plan.cu -- the SEGMENTED map's plan built on the device (SURVEY §8(a)
// a1/a6-a7: the segmented reduction of P:721-731 / P:856-871 planned once per
// mesh).  Produces the same arrays as the host builder in seg_map.cu (same
// tiles, instance order, entry order, chunk layout and bank schedule), so the
// two plans are interchangeable word for word (EBB_SEG_PLAN=host selects the
// host one; tests compare the results bitwise):
//   1. vertex -> incident tets (CUB radix sort of the 4T (vertex, tet) pairs)
//   2. self row and canonical-row count of every vertex
//   3. tiles: greedy within blocks of kSegBlock consecutive vertices (one
//      thread per block; a tile never crosses a block boundary)
//   4. instances: unique (tile, tet) pairs (64-bit radix sort + unique)
//   5. entries: the 10 blocks of every tet keyed (tile, kind, slot, instance,
//      pair) and sorted; per-tile lists padded to 4 words
//   6. items: one thread per tile (chunk length L chosen as on the host),
//      bank schedule one thread per warp of items
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <vector>

#include "ebb_internal.cuh"
#include "seg_common.cuh"

namespace ebb {
namespace {

struct DBuf {
    void* p = nullptr;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { cudaFree(p); }
    void reset() {
        cudaFree(p);
        p = nullptr;
    }
    cudaError_t alloc(size_t b) { return cudaMalloc(&p, b + 16); }
    template <typename T>
    T* as() const { return (T*)p; }
};

__device__ __forceinline__ uint32_t lbound(const uint32_t* a, uint32_t lo, uint32_t hi, uint32_t x) {
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void ksp_vt_pairs(const uint32_t* __restrict__ tv, uint64_t n4, uint32_t* __restrict__ key,
                             uint32_t* __restrict__ val) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n4) return;
    key[i] = tv[i];
    val[i] = (uint32_t)(i >> 2);
}

__global__ void ksp_ptr(const uint32_t* __restrict__ sorted, uint64_t n, uint32_t* __restrict__ ptr, uint64_t nv) {
    const uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (v > nv) return;
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (sorted[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    ptr[v] = (uint32_t)lo;
}

// self row of every vertex; its number of canonical rows (tail <= head)
__global__ void ksp_rself(uint64_t nv, const uint32_t* __restrict__ index, const uint32_t* __restrict__ head,
                          uint32_t* __restrict__ rself, uint32_t* __restrict__ ccount, unsigned int* __restrict__ bad) {
    const uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (v >= nv) return;
    const uint32_t r = lbound(head, index[v], index[v + 1], (uint32_t)v);
    if (r >= index[v + 1] || head[r] != v) atomicOr(bad, 1u);
    rself[v] = r;
    ccount[v] = index[v + 1] - r;
}

// greedy tiles inside one block of consecutive vertices (thread = block):
// a tet is new to the tile iff none of its other vertices joined the tile
// already; a tile closes when the next vertex would push its instances past
// ni or it holds 4096 vertices
__global__ void ksp_tiles(uint64_t nv, uint32_t blk, int ni, const uint32_t* __restrict__ tv,
                          const uint32_t* __restrict__ vt_ptr, const uint32_t* __restrict__ vt,
                          uint32_t* __restrict__ starts, uint32_t* __restrict__ nstart, unsigned int* __restrict__ bad) {
    const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t v0 = b * blk;
    if (v0 >= nv) return;
    const uint64_t v1 = v0 + blk < nv ? v0 + blk : nv;
    uint32_t k = 0, ci = 0, cv = 0;
    uint64_t s = v0;
    for (uint64_t v = v0; v < v1; ++v) {
        const uint32_t deg = vt_ptr[v + 1] - vt_ptr[v];
        if (deg > (uint32_t)ni) atomicOr(bad, 2u);
        uint32_t nw = 0;
        for (uint32_t q = vt_ptr[v]; q < vt_ptr[v + 1]; ++q) {
            const uint32_t* tt = tv + 4ull * vt[q];
            bool old = false;
            for (int c = 0; c < 4; ++c) old |= tt[c] != v && tt[c] >= s && tt[c] < v;
            nw += !old;
        }
        if (cv == 0) {
            starts[v0 + k++] = (uint32_t)v;
            s = v;
            nw = deg;
        } else if (ci + nw > (uint32_t)ni || cv >= 4096) {
            starts[v0 + k++] = (uint32_t)v;
            s = v;
            ci = 0;
            cv = 0;
            nw = deg;
        }
        ci += nw;
        ++cv;
    }
    nstart[b] = k;
}

__global__ void ksp_compact_tiles(uint64_t nblk, uint32_t blk, const uint32_t* __restrict__ starts,
                                  const uint32_t* __restrict__ nstart, const uint32_t* __restrict__ off,
                                  uint32_t* __restrict__ tile_v) {
    const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (b >= nblk) return;
    for (uint32_t k = 0; k < nstart[b]; ++k) tile_v[off[b] + k] = starts[b * blk + k];
}

__global__ void ksp_tile_of(uint32_t ntiles, const uint32_t* __restrict__ tile_v, uint32_t* __restrict__ tile_of_v) {
    const uint64_t T = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (T >= ntiles) return;
    for (uint32_t v = tile_v[T]; v < tile_v[T + 1]; ++v) tile_of_v[v] = (uint32_t)T;
}

__global__ void ksp_inst_keys(uint64_t n4, const uint32_t* __restrict__ vkey, const uint32_t* __restrict__ vt,
                              const uint32_t* __restrict__ tile_of_v, uint64_t* __restrict__ key) {
    const uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (q < n4) key[q] = ((uint64_t)tile_of_v[vkey[q]] << 32) | vt[q];
}

// per tile: the number of sorted keys whose high bits (>> shift) equal the
// tile (two lower bounds in the sorted key array; no atomics)
__global__ void ksp_hist_hi(const uint64_t* __restrict__ k, uint64_t n, int shift, uint32_t* __restrict__ cnt,
                            uint32_t ntiles) {
    const uint64_t T = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (T >= ntiles) return;
    auto lb = [&](uint64_t x) {
        uint64_t lo = 0, hi = n;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if ((k[mid] >> shift) < x) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    cnt[T] = (uint32_t)(lb(T + 1) - lb(T));
}

// instance records (tet, slot | energy owner << 16); slot = position in the tile
__global__ void ksp_inst(uint64_t n, const uint64_t* __restrict__ ukey, const uint32_t* __restrict__ inst0,
                         const uint32_t* __restrict__ tv, const uint32_t* __restrict__ tile_of_v,
                         uint2* __restrict__ inst) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t T = (uint32_t)(ukey[k] >> 32), t = (uint32_t)ukey[k];
    const uint32_t l = (uint32_t)(k - inst0[T]);
    const uint32_t* vv = tv + 4ull * t;
    const uint32_t vmin = min(min(vv[0], vv[1]), min(vv[2], vv[3]));
    inst[k] = make_uint2(t, l | (tile_of_v[vmin] == T ? 1u << 16 : 0u));
}

// the 10 blocks of every instance whose canonical row lies in its tile
// key = tile[24] | kind[1] (0 self row, 1 off-diagonal) | slot[13] | l[9] | pair[4]
__global__ void ksp_entries(uint64_t ninst, const uint2* __restrict__ inst, const uint64_t* __restrict__ ukey,
                            int ni, const uint32_t* __restrict__ tv, const uint32_t* __restrict__ tile_of_v,
                            const uint32_t* __restrict__ tile_v, const uint32_t* __restrict__ index,
                            const uint32_t* __restrict__ head, const uint32_t* __restrict__ rself,
                            const uint32_t* __restrict__ cs, uint64_t* __restrict__ key, uint32_t* __restrict__ val,
                            unsigned long long* __restrict__ nout, uint32_t* __restrict__ slot_cnt) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= ninst) return;
    const uint32_t T = (uint32_t)(ukey[k] >> 32), t = inst[k].x, l = inst[k].y & 0xFFFFu;
    const uint32_t* vv = tv + 4ull * t;
    for (int p = 0; p < 10; ++p) {
        const int i = pair_i(p), j = pair_j(p);
        const uint32_t lo = min(vv[i], vv[j]), hi = max(vv[i], vv[j]);
        if (tile_of_v[lo] != T) continue;
        const uint32_t r = lbound(head, rself[lo], index[lo + 1], hi);
        const uint32_t slot = cs[lo] - cs[tile_v[T]] + (r - rself[lo]);
        const uint32_t bi = vv[i] <= vv[j] ? i : j, bj = vv[i] <= vv[j] ? j : i;
        const unsigned long long o = atomicAdd(nout, 1ull);
        const uint64_t kind = lo == hi ? 0u : 1u;
        key[o] = ((uint64_t)T << 27) | (kind << 26) | ((uint64_t)slot << 13) | ((uint64_t)l << 4) | (uint64_t)p;
        val[o] = (3 * bi * (uint32_t)ni + l) | ((3 * bj * (uint32_t)ni + l) << 13) | ((uint32_t)p << 26);
        atomicAdd(slot_cnt + cs[lo] + (r - rself[lo]), 1u);
    }
}

__global__ void ksp_pad4(uint32_t n, const uint32_t* __restrict__ c, uint32_t* __restrict__ p) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = (c[i] + 3u) & ~3u;
}

__global__ void ksp_place(uint64_t n, const uint64_t* __restrict__ key, const uint32_t* __restrict__ val,
                          const uint32_t* __restrict__ e0u, const uint32_t* __restrict__ e0p, uint32_t* __restrict__ ents) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t T = (uint32_t)(key[i] >> 27);
    ents[e0p[T] + (i - e0u[T])] = val[i];
}

// one tile's chunked item layout, as seg_map.cu's host layout()
struct TileSlots {
    const uint32_t *tile_v, *index, *head, *rself, *ccount, *cs, *slot_cnt;
    int ni;
};

__device__ uint32_t ksp_layout_one(const TileSlots& S, uint32_t T, uint32_t L, bool emit, uint4* out) {
    const uint32_t a = S.tile_v[T], b = S.tile_v[T + 1];
    uint32_t n = 0, beg = 0;
    auto pad = [&]() {
        while (n % 32) {
            if (emit) out[n] = make_uint4(0, 0xFFFFFFFFu, 0xFFFFFFFFu, 0);
            ++n;
        }
    };
    // kind 1 (self rows + forces) first, in vertex order; then kind 0 (off-diagonal) in slot order
    for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) pad();   // kinds start a warp
        uint32_t qi = 0;
        for (uint32_t v = a; v < b; ++v) {
            const uint32_t k0 = pass == 0 ? 0u : 1u, k1 = pass == 0 ? 1u : S.ccount[v];
            for (uint32_t kk = k0; kk < k1; ++kk, ++qi) {
                const uint32_t cnt = S.slot_cnt[S.cs[v] + kk];
                const uint32_t nc = cnt == 0 ? 1u : (cnt + L - 1) / L;
                if ((n % 32) + nc > 32) pad();
                const uint32_t r = S.rself[v] + kk;
                uint32_t bb = beg;
                for (uint32_t cc = 0; cc < nc; ++cc, ++n) {
                    const uint32_t sz = cnt / nc + (cc < cnt % nc ? 1u : 0u);
                    if (emit) {
                        const uint32_t kind = pass == 0 ? 1u : 0u;
                        const uint32_t meta = bb | (sz << 16) | (cc << 23) | ((nc - 1) << 26) | (kind << 29);
                        if (kind == 1) {
                            out[n] = make_uint4(meta, r, v, 0);
                        } else {
                            const uint32_t hd = S.head[r];
                            out[n] = make_uint4(meta, r, lbound(S.head, S.index[hd], S.index[hd + 1], v), 0);
                        }
                    }
                    bb += sz;
                }
                beg += cnt;
            }
        }
    }
    pad();
    return n;
}

__global__ void ksp_layout_count(TileSlots S, uint32_t ntiles, uint32_t* __restrict__ tileL,
                                 uint32_t* __restrict__ nitems, unsigned int* __restrict__ bad) {
    const uint64_t T = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (T >= ntiles) return;
    uint64_t tot = 0, longest = 0;
    for (uint32_t v = S.tile_v[T]; v < S.tile_v[T + 1]; ++v)
        for (uint32_t kk = 0; kk < S.ccount[v]; ++kk) {
            const uint32_t c = S.slot_cnt[S.cs[v] + kk];
            tot += c;
            longest = longest > c ? longest : c;
        }
    const uint64_t ni = (uint64_t)S.ni;
    uint64_t L0 = (tot + ni - 1) / ni;
    L0 = L0 > 2 ? L0 : 2;
    L0 = L0 > (longest + 7) / 8 ? L0 : (longest + 7) / 8;
    const uint64_t Lcap = L0 > (4 * L0 < 127 ? 4 * L0 : 127) ? L0 : (4 * L0 < 127 ? 4 * L0 : 127);
    uint64_t L = L0;
    while (L < Lcap && L < longest && ksp_layout_one(S, (uint32_t)T, (uint32_t)L, false, nullptr) > ni) ++L;
    if (L > 127) {
        atomicOr(bad, 4u);
        L = 127;
    }
    tileL[T] = (uint32_t)L;
    nitems[T] = ksp_layout_one(S, (uint32_t)T, (uint32_t)L, false, nullptr);
}

__global__ void ksp_layout_emit(TileSlots S, uint32_t ntiles, const uint32_t* __restrict__ tileL,
                                const uint32_t* __restrict__ item0, uint4* __restrict__ items) {
    const uint64_t T = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (T >= ntiles) return;
    ksp_layout_one(S, (uint32_t)T, tileL[T], true, items + item0[T]);
}

// warp group g -> its tile (items of a tile are whole warps)
__global__ void ksp_group_tile(uint32_t ntiles, const uint32_t* __restrict__ item0, uint32_t* __restrict__ gt) {
    const uint64_t T = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (T >= ntiles) return;
    for (uint32_t g = item0[T] / 32; g < item0[T + 1] / 32; ++g) gt[g] = (uint32_t)T;
}

// seg_map.cu bank_schedule, one warp group of items per thread
__global__ void ksp_bank(uint32_t ngroups, const uint32_t* __restrict__ gt, const uint4* __restrict__ items,
                         const uint32_t* __restrict__ ent0, uint32_t* __restrict__ ents, int ni) {
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (g >= ngroups) return;
    const uint4* it = items + 32ull * g;
    uint32_t* ent = ents + ent0[gt[g]];
    uint32_t steps = 0;
    for (int l = 0; l < 32; ++l) steps = max(steps, (it[l].x >> 16) & 0x7Fu);
    if (steps < 2) return;
    uint8_t used[127 * 2 * 16];
    for (uint32_t q = 0; q < steps * 2 * 16; ++q) used[q] = 0;
    uint32_t tmp[127];
    uint8_t taken[127];
    for (int l = 0; l < 32; ++l) {
        const uint32_t meta = it[l].x, beg = meta & 0xFFFFu, sz = (meta >> 16) & 0x7Fu;
        if (sz < 2) {
            if (sz == 1) {
                const uint32_t lr = (ent[beg] & 0x1FFFu) % (uint32_t)ni;
                used[(0 * 2 + (l >> 4)) * 16 + (lr & 15)]++;
            }
            continue;
        }
        for (uint32_t e = 0; e < sz; ++e) {
            tmp[e] = ent[beg + e];
            taken[e] = 0;
        }
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

__global__ void ksp_tdesc(uint32_t ntiles, const uint32_t* __restrict__ tile_v, const uint32_t* __restrict__ inst0,
                          const uint32_t* __restrict__ item0, const uint32_t* __restrict__ ent0,
                          uint4* __restrict__ tdesc) {
    const uint64_t T = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (T > ntiles) return;
    tdesc[T] = make_uint4(tile_v[T], inst0[T], item0[T], ent0[T]);
}

template <typename T>
ebb_status exscan(Ctx* c, const T* in, T* out, uint64_t n) {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int64_t)n);
    DBuf tmp;
    EBB_CUDA(c, tmp.alloc(tb));
    EBB_CUDA(c, cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, (int64_t)n));
    return EBB_OK;
}

template <typename T>
T read1(const T* d) {
    T h{};
    cudaMemcpy(&h, d, sizeof(T), cudaMemcpyDeviceToHost);
    return h;
}

}  // namespace

ebb_status build_seg_plan_device(Ctx* c, const uint32_t* tv, uint64_t nt, const uint32_t* index,
                                 const uint32_t* head, uint64_t nv, int ni, SegPlan* P) {
    const auto t0 = std::chrono::steady_clock::now();
    const unsigned B = 256;
    const uint64_t n4 = nt * 4;
    // 1. vertex -> incident tets
    DBuf k1, v1, k2, v2, vt_ptr, tmp;
    EBB_CUDA(c, k1.alloc(n4 * 4));
    EBB_CUDA(c, v1.alloc(n4 * 4));
    EBB_CUDA(c, k2.alloc(n4 * 4));
    EBB_CUDA(c, v2.alloc(n4 * 4));
    EBB_CUDA(c, vt_ptr.alloc((nv + 1) * 4));
    if (n4) ksp_vt_pairs<<<grid_for(n4, B), B>>>(tv, n4, k1.as<uint32_t>(), v1.as<uint32_t>());
    size_t tb = 0;
    const int vbits = std::max(1, 64 - __builtin_clzll((unsigned long long)nv));
    cub::DeviceRadixSort::SortPairs(nullptr, tb, k1.as<uint32_t>(), k2.as<uint32_t>(), v1.as<uint32_t>(),
                                    v2.as<uint32_t>(), (int64_t)n4, 0, vbits);
    EBB_CUDA(c, tmp.alloc(tb));
    EBB_CUDA(c, cub::DeviceRadixSort::SortPairs(tmp.p, tb, k1.as<uint32_t>(), k2.as<uint32_t>(), v1.as<uint32_t>(),
                                                v2.as<uint32_t>(), (int64_t)n4, 0, vbits));
    ksp_ptr<<<grid_for(nv + 1, B), B>>>(k2.as<uint32_t>(), n4, vt_ptr.as<uint32_t>(), nv);
    const uint32_t* vkey = k2.as<uint32_t>();
    const uint32_t* vt = v2.as<uint32_t>();
    // 2. self rows, canonical-row counts and their prefix
    DBuf rself, ccount, cs, bad;
    EBB_CUDA(c, rself.alloc(nv * 4));
    EBB_CUDA(c, ccount.alloc((nv + 1) * 4));
    EBB_CUDA(c, cs.alloc((nv + 1) * 4));
    EBB_CUDA(c, bad.alloc(4));
    EBB_CUDA(c, cudaMemset(bad.p, 0, 4));
    EBB_CUDA(c, cudaMemset(ccount.p, 0, (nv + 1) * 4));
    ksp_rself<<<grid_for(nv, B), B>>>(nv, index, head, rself.as<uint32_t>(), ccount.as<uint32_t>(),
                                      bad.as<unsigned int>());
    EBB_TRY(exscan<uint32_t>(c, ccount.as<uint32_t>(), cs.as<uint32_t>(), nv + 1));
    // 3. tiles (greedy inside blocks of kSegBlock vertices)
    const uint64_t nblk = (nv + kSegBlock - 1) / kSegBlock;
    DBuf starts, nstart, soff, tile_v_d, tile_of_v;
    EBB_CUDA(c, starts.alloc(nv * 4));
    EBB_CUDA(c, nstart.alloc((nblk + 1) * 4));
    EBB_CUDA(c, soff.alloc((nblk + 1) * 4));
    EBB_CUDA(c, cudaMemset(nstart.p, 0, (nblk + 1) * 4));
    ksp_tiles<<<grid_for(nblk, 64), 64>>>(nv, kSegBlock, ni, tv, vt_ptr.as<uint32_t>(), vt, starts.as<uint32_t>(),
                                          nstart.as<uint32_t>(), bad.as<unsigned int>());
    EBB_TRY(exscan<uint32_t>(c, nstart.as<uint32_t>(), soff.as<uint32_t>(), nblk + 1));
    const uint32_t ntiles = read1(soff.as<uint32_t>() + nblk);
    unsigned int hbad = read1(bad.as<unsigned int>());
    if (hbad & 1u) return fail(c, EBB_E_STATE, "segmented map: a vertex has no self-loop edge row");
    if (hbad & 2u) return fail(c, EBB_E_RANGE, "segmented map: a vertex touches more than %d tets (one tile)", ni);
    EBB_CUDA(c, tile_v_d.alloc((ntiles + 1) * 4));
    EBB_CUDA(c, tile_of_v.alloc(nv * 4));
    ksp_compact_tiles<<<grid_for(nblk, B), B>>>(nblk, kSegBlock, starts.as<uint32_t>(), nstart.as<uint32_t>(),
                                                soff.as<uint32_t>(), tile_v_d.as<uint32_t>());
    const uint32_t nv32 = (uint32_t)nv;
    EBB_CUDA(c, cudaMemcpy(tile_v_d.as<uint32_t>() + ntiles, &nv32, 4, cudaMemcpyHostToDevice));
    ksp_tile_of<<<grid_for(ntiles, B), B>>>(ntiles, tile_v_d.as<uint32_t>(), tile_of_v.as<uint32_t>());
    // 4. instances: unique (tile, tet) pairs, ascending
    DBuf ik, ik2, uk, nu, icnt, inst0, tmp2;
    EBB_CUDA(c, ik.alloc(n4 * 8));
    EBB_CUDA(c, ik2.alloc(n4 * 8));
    EBB_CUDA(c, uk.alloc(n4 * 8));
    EBB_CUDA(c, nu.alloc(8));
    if (n4) ksp_inst_keys<<<grid_for(n4, B), B>>>(n4, vkey, vt, tile_of_v.as<uint32_t>(), ik.as<uint64_t>());
    size_t tb2 = 0, tb3 = 0;
    const int tbits = std::max(1, 64 - __builtin_clzll((unsigned long long)ntiles + 1));
    cub::DeviceRadixSort::SortKeys(nullptr, tb2, ik.as<uint64_t>(), ik2.as<uint64_t>(), (int64_t)n4, 0, 32 + tbits);
    cub::DeviceSelect::Unique(nullptr, tb3, ik2.as<uint64_t>(), uk.as<uint64_t>(), nu.as<uint64_t>(), (int64_t)n4);
    EBB_CUDA(c, tmp2.alloc(std::max(tb2, tb3)));
    EBB_CUDA(c, cub::DeviceRadixSort::SortKeys(tmp2.p, tb2, ik.as<uint64_t>(), ik2.as<uint64_t>(), (int64_t)n4, 0,
                                               32 + tbits));
    EBB_CUDA(c, cub::DeviceSelect::Unique(tmp2.p, tb3, ik2.as<uint64_t>(), uk.as<uint64_t>(), nu.as<uint64_t>(),
                                          (int64_t)n4));
    const uint64_t ninst = read1(nu.as<uint64_t>());
    EBB_CUDA(c, icnt.alloc((ntiles + 1) * 4));
    EBB_CUDA(c, inst0.alloc((ntiles + 1) * 4));
    EBB_CUDA(c, cudaMemset(icnt.p, 0, (ntiles + 1) * 4));
    if (ninst) ksp_hist_hi<<<grid_for(ntiles, B), B>>>(uk.as<uint64_t>(), ninst, 32, icnt.as<uint32_t>(), ntiles);
    EBB_TRY(exscan<uint32_t>(c, icnt.as<uint32_t>(), inst0.as<uint32_t>(), ntiles + 1));
    EBB_CUDA(c, cudaMalloc(&P->inst, ninst * 8 + 16));
    if (ninst)
        ksp_inst<<<grid_for(ninst, B), B>>>(ninst, uk.as<uint64_t>(), inst0.as<uint32_t>(), tv,
                                            tile_of_v.as<uint32_t>(), P->inst);
    ik.reset();
    ik2.reset();
    // 5. entries: keyed (tile, kind, slot, instance, pair), sorted, per tile padded to 4 words
    const uint64_t n10 = nt * 10;
    DBuf ek, ek2, ev, ev2, cnt64, slot_cnt, ecnt, ecntp, e0u, e0p, tmp3;
    EBB_CUDA(c, ek.alloc(n10 * 8));
    EBB_CUDA(c, ek2.alloc(n10 * 8));
    EBB_CUDA(c, ev.alloc(n10 * 4));
    EBB_CUDA(c, ev2.alloc(n10 * 4));
    EBB_CUDA(c, cnt64.alloc(8));
    const uint32_t ncanon = read1(cs.as<uint32_t>() + nv);
    EBB_CUDA(c, slot_cnt.alloc((uint64_t)ncanon * 4));
    EBB_CUDA(c, cudaMemset(slot_cnt.p, 0, (uint64_t)ncanon * 4));
    EBB_CUDA(c, cudaMemset(cnt64.p, 0, 8));
    if (ninst)
        ksp_entries<<<grid_for(ninst, B), B>>>(ninst, P->inst, uk.as<uint64_t>(), ni, tv, tile_of_v.as<uint32_t>(),
                                               tile_v_d.as<uint32_t>(), index, head, rself.as<uint32_t>(),
                                               cs.as<uint32_t>(), ek.as<uint64_t>(), ev.as<uint32_t>(),
                                               cnt64.as<unsigned long long>(), slot_cnt.as<uint32_t>());
    const uint64_t nent_raw = read1(cnt64.as<unsigned long long>());
    size_t tb4 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb4, ek.as<uint64_t>(), ek2.as<uint64_t>(), ev.as<uint32_t>(),
                                    ev2.as<uint32_t>(), (int64_t)nent_raw, 0, 27 + tbits);
    EBB_CUDA(c, tmp3.alloc(tb4));
    EBB_CUDA(c, cub::DeviceRadixSort::SortPairs(tmp3.p, tb4, ek.as<uint64_t>(), ek2.as<uint64_t>(), ev.as<uint32_t>(),
                                                ev2.as<uint32_t>(), (int64_t)nent_raw, 0, 27 + tbits));
    EBB_CUDA(c, ecnt.alloc((ntiles + 1) * 4));
    EBB_CUDA(c, ecntp.alloc((ntiles + 1) * 4));
    EBB_CUDA(c, e0u.alloc((ntiles + 1) * 4));
    EBB_CUDA(c, e0p.alloc((ntiles + 1) * 4));
    EBB_CUDA(c, cudaMemset(ecnt.p, 0, (ntiles + 1) * 4));
    if (nent_raw) ksp_hist_hi<<<grid_for(ntiles, B), B>>>(ek2.as<uint64_t>(), nent_raw, 27, ecnt.as<uint32_t>(), ntiles);
    ksp_pad4<<<grid_for(ntiles + 1, B), B>>>(ntiles + 1, ecnt.as<uint32_t>(), ecntp.as<uint32_t>());
    EBB_TRY(exscan<uint32_t>(c, ecnt.as<uint32_t>(), e0u.as<uint32_t>(), ntiles + 1));
    EBB_TRY(exscan<uint32_t>(c, ecntp.as<uint32_t>(), e0p.as<uint32_t>(), ntiles + 1));
    const uint32_t nent = read1(e0p.as<uint32_t>() + ntiles);
    EBB_CUDA(c, cudaMalloc(&P->ents, (uint64_t)nent * 4 + 16));
    EBB_CUDA(c, cudaMemset(P->ents, 0, (uint64_t)nent * 4 + 16));
    if (nent_raw)
        ksp_place<<<grid_for(nent_raw, B), B>>>(nent_raw, ek2.as<uint64_t>(), ev2.as<uint32_t>(), e0u.as<uint32_t>(),
                                                e0p.as<uint32_t>(), P->ents);
    ek.reset();
    ek2.reset();
    ev.reset();
    ev2.reset();
    // 6. items
    TileSlots S{tile_v_d.as<uint32_t>(), index, head, rself.as<uint32_t>(), ccount.as<uint32_t>(), cs.as<uint32_t>(),
                slot_cnt.as<uint32_t>(), ni};
    DBuf tileL, nitems, item0, gt;
    EBB_CUDA(c, tileL.alloc((ntiles + 1) * 4));
    EBB_CUDA(c, nitems.alloc((ntiles + 1) * 4));
    EBB_CUDA(c, item0.alloc((ntiles + 1) * 4));
    EBB_CUDA(c, cudaMemset(nitems.p, 0, (ntiles + 1) * 4));
    ksp_layout_count<<<grid_for(ntiles, 64), 64>>>(S, ntiles, tileL.as<uint32_t>(), nitems.as<uint32_t>(),
                                                    bad.as<unsigned int>());
    EBB_TRY(exscan<uint32_t>(c, nitems.as<uint32_t>(), item0.as<uint32_t>(), ntiles + 1));
    const uint32_t nit = read1(item0.as<uint32_t>() + ntiles);
    hbad = read1(bad.as<unsigned int>());
    if (hbad & 4u) return fail(c, EBB_E_RANGE, "segmented map: a list of more than 8 x 127 entries");
    EBB_CUDA(c, cudaMalloc(&P->items, (uint64_t)nit * 16 + 16));
    ksp_layout_emit<<<grid_for(ntiles, 64), 64>>>(S, ntiles, tileL.as<uint32_t>(), item0.as<uint32_t>(), P->items);
    const uint32_t ngroups = nit / 32;
    EBB_CUDA(c, gt.alloc((uint64_t)ngroups * 4));
    ksp_group_tile<<<grid_for(ntiles, B), B>>>(ntiles, item0.as<uint32_t>(), gt.as<uint32_t>());
    if (!getenv("EBB_SEG_NO_BANK_SCHED") && ngroups)
        ksp_bank<<<grid_for(ngroups, 64), 64>>>(ngroups, gt.as<uint32_t>(), P->items, e0p.as<uint32_t>(), P->ents, ni);
    EBB_CUDA(c, cudaMalloc(&P->tdesc, (uint64_t)(ntiles + 1) * 16));
    ksp_tdesc<<<grid_for(ntiles + 1, B), B>>>(ntiles, tile_v_d.as<uint32_t>(), inst0.as<uint32_t>(),
                                              item0.as<uint32_t>(), e0p.as<uint32_t>(), P->tdesc);
    EBB_CUDA(c, cudaDeviceSynchronize());
    EBB_CUDA(c, cudaGetLastError());
    // the largest tile's entries / items (the kernel's shared-memory budget)
    std::vector<uint32_t> h0(ntiles + 1), h1(ntiles + 1);
    EBB_CUDA(c, cudaMemcpy(h0.data(), e0p.p, (ntiles + 1) * 4, cudaMemcpyDeviceToHost));
    EBB_CUDA(c, cudaMemcpy(h1.data(), item0.p, (ntiles + 1) * 4, cudaMemcpyDeviceToHost));
    uint32_t max_ent = 0, max_items = 0;
    for (uint32_t T = 0; T < ntiles; ++T) {
        max_ent = std::max(max_ent, h0[T + 1] - h0[T]);
        max_items = std::max(max_items, h1[T + 1] - h1[T]);
    }
    if (max_ent >= 65536) return fail(c, EBB_E_RANGE, "segmented map: a tile has %u entries (> 65535)", max_ent);
    P->ntiles = ntiles;
    P->max_ent = max_ent;
    P->max_items = max_items;
    P->ninst = ninst;
    P->run = 1;
    P->nent = nent;
    P->nitems = nit;
    P->host_threads = 0;
    P->host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return EBB_OK;
}

}  // namespace ebb
