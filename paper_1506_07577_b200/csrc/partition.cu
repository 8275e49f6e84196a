// partition.cu -- the local problem of one rank of the multi-GPU domain
// decomposition (SURVEY §8(e), O4 and its overlapping reading),
// built on the device from the global owner maps of ebb_partition, and the
// relation / field lifetime calls (a rank frees the global mesh it partitioned).
//
//   local tets   EBB_PART_OVERLAP: every tet with a vertex owned by the rank
//                (ghost tets: every block of every owned edge row is local);
//                EBB_PART_OWN: the tets the rank owns (O4: owner_t == rank)
//   local verts  the owned vertices ascending, then the ghosts (vertices of
//                local tets owned elsewhere) ascending -- global ids
//   halo lists   send to q = owned vertices that are ghosts on q, recv from q =
//                ghosts owned by q, both ascending in global id, so both ends
//                of a pair derive the same order without negotiation
// All of it is stream compaction, sorts and scans (CUB) over the global
// arrays; the host only reads the counts.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <string>
#include <vector>

#include "ebb_internal.cuh"

namespace ebb {
namespace {

struct Buf {
    void* p = nullptr;
    ~Buf() { cudaFree(p); }
    cudaError_t alloc(size_t b) { return cudaMalloc(&p, b + 16); }
    template <typename T>
    T* as() const { return (T*)p; }
};

// local-tet flag of every global tet
__global__ void kpl_tet_flag(const uint4* __restrict__ tv, uint64_t nt, const int32_t* __restrict__ owner_t,
                             const int32_t* __restrict__ owner_v, int32_t rank, int mode, uint8_t* __restrict__ flag) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    if (mode == EBB_PART_OWN) {
        flag[t] = owner_t[t] == rank;
        return;
    }
    const uint4 v = tv[t];
    flag[t] = owner_v[v.x] == rank || owner_v[v.y] == rank || owner_v[v.z] == rank || owner_v[v.w] == rank;
}

// vertices of the local tets
__global__ void kpl_vert_mark(const uint4* __restrict__ tv, const uint32_t* __restrict__ lt, uint64_t n,
                              uint8_t* __restrict__ used) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint4 v = tv[lt[i]];
    used[v.x] = used[v.y] = used[v.z] = used[v.w] = 1;
}

// owned flag (every owned vertex is local, isolated ones too) and ghost flag
__global__ void kpl_vert_flags(uint64_t nv, const int32_t* __restrict__ owner_v, int32_t rank,
                               const uint8_t* __restrict__ used, uint8_t* __restrict__ fo, uint8_t* __restrict__ fg) {
    const uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (v >= nv) return;
    fo[v] = owner_v[v] == rank;
    fg[v] = used[v] && owner_v[v] != rank;
}

__global__ void kpl_g2l(const uint32_t* __restrict__ lv, uint64_t n, uint32_t* __restrict__ g2l) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) g2l[lv[i]] = (uint32_t)i;
}

// local tets' vertex keys in the local numbering (u64 for ebb_key_field)
__global__ void kpl_local_keys(const uint4* __restrict__ tv, const uint32_t* __restrict__ lt, uint64_t n,
                               const uint32_t* __restrict__ g2l, uint64_t* __restrict__ keys) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint4 v = tv[lt[i]];
    keys[4 * i + 0] = g2l[v.x];
    keys[4 * i + 1] = g2l[v.y];
    keys[4 * i + 2] = g2l[v.z];
    keys[4 * i + 3] = g2l[v.w];
}

// send candidates (peer << 32 | local row of an owned vertex), ~0 = none.
// OVERLAP: owned vertex a shares a tet with a vertex owned by q (then that tet
// is local on q and a is a ghost there); scanning the local tets suffices.
// OWN: owned vertex a lies in a tet owned by q (a vertex of q's own tets);
// every global tet is scanned.
__global__ void kpl_send_pairs(const uint4* __restrict__ tv, const uint32_t* __restrict__ tl, uint64_t n,
                               const int32_t* __restrict__ owner_t, const int32_t* __restrict__ owner_v, int32_t rank,
                               int mode, const uint32_t* __restrict__ g2l, uint64_t* __restrict__ out) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t t = tl ? tl[i] : i;
    const uint4 v4 = tv[t];
    const uint32_t v[4] = {v4.x, v4.y, v4.z, v4.w};
    uint64_t* o = out + 16 * i;
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
            uint64_t k = ~0ull;
            if (mode == EBB_PART_OWN) {
                if (b == 0 && owner_v[v[a]] == rank && owner_t[t] != rank)
                    k = ((uint64_t)(uint32_t)owner_t[t] << 32) | g2l[v[a]];
            } else if (a != b && owner_v[v[a]] == rank && owner_v[v[b]] != rank) {
                k = ((uint64_t)(uint32_t)owner_v[v[b]] << 32) | g2l[v[a]];
            }
            o[4 * a + b] = k;
        }
}

// ghosts (local rows n_owned..) keyed by (owner << 32 | local row)
__global__ void kpl_recv_keys(const uint32_t* __restrict__ gh, uint64_t n, uint64_t n_owned,
                              const int32_t* __restrict__ owner_v, uint64_t* __restrict__ out) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = ((uint64_t)(uint32_t)owner_v[gh[i]] << 32) | (n_owned + i);
}

// split sorted (peer << 32 | row) keys into per-peer counts and the rows
__global__ void kpl_split(const uint64_t* __restrict__ k, uint64_t n, uint32_t* __restrict__ rows,
                          unsigned long long* __restrict__ cnt) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    rows[i] = (uint32_t)k[i];
    atomicAdd(cnt + (k[i] >> 32), 1ull);
}


// ---- reverse-add lists (EBB_PART_OVERLAP local mesh, one computing rank per tet)
// rank of a tet in the reverse-add variant: the owner of its lowest-gid vertex
__device__ __forceinline__ int32_t tet_rank(const uint32_t v[4], const uint32_t* __restrict__ gid,
                                            const int32_t* __restrict__ owner) {
    int k = 0;
    for (int i = 1; i < 4; ++i)
        if (gid[v[i]] < gid[v[k]]) k = i;
    return owner[v[k]];
}

// candidates (key = gid order, val = peer << 32 | local row), key ~0 = none:
//   f send: own tet, vertex owned by q != rank       f recv: tet of q, vertex owned by rank
//   K send: own tet, (i, j) with tail owned by q      K recv: tet of q, (i, j) with tail owned by rank
__global__ void kpl_reverse(const uint4* __restrict__ tv, const uint32_t* __restrict__ te, uint64_t n,
                            const uint32_t* __restrict__ gid, const int32_t* __restrict__ owner, int32_t rank,
                            uint8_t* __restrict__ own, uint64_t* __restrict__ fk, uint64_t* __restrict__ fv,
                            uint64_t* __restrict__ kk, uint64_t* __restrict__ kv) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint4 v4 = tv[t];
    const uint32_t v[4] = {v4.x, v4.y, v4.z, v4.w};
    const int32_t tr = tet_rank(v, gid, owner);
    own[t] = tr == rank;
    for (int i = 0; i < 4; ++i) {
        const int32_t oi = owner[v[i]];
        const bool snd = tr == rank && oi != rank, rcv = tr != rank && oi == rank;
        const uint32_t peer = (uint32_t)(snd ? oi : tr);
        fk[4 * t + i] = (snd || rcv) ? gid[v[i]] : ~0ull;
        fv[4 * t + i] = ((uint64_t)peer << 32) | v[i];
        for (int j = 0; j < 4; ++j) {
            kk[16 * t + 4 * i + j] = (snd || rcv) ? ((uint64_t)gid[v[i]] << 32 | gid[v[j]]) : ~0ull;
            kv[16 * t + 4 * i + j] = ((uint64_t)peer << 32) | te[16 * t + 4 * i + j];
        }
    }
}

// keep the candidates of one role (0: own tet = send, 1: receive)
__global__ void kpl_role(uint64_t* __restrict__ k, const uint64_t* __restrict__ v, uint64_t n, int per,
                         const uint8_t* __restrict__ own, int role) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    if ((own[i / per] != 0) != (role == 0)) k[i] = ~0ull;
    (void)v;
}

__global__ void kpl_peer_key(const uint64_t* __restrict__ v, uint64_t n, uint32_t* __restrict__ q) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) q[i] = (uint32_t)(v[i] >> 32);
}

}  // namespace
}  // namespace ebb

using namespace ebb;

extern "C" {

ebb_status ebb_partition_local(ebb_ctx ctx, ebb_field tets_v, ebb_field owner_t, ebb_field owner_v, int32_t nparts,
                               int32_t rank, int32_t mode, const char* name, ebb_partition_info* out,
                               uint64_t* send_ptr, uint64_t* recv_ptr) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !name || !out || !send_ptr || !recv_ptr) return fail(c, EBB_E_ARG, "null argument");
    if (nparts < 1 || rank < 0 || rank >= nparts) return fail(c, EBB_E_ARG, "rank %d of %d parts", rank, nparts);
    if (mode != EBB_PART_OVERLAP && mode != EBB_PART_OWN) return fail(c, EBB_E_ARG, "unknown partition mode %d", mode);
    Field* V = get_field(c, tets_v);
    Field* OT = get_field(c, owner_t);
    Field* OV = get_field(c, owner_v);
    if (!V || !OT || !OV) return fail(c, EBB_E_ARG, "bad field handle");
    if (V->dtype != EBB_KEY || V->comps() != 4 || V->layout != EBB_AOS)
        return fail(c, EBB_E_TYPE, "'%s' must be a 4x1 key-field (tets.v)", V->name.c_str());
    if (OT->dtype != EBB_I32 || OT->rel != V->rel || OV->dtype != EBB_I32 || OV->rel != V->key_target)
        return fail(c, EBB_E_TYPE, "owner fields must be I32 on tets / verts (ebb_partition)");
    const uint64_t nt = c->rels[V->rel].size, nv = c->rels[V->key_target].size;
    const uint4* tv = (const uint4*)V->ptr;
    const int32_t* ot = (const int32_t*)OT->ptr;
    const int32_t* ov = (const int32_t*)OV->ptr;
    const unsigned B = 256;
    *out = ebb_partition_info{};
    out->ltets = out->lverts = out->send = out->recv = EBB_NONE;
    out->tet_gid = out->vert_gid = out->v = out->send_rows = out->recv_rows = EBB_NONE;
    // 1. local tets (ascending global id)
    Buf flag, lt, cnt, tmp;
    EBB_CUDA(c, flag.alloc(std::max(nt, nv)));
    EBB_CUDA(c, lt.alloc(nt * 4));
    EBB_CUDA(c, cnt.alloc(64));
    if (nt) kpl_tet_flag<<<grid_for(nt, B), B>>>(tv, nt, ot, ov, rank, mode, flag.as<uint8_t>());
    thrust::counting_iterator<uint32_t> iota(0);
    size_t tb = 0, tb2 = 0;
    cub::DeviceSelect::Flagged(nullptr, tb, iota, flag.as<uint8_t>(), lt.as<uint32_t>(), cnt.as<uint64_t>(),
                               (int64_t)std::max(nt, nv));
    cub::DeviceRadixSort::SortKeys(nullptr, tb2, (uint64_t*)nullptr, (uint64_t*)nullptr, (int64_t)(16 * nt + nv));
    size_t tb3 = 0;
    cub::DeviceSelect::Unique(nullptr, tb3, (uint64_t*)nullptr, (uint64_t*)nullptr, cnt.as<uint64_t>(),
                              (int64_t)(16 * nt + nv));
    EBB_CUDA(c, tmp.alloc(std::max(tb, std::max(tb2, tb3))));
    EBB_CUDA(c, cub::DeviceSelect::Flagged(tmp.p, tb, iota, flag.as<uint8_t>(), lt.as<uint32_t>(), cnt.as<uint64_t>(),
                                           (int64_t)nt));
    uint64_t n_lt = 0;
    EBB_CUDA(c, cudaMemcpy(&n_lt, cnt.p, 8, cudaMemcpyDeviceToHost));
    // 2. local vertices: owned ascending, then ghosts ascending
    Buf used, fo, fg, lv, g2l;
    EBB_CUDA(c, used.alloc(nv));
    EBB_CUDA(c, fo.alloc(nv));
    EBB_CUDA(c, fg.alloc(nv));
    EBB_CUDA(c, lv.alloc(nv * 4));
    EBB_CUDA(c, g2l.alloc(nv * 4));
    EBB_CUDA(c, cudaMemset(used.p, 0, nv));
    if (n_lt) kpl_vert_mark<<<grid_for(n_lt, B), B>>>(tv, lt.as<uint32_t>(), n_lt, used.as<uint8_t>());
    if (nv) kpl_vert_flags<<<grid_for(nv, B), B>>>(nv, ov, rank, used.as<uint8_t>(), fo.as<uint8_t>(), fg.as<uint8_t>());
    EBB_CUDA(c, cub::DeviceSelect::Flagged(tmp.p, tb, iota, fo.as<uint8_t>(), lv.as<uint32_t>(), cnt.as<uint64_t>(),
                                           (int64_t)nv));
    uint64_t n_own = 0, n_gh = 0;
    EBB_CUDA(c, cudaMemcpy(&n_own, cnt.p, 8, cudaMemcpyDeviceToHost));
    EBB_CUDA(c, cub::DeviceSelect::Flagged(tmp.p, tb, iota, fg.as<uint8_t>(), lv.as<uint32_t>() + n_own,
                                           cnt.as<uint64_t>(), (int64_t)nv));
    EBB_CUDA(c, cudaMemcpy(&n_gh, cnt.p, 8, cudaMemcpyDeviceToHost));
    const uint64_t n_lv = n_own + n_gh;
    if (n_lt == 0 || n_lv == 0) return fail(c, EBB_E_SIZE, "partition: rank %d has an empty local mesh", rank);
    if (n_lv) kpl_g2l<<<grid_for(n_lv, B), B>>>(lv.as<uint32_t>(), n_lv, g2l.as<uint32_t>());
    // 3. halo lists
    const uint64_t ncand = mode == EBB_PART_OWN ? nt : n_lt;
    Buf sk, sk2, su, rk, rk2, rows, pc;
    EBB_CUDA(c, sk.alloc(16 * ncand * 8));
    EBB_CUDA(c, sk2.alloc(16 * ncand * 8));
    EBB_CUDA(c, su.alloc(16 * ncand * 8));
    EBB_CUDA(c, pc.alloc((uint64_t)nparts * 16));
    if (ncand)
        kpl_send_pairs<<<grid_for(ncand, B), B>>>(tv, mode == EBB_PART_OWN ? nullptr : lt.as<uint32_t>(), ncand, ot, ov,
                                                  rank, mode, g2l.as<uint32_t>(), sk.as<uint64_t>());
    EBB_CUDA(c, cub::DeviceRadixSort::SortKeys(tmp.p, tb2, sk.as<uint64_t>(), sk2.as<uint64_t>(), (int64_t)(16 * ncand)));
    EBB_CUDA(c, cub::DeviceSelect::Unique(tmp.p, tb3, sk2.as<uint64_t>(), su.as<uint64_t>(), cnt.as<uint64_t>(),
                                          (int64_t)(16 * ncand)));
    uint64_t n_su = 0;
    EBB_CUDA(c, cudaMemcpy(&n_su, cnt.p, 8, cudaMemcpyDeviceToHost));
    uint64_t last = 0;
    if (n_su) EBB_CUDA(c, cudaMemcpy(&last, su.as<uint64_t>() + n_su - 1, 8, cudaMemcpyDeviceToHost));
    const uint64_t n_send = (n_su && last == ~0ull) ? n_su - 1 : n_su;   // drop the "none" key (sorts last)
    EBB_CUDA(c, rk.alloc(n_gh * 8));
    EBB_CUDA(c, rk2.alloc(n_gh * 8));
    if (n_gh) kpl_recv_keys<<<grid_for(n_gh, B), B>>>(lv.as<uint32_t>() + n_own, n_gh, n_own, ov, rk.as<uint64_t>());
    EBB_CUDA(c, cub::DeviceRadixSort::SortKeys(tmp.p, tb2, rk.as<uint64_t>(), rk2.as<uint64_t>(), (int64_t)n_gh));
    // 4. library relations and fields of the local problem
    const std::string nm(name);
    EBB_TRY(ebb_relation_new(ctx, (nm + ".ltets").c_str(), n_lt, &out->ltets));
    EBB_TRY(ebb_relation_new(ctx, (nm + ".lverts").c_str(), n_lv, &out->lverts));
    EBB_TRY(new_internal_field(c, out->ltets, "gid", EBB_U32, 1, 1, EBB_AOS, &out->tet_gid));
    EBB_TRY(new_internal_field(c, out->lverts, "gid", EBB_U32, 1, 1, EBB_AOS, &out->vert_gid));
    EBB_CUDA(c, cudaMemcpy(c->fields[out->tet_gid].ptr, lt.p, n_lt * 4, cudaMemcpyDeviceToDevice));
    EBB_CUDA(c, cudaMemcpy(c->fields[out->vert_gid].ptr, lv.p, n_lv * 4, cudaMemcpyDeviceToDevice));
    {
        Buf keys;
        EBB_CUDA(c, keys.alloc(n_lt * 32));
        kpl_local_keys<<<grid_for(n_lt, B), B>>>(tv, lt.as<uint32_t>(), n_lt, g2l.as<uint32_t>(), keys.as<uint64_t>());
        EBB_CUDA(c, cudaGetLastError());
        EBB_TRY(ebb_key_field(ctx, out->ltets, "v", out->lverts, 4, 1, keys.as<uint64_t>(), 1, &out->v));
    }
    std::vector<unsigned long long> hc(nparts);
    auto lists = [&](const uint64_t* k, uint64_t n, const char* suffix, ebb_rel* rel, ebb_field* rf, uint64_t* ptr) {
        for (int q = 0; q <= nparts; ++q) ptr[q] = 0;
        if (n == 0) return EBB_OK;
        EBB_CUDA(c, cudaMemset(pc.p, 0, (size_t)nparts * 8));
        EBB_TRY(ebb_relation_new(ctx, (nm + suffix).c_str(), n, rel));
        EBB_TRY(new_internal_field(c, *rel, "rows", EBB_U32, 1, 1, EBB_AOS, rf));
        kpl_split<<<grid_for(n, B), B>>>(k, n, (uint32_t*)c->fields[*rf].ptr, pc.as<unsigned long long>());
        EBB_CUDA(c, cudaGetLastError());
        EBB_CUDA(c, cudaMemcpy(hc.data(), pc.p, (size_t)nparts * 8, cudaMemcpyDeviceToHost));
        for (int q = 0; q < nparts; ++q) ptr[q + 1] = ptr[q] + hc[q];
        return EBB_OK;
    };
    EBB_TRY(lists(su.as<uint64_t>(), n_send, ".send", &out->send, &out->send_rows, send_ptr));
    EBB_TRY(lists(rk2.as<uint64_t>(), n_gh, ".recv", &out->recv, &out->recv_rows, recv_ptr));
    EBB_CUDA(c, cudaDeviceSynchronize());
    out->n_ltets = n_lt;
    out->n_lverts = n_lv;
    out->n_owned = n_own;
    return EBB_OK;
}

// a (gid-key, peer|row) candidate set -> rows grouped by peer in gid order,
// duplicates (several tets of one row) removed; creates relation `rel_name`
static ebb_status reverse_list(Ctx* c, uint64_t* k, uint64_t* v, uint64_t n, int32_t nparts,
                               const std::string& rel_name, ebb_rel* rel, ebb_field* rows, uint64_t* ptr) {
    ebb_ctx ctx = (ebb_ctx)c;
    for (int q = 0; q <= nparts; ++q) ptr[q] = 0;
    *rel = EBB_NONE;
    *rows = EBB_NONE;
    const unsigned B = 256;
    Buf k2, v2, v3, q1, q2, tmp, cnt, pc;
    EBB_CUDA(c, k2.alloc(n * 8));
    EBB_CUDA(c, v2.alloc(n * 8));
    EBB_CUDA(c, v3.alloc(n * 8));
    EBB_CUDA(c, q1.alloc(n * 4));
    EBB_CUDA(c, q2.alloc(n * 4));
    EBB_CUDA(c, cnt.alloc(8));
    EBB_CUDA(c, pc.alloc((size_t)nparts * 8));
    size_t t1 = 0, t2 = 0, t3 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, k, k2.as<uint64_t>(), v, v2.as<uint64_t>(), (int64_t)n);
    cub::DeviceRadixSort::SortPairs(nullptr, t2, q1.as<uint32_t>(), q2.as<uint32_t>(), v2.as<uint64_t>(),
                                    v3.as<uint64_t>(), (int64_t)n);
    cub::DeviceSelect::Unique(nullptr, t3, v3.as<uint64_t>(), k2.as<uint64_t>(), cnt.as<uint64_t>(), (int64_t)n);
    EBB_CUDA(c, tmp.alloc(std::max(t1, std::max(t2, t3))));
    // by (tail gid, head gid), then stably by peer; the "none" keys sort last
    EBB_CUDA(c, cub::DeviceRadixSort::SortPairs(tmp.p, t1, k, k2.as<uint64_t>(), v, v2.as<uint64_t>(), (int64_t)n));
    uint64_t nvalid = n;
    {
        // count the valid candidates: keys != ~0 form a prefix after the sort
        std::vector<uint64_t> probe(1);
        uint64_t lo = 0, hi = n;
        while (lo < hi) {   // first ~0 key (binary search with single-element reads)
            const uint64_t mid = (lo + hi) / 2;
            EBB_CUDA(c, cudaMemcpy(probe.data(), k2.as<uint64_t>() + mid, 8, cudaMemcpyDeviceToHost));
            if (probe[0] == ~0ull) hi = mid;
            else lo = mid + 1;
        }
        nvalid = lo;
    }
    if (nvalid == 0) return EBB_OK;
    kpl_peer_key<<<grid_for(nvalid, B), B>>>(v2.as<uint64_t>(), nvalid, q1.as<uint32_t>());
    EBB_CUDA(c, cub::DeviceRadixSort::SortPairs(tmp.p, t2, q1.as<uint32_t>(), q2.as<uint32_t>(), v2.as<uint64_t>(),
                                                v3.as<uint64_t>(), (int64_t)nvalid));
    EBB_CUDA(c, cub::DeviceSelect::Unique(tmp.p, t3, v3.as<uint64_t>(), k2.as<uint64_t>(), cnt.as<uint64_t>(),
                                          (int64_t)nvalid));
    uint64_t nu = 0;
    EBB_CUDA(c, cudaMemcpy(&nu, cnt.p, 8, cudaMemcpyDeviceToHost));
    EBB_TRY(ebb_relation_new(ctx, rel_name.c_str(), nu, rel));
    EBB_TRY(new_internal_field(c, *rel, "rows", EBB_U32, 1, 1, EBB_AOS, rows));
    EBB_CUDA(c, cudaMemset(pc.p, 0, (size_t)nparts * 8));
    kpl_split<<<grid_for(nu, B), B>>>(k2.as<uint64_t>(), nu, (uint32_t*)c->fields[*rows].ptr,
                                      pc.as<unsigned long long>());
    EBB_CUDA(c, cudaGetLastError());
    std::vector<unsigned long long> hc(nparts);
    EBB_CUDA(c, cudaMemcpy(hc.data(), pc.p, (size_t)nparts * 8, cudaMemcpyDeviceToHost));
    for (int q = 0; q < nparts; ++q) ptr[q + 1] = ptr[q] + hc[q];
    return EBB_OK;
}

ebb_status ebb_partition_reverse(ebb_ctx ctx, ebb_field tets_v, ebb_field tets_e, ebb_field vert_gid,
                                 ebb_field owner_lv, int32_t nparts, int32_t rank, const char* name,
                                 ebb_reverse_info* out, uint64_t* ptrs) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !name || !out || !ptrs) return fail(c, EBB_E_ARG, "null argument");
    if (nparts < 1 || rank < 0 || rank >= nparts) return fail(c, EBB_E_ARG, "rank %d of %d parts", rank, nparts);
    Field* V = get_field(c, tets_v);
    Field* E = get_field(c, tets_e);
    Field* G = get_field(c, vert_gid);
    Field* O = get_field(c, owner_lv);
    if (!V || !E || !G || !O) return fail(c, EBB_E_ARG, "bad field handle");
    if (V->dtype != EBB_KEY || V->comps() != 4 || E->dtype != EBB_KEY || E->comps() != 16 || E->rel != V->rel)
        return fail(c, EBB_E_TYPE, "tets_v / tets_e must be the 4x1 / 4x4 key-fields of one tet relation");
    if (G->dtype != EBB_U32 || G->rel != V->key_target || O->dtype != EBB_I32 || O->rel != V->key_target)
        return fail(c, EBB_E_TYPE, "vert_gid (U32) and owner_lv (I32) must be fields on the local vertices");
    const uint64_t nt = c->rels[V->rel].size;
    const std::string nm(name);
    *out = ebb_reverse_info{};
    EBB_TRY(new_internal_field(c, V->rel, nm + "_own", EBB_U8, 1, 1, EBB_AOS, &out->own));
    V = get_field(c, tets_v);
    E = get_field(c, tets_e);
    G = get_field(c, vert_gid);
    O = get_field(c, owner_lv);
    Buf fk, fv, kk, kv;
    EBB_CUDA(c, fk.alloc(nt * 32));
    EBB_CUDA(c, fv.alloc(nt * 32));
    EBB_CUDA(c, kk.alloc(nt * 128));
    EBB_CUDA(c, kv.alloc(nt * 128));
    if (nt)
        kpl_reverse<<<grid_for(nt, 256), 256>>>((const uint4*)V->ptr, (const uint32_t*)E->ptr, nt,
                                                (const uint32_t*)G->ptr, (const int32_t*)O->ptr, rank,
                                                (uint8_t*)c->fields[out->own].ptr, fk.as<uint64_t>(),
                                                fv.as<uint64_t>(), kk.as<uint64_t>(), kv.as<uint64_t>());
    EBB_CUDA(c, cudaGetLastError());
    // the candidates mix sends (own tets) and receives (tets of other ranks):
    // per role, the other role's keys are set to ~0 (kpl_role), then one list
    const uint64_t n4 = 4 * nt, n16 = 16 * nt;
    Buf fk2, kk2;
    EBB_CUDA(c, fk2.alloc(n4 * 8));
    EBB_CUDA(c, kk2.alloc(n16 * 8));
    for (int role = 0; role < 2; ++role) {   // 0 send, 1 recv
        EBB_CUDA(c, cudaMemcpy(fk2.p, fk.p, n4 * 8, cudaMemcpyDeviceToDevice));
        EBB_CUDA(c, cudaMemcpy(kk2.p, kk.p, n16 * 8, cudaMemcpyDeviceToDevice));
        if (nt) {
            kpl_role<<<grid_for(n4, 256), 256>>>(fk2.as<uint64_t>(), fv.as<uint64_t>(), n4, 4, (const uint8_t*)c->fields[out->own].ptr, role);
            kpl_role<<<grid_for(n16, 256), 256>>>(kk2.as<uint64_t>(), kv.as<uint64_t>(), n16, 16, (const uint8_t*)c->fields[out->own].ptr, role);
        }
        EBB_CUDA(c, cudaGetLastError());
        Buf fvc, kvc;
        EBB_CUDA(c, fvc.alloc(n4 * 8));
        EBB_CUDA(c, kvc.alloc(n16 * 8));
        EBB_CUDA(c, cudaMemcpy(fvc.p, fv.p, n4 * 8, cudaMemcpyDeviceToDevice));
        EBB_CUDA(c, cudaMemcpy(kvc.p, kv.p, n16 * 8, cudaMemcpyDeviceToDevice));
        const char* rn = role == 0 ? "send" : "recv";
        EBB_TRY(reverse_list(c, fk2.as<uint64_t>(), fvc.as<uint64_t>(), n4, nparts, nm + ".f" + rn,
                             role == 0 ? &out->fsend : &out->frecv, role == 0 ? &out->fsend_rows : &out->frecv_rows,
                             ptrs + (role == 0 ? 0 : 1) * (nparts + 1)));
        EBB_TRY(reverse_list(c, kk2.as<uint64_t>(), kvc.as<uint64_t>(), n16, nparts, nm + ".k" + rn,
                             role == 0 ? &out->ksend : &out->krecv, role == 0 ? &out->ksend_rows : &out->krecv_rows,
                             ptrs + (role == 0 ? 2 : 3) * (nparts + 1)));
    }
    EBB_CUDA(c, cudaDeviceSynchronize());
    return EBB_OK;
}

ebb_status ebb_field_free(ebb_ctx ctx, ebb_field f) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    Field* F = get_field(c, f);
    if (!F) return fail(c, EBB_E_ARG, "bad field handle");
    for (auto& R : c->rels)
        if (R.alive && (R.grouped_by == f || R.index == f))
            return fail(c, EBB_E_STATE, "field '%s' groups or indexes relation '%s' (free the relation)",
                        F->name.c_str(), R.name.c_str());
    release_plans(c);   // plans are keyed by field handles
    if (F->owned && F->ptr) cudaFree(F->ptr);
    F->ptr = nullptr;
    F->alive = false;
    return EBB_OK;
}

ebb_status ebb_relation_free(ebb_ctx ctx, ebb_rel rel) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    Relation* R = get_rel(c, rel);
    if (!R) return fail(c, EBB_E_ARG, "bad relation handle");
    // refused while another live relation keeps key-fields into it
    for (size_t k = 0; k < c->fields.size(); ++k) {
        const Field& F = c->fields[k];
        if (F.alive && F.dtype == EBB_KEY && F.key_target == rel && F.rel != rel && c->rels[F.rel].alive)
            return fail(c, EBB_E_STATE, "relation '%s' is the target of key-field '%s' on '%s' (free that first)",
                        R->name.c_str(), F.name.c_str(), c->rels[F.rel].name.c_str());
    }
    release_plans(c);
    // its hidden group index (on its own hidden relation) and the index the
    // grouping left on the source relation
    std::vector<ebb_rel> hidden;
    if (R->index != EBB_NONE && R->grouped_by != EBB_NONE) {
        const ebb_rel ir = c->fields[R->index].rel;
        for (auto& S : c->rels)
            if (S.alive && S.index == R->index && &S != R) S.index = EBB_NONE;
        if (ir != rel) hidden.push_back(ir);
    }
    hidden.push_back(rel);
    for (ebb_rel r : hidden) {
        Relation& Q = c->rels[r];
        for (ebb_field f : Q.fields) {
            Field& F = c->fields[f];
            if (!F.alive) continue;
            if (F.owned && F.ptr) cudaFree(F.ptr);
            F.ptr = nullptr;
            F.alive = false;
        }
        Q.fields.clear();
        Q.alive = false;
        Q.size = 0;
        Q.index = Q.grouped_by = EBB_NONE;
        Q.name = "__freed";
    }
    return EBB_OK;
}

}  // extern "C"
