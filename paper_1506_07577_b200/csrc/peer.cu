// peer.cu -- host side of the fused multi-GPU PCG over peer memory (SURVEY
// §8(e): the halo of the gathered CG operand and the allreduce of the CG
// scalars without NCCL on the iteration path; the kernels are in
// peer_cg.cu): the per-source-row send lists (a CSR over the source rows,
// built on the device from the per-peer halo lists of ebb_partition_local /
// ebb_partition_reverse)
// and CUDA IPC of library fields (one process per GPU maps its peers'
// buffers; ranks emulated on one device use the fields' own addresses).
#include <cub/cub.cuh>

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

// entries of peer k: key = local row, value = (peer rank, remote row); rows
// out of range raise bad[0]
__global__ void kpe_fill(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ remote, uint64_t n,
                         uint32_t peer, uint64_t n_src, uint64_t peer_nv, uint32_t* __restrict__ key,
                         uint64_t* __restrict__ val, unsigned int* __restrict__ bad) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t r = rows[i], q = remote[i];
    if (r >= n_src || q >= peer_nv) atomicAdd(bad, 1u);
    key[i] = r;
    val[i] = ((uint64_t)q << 32) | peer;   // uint2 (peer, remote row) in little-endian order
}

// off[v] = first entry with key >= v (keys sorted), v in [0, n_src]
__global__ void kpe_offsets(const uint32_t* __restrict__ key, uint64_t n, uint64_t n_src, uint32_t* __restrict__ off) {
    const uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (v > n_src) return;
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (key[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    off[v] = (uint32_t)lo;
}

}  // namespace
}  // namespace ebb

using namespace ebb;

extern "C" {

ebb_status ebb_peer_send_csr(ebb_ctx ctx, uint64_t n_src, int32_t npeers, const int32_t* peers,
                             const ebb_field* send_rows, const ebb_field* remote_rows, const uint64_t* peer_nv,
                             const char* name, ebb_field* send_off, ebb_field* send_dst) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !send_off || !send_dst || npeers < 0 || npeers > EBB_MAX_RANKS || n_src >= 0xffffffffull)
        return EBB_E_ARG;
    if (npeers > 0 && (!peers || !send_rows || !remote_rows || !peer_nv)) return EBB_E_ARG;
    const std::string nm = name ? name : "peer";
    uint64_t n = 0;
    for (int k = 0; k < npeers; ++k) {
        Field* S = get_field(c, send_rows[k]);
        Field* Q = get_field(c, remote_rows[k]);
        if (!S || !Q) return fail(c, EBB_E_ARG, "peer_send_csr: bad row field of peer %d", k);
        if (S->dtype != EBB_U32 || Q->dtype != EBB_U32 || S->comps() != 1 || Q->comps() != 1)
            return fail(c, EBB_E_TYPE, "peer_send_csr: row lists must be U32 scalar fields");
        if (c->rels[S->rel].size != c->rels[Q->rel].size)
            return fail(c, EBB_E_SIZE, "peer_send_csr: peer %d: %llu send rows vs %llu remote rows", k,
                        (unsigned long long)c->rels[S->rel].size, (unsigned long long)c->rels[Q->rel].size);
        if (peers[k] < 0 || peers[k] >= EBB_MAX_RANKS) return fail(c, EBB_E_ARG, "peer_send_csr: bad peer rank");
        n += c->rels[S->rel].size;
    }
    if (n >= 0xffffffffull) return fail(c, EBB_E_SIZE, "peer_send_csr: too many entries");
    ebb_rel roff, rdst;
    EBB_TRY(ebb_relation_new(ctx, (nm + ".off").c_str(), n_src + 1, &roff));
    EBB_TRY(new_internal_field(c, roff, "off", EBB_U32, 1, 1, EBB_AOS, send_off));
    EBB_TRY(ebb_relation_new(ctx, (nm + ".dst").c_str(), n ? n : 1, &rdst));
    EBB_TRY(new_internal_field(c, rdst, "dst", EBB_U32, 2, 1, EBB_AOS, send_dst));
    const unsigned B = 256;
    Buf key, key2, val, bad, tmp;
    EBB_CUDA(c, key.alloc(n * 4));
    EBB_CUDA(c, key2.alloc(n * 4));
    EBB_CUDA(c, val.alloc(n * 8));
    EBB_CUDA(c, bad.alloc(4));
    EBB_CUDA(c, cudaMemset(bad.p, 0, 4));
    uint64_t at = 0;
    for (int k = 0; k < npeers; ++k) {
        Field* S = get_field(c, send_rows[k]);
        Field* Q = get_field(c, remote_rows[k]);
        const uint64_t m = c->rels[S->rel].size;
        if (m == 0) continue;
        kpe_fill<<<grid_for(m, B), B>>>((const uint32_t*)S->ptr, (const uint32_t*)Q->ptr, m, (uint32_t)peers[k],
                                        n_src, peer_nv[k], key.as<uint32_t>() + at, val.as<uint64_t>() + at,
                                        bad.as<unsigned int>());
        EBB_CUDA(c, cudaGetLastError());
        at += m;
    }
    uint64_t* dst = (uint64_t*)c->fields[*send_dst].ptr;
    if (n > 0) {
        // stable radix sort by local row: the entries of a vertex keep the peers[] order
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, key.as<uint32_t>(), key2.as<uint32_t>(), val.as<uint64_t>(), dst,
                                        (int)n, 0, 32);
        EBB_CUDA(c, tmp.alloc(tb));
        EBB_CUDA(c, cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.as<uint32_t>(), key2.as<uint32_t>(),
                                                    val.as<uint64_t>(), dst, (int)n, 0, 32));
    }
    kpe_offsets<<<grid_for(n_src + 1, B), B>>>(key2.as<uint32_t>(), n, n_src,
                                                 (uint32_t*)c->fields[*send_off].ptr);
    EBB_CUDA(c, cudaGetLastError());
    unsigned int hb = 0;
    EBB_CUDA(c, cudaMemcpy(&hb, bad.p, 4, cudaMemcpyDeviceToHost));
    if (hb) return fail(c, EBB_E_RANGE, "peer_send_csr: %u rows out of range (local rows < n_src, remote < peer_nv)", hb);
    return EBB_OK;
}

ebb_status ebb_ipc_handle(ebb_ctx ctx, ebb_field f, void* handle64) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !handle64) return EBB_E_ARG;
    Field* F = get_field(c, f);
    if (!F) return fail(c, EBB_E_ARG, "ipc_handle: bad field");
    if (!F->owned) return fail(c, EBB_E_TYPE, "ipc_handle: '%s' is borrowed memory", F->name.c_str());
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "64-byte IPC handle");
    cudaIpcMemHandle_t h;
    EBB_CUDA(c, cudaIpcGetMemHandle(&h, F->ptr));
    memcpy(handle64, &h, 64);
    return EBB_OK;
}

ebb_status ebb_ipc_open(ebb_ctx ctx, const void* handle64, uint64_t* dev_addr) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !handle64 || !dev_addr) return EBB_E_ARG;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    void* p = nullptr;
    EBB_CUDA(c, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    *dev_addr = (uint64_t)(uintptr_t)p;
    return EBB_OK;
}

ebb_status ebb_ipc_close(ebb_ctx ctx, uint64_t dev_addr) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !dev_addr) return EBB_E_ARG;
    EBB_CUDA(c, cudaIpcCloseMemHandle((void*)(uintptr_t)dev_addr));
    return EBB_OK;
}

}  // extern "C"
