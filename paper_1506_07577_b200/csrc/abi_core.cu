// abi_core.cu -- context, relations, fields, key-fields, globals, GroupBy.
//
// The relational runtime of the paper's L1 layer, re-designed as a
// C ABI over device-resident SoA/AoS columns.  Setup calls are synchronous and
// may allocate; the per-step calls (maps, CG) never allocate.
#include <cub/cub.cuh>

#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "ebb_internal.cuh"

using namespace ebb;

namespace ebb {

size_t dtype_size(ebb_dtype d) {
    switch (d) {
        case EBB_F32: return 4;
        case EBB_F64: return 8;
        case EBB_I32: return 4;
        case EBB_I64: return 8;
        case EBB_U8: return 1;
        case EBB_U32: return 4;
        case EBB_KEY: return 4;
    }
    return 0;
}

ebb_status fail(Ctx* c, ebb_status code, const char* fmt, ...) {
    if (c) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof(buf), fmt, ap);
        va_end(ap);
        c->err = buf;
    }
    return code;
}

ebb_status cuda_fail(Ctx* c, cudaError_t e, const char* where) {
    cudaGetLastError();
    return fail(c, e == cudaErrorMemoryAllocation ? EBB_E_NOMEM : EBB_E_CUDA, "CUDA error %s in %s",
                cudaGetErrorString(e), where);
}

Field* get_field(Ctx* c, ebb_field f) {
    if (!c || f >= c->fields.size() || !c->fields[f].alive) return nullptr;
    return &c->fields[f];
}

Relation* get_rel(Ctx* c, ebb_rel r) {
    if (!c || r >= c->rels.size() || !c->rels[r].alive) return nullptr;
    return &c->rels[r];
}

ebb_status scratch_reserve(Ctx* c, size_t bytes) {
    if (bytes <= c->scratch_bytes) return EBB_OK;
    if (c->scratch) cudaFree(c->scratch);
    c->scratch = nullptr;
    c->scratch_bytes = 0;
    EBB_CUDA(c, cudaMalloc(&c->scratch, bytes));
    c->scratch_bytes = bytes;
    return EBB_OK;
}

}  // namespace ebb

namespace {

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

ebb_status add_field(Ctx* c, ebb_rel rel, const char* name, ebb_dtype dt, uint32_t rows, uint32_t cols,
                     ebb_layout layout, void* ptr, bool owned, ebb_field* out) {
    Relation* R = get_rel(c, rel);
    if (!R) return fail(c, EBB_E_ARG, "bad relation handle %u", rel);
    if (!name || !*name) return fail(c, EBB_E_ARG, "field name is empty");
    // vectors/matrices up to 4x4 (Ebb's small types); column vectors up to 32
    // rows (per-element state records, e.g. the 26-word StVK stiffness state)
    if (rows == 0 || cols == 0 || cols > 4 || rows > (cols == 1 ? 32u : 4u))
        return fail(c, EBB_E_SIZE, "field shape %ux%u", rows, cols);
    if (dtype_size(dt) == 0) return fail(c, EBB_E_ARG, "bad dtype %d", (int)dt);
    if (layout != EBB_AOS && layout != EBB_SOA) return fail(c, EBB_E_ARG, "bad layout");
    for (ebb_field f : R->fields)
        if (c->fields[f].alive && c->fields[f].name == name)
            return fail(c, EBB_E_DUP, "field '%s' already exists on relation '%s'", name, R->name.c_str());
    Field F;
    F.name = name;
    F.rel = rel;
    F.dtype = dt;
    F.rows = rows;
    F.cols = cols;
    F.layout = layout;
    F.ptr = ptr;
    F.owned = owned;
    F.alive = true;
    c->fields.push_back(F);
    ebb_field h = (ebb_field)(c->fields.size() - 1);
    R->fields.push_back(h);
    *out = h;
    return EBB_OK;
}

// ---- layout conversion kernels (element-major host order <-> SoA planes)
template <typename T>
__global__ void k_aos_to_soa(const T* __restrict__ in, T* __restrict__ out, uint64_t n, uint32_t comps) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n * comps) return;
    uint64_t e = i / comps;
    uint32_t c = (uint32_t)(i % comps);
    out[(uint64_t)c * n + e] = in[i];
}
template <typename T>
__global__ void k_soa_to_aos(const T* __restrict__ in, T* __restrict__ out, uint64_t n, uint32_t comps) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n * comps) return;
    uint64_t e = i / comps;
    uint32_t c = (uint32_t)(i % comps);
    out[i] = in[(uint64_t)c * n + e];
}

ebb_status convert_layout(Ctx* c, const Field& F, uint64_t n, const void* src, void* dst, bool to_soa,
                          cudaStream_t s) {
    uint64_t tot = n * F.comps();
    size_t es = dtype_size(F.dtype);
    unsigned g = grid_for(tot, 256);
    if (es == 8) {
        if (to_soa) k_aos_to_soa<uint64_t><<<g, 256, 0, s>>>((const uint64_t*)src, (uint64_t*)dst, n, F.comps());
        else k_soa_to_aos<uint64_t><<<g, 256, 0, s>>>((const uint64_t*)src, (uint64_t*)dst, n, F.comps());
    } else if (es == 4) {
        if (to_soa) k_aos_to_soa<uint32_t><<<g, 256, 0, s>>>((const uint32_t*)src, (uint32_t*)dst, n, F.comps());
        else k_soa_to_aos<uint32_t><<<g, 256, 0, s>>>((const uint32_t*)src, (uint32_t*)dst, n, F.comps());
    } else {
        if (to_soa) k_aos_to_soa<uint8_t><<<g, 256, 0, s>>>((const uint8_t*)src, (uint8_t*)dst, n, F.comps());
        else k_soa_to_aos<uint8_t><<<g, 256, 0, s>>>((const uint8_t*)src, (uint8_t*)dst, n, F.comps());
    }
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

template <typename D, typename S>
__global__ void k_convert(D* __restrict__ d, const S* __restrict__ s, uint64_t n) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) d[i] = (D)s[i];
}

template <typename T>
__global__ void k_fill(T* p, uint64_t n, T v) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// bounds check of u32 keys written into an existing key-field
__global__ void k_keys_check(const uint32_t* __restrict__ in, uint64_t n, uint64_t target_size,
                             unsigned long long* bad_count) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n && in[i] >= target_size) atomicAdd(bad_count, 1ull);
}

// bounds check + narrowing of uint64 keys to uint32 storage
__global__ void k_keys_narrow(const uint64_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t n,
                              uint64_t target_size, unsigned long long* bad_count,
                              unsigned long long* first_bad) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t k = in[i];
    if (k >= target_size) {
        atomicAdd(bad_count, 1ull);
        atomicMin(first_bad, (unsigned long long)i);
        out[i] = 0;
    } else {
        out[i] = (uint32_t)k;
    }
}

// gathers for permutations
template <typename T>
__global__ void k_gather_rows(const T* __restrict__ in, T* __restrict__ out, const uint32_t* __restrict__ new_to_old,
                              uint64_t n, uint32_t comps, int soa) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n * comps) return;
    if (soa) {
        uint64_t c = i / n, e = i % n;
        out[i] = in[c * n + new_to_old[e]];
    } else {
        uint64_t e = i / comps, c = i % comps;
        out[i] = in[(uint64_t)new_to_old[e] * comps + c];
    }
}

__global__ void k_remap_keys(uint32_t* keys, uint64_t n, const uint32_t* __restrict__ old_to_new) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) keys[i] = old_to_new[keys[i]];
}

// halo pack / unpack: element = `words` 32-bit words
__global__ void k_rows_gather(const uint32_t* __restrict__ f, const uint32_t* __restrict__ rows, uint32_t* __restrict__ buf,
                              uint64_t n, uint32_t words) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n * words) return;
    uint64_t k = i / words, w = i % words;
    buf[i] = f[(uint64_t)rows[k] * words + w];
}
__global__ void k_rows_scatter(uint32_t* __restrict__ f, const uint32_t* __restrict__ rows, const uint32_t* __restrict__ buf,
                               uint64_t n, uint32_t words) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n * words) return;
    uint64_t k = i / words, w = i % words;
    f[(uint64_t)rows[k] * words + w] = buf[i];
}

// component-planar (SOA) fields: component q of row r at f[q N + r]; the
// buffer stays element-major (AOS)
template <typename T>
__global__ void k_rows_gather_soa(const T* __restrict__ f, uint64_t N, const uint32_t* __restrict__ rows,
                                  T* __restrict__ buf, uint64_t n, uint32_t comps) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n * comps) return;
    uint64_t k = i / comps, q = i % comps;
    buf[i] = f[q * N + rows[k]];
}
template <typename T>
__global__ void k_rows_scatter_soa(T* __restrict__ f, uint64_t N, const uint32_t* __restrict__ rows,
                                   const T* __restrict__ buf, uint64_t n, uint32_t comps, int add) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n * comps) return;
    uint64_t k = i / comps, q = i % comps;
    T* d = f + q * N + rows[k];
    *d = add ? *d + buf[i] : buf[i];
}

template <typename T>
__global__ void k_rows_add_aos(T* __restrict__ f, const uint32_t* __restrict__ rows, const T* __restrict__ buf,
                               uint64_t n, uint32_t comps) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n * comps) return;
    uint64_t k = i / comps, q = i % comps;
    f[(uint64_t)rows[k] * comps + q] += buf[i];
}

__global__ void k_iota(uint32_t* p, uint64_t n) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = (uint32_t)i;
}

__global__ void k_invert_perm(const uint32_t* __restrict__ new_to_old, uint32_t* __restrict__ old_to_new, uint64_t n) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) old_to_new[new_to_old[i]] = (uint32_t)i;
}

// row_ptr[s] = first position with sorted_key >= s (lower bound), s in [0, ns]
__global__ void k_lower_bound_index(const uint32_t* __restrict__ sorted, uint64_t n, uint32_t* __restrict__ index,
                                    uint64_t ns) {
    uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (s > ns) return;
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if (sorted[mid] < s) lo = mid + 1;
        else hi = mid;
    }
    index[s] = (uint32_t)lo;
}

__global__ void k_index_stats(const uint32_t* __restrict__ index, uint64_t ns, unsigned int* out) {
    const uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (s >= ns) return;
    atomicMax(out, index[s + 1] - index[s]);
    if (s % 16 == 0) atomicMax(out + 1, index[s + 16 < ns ? s + 16 : ns] - index[s]);
    if (s % 64 == 0) atomicMax(out + 2, index[s + 64 < ns ? s + 64 : ns] - index[s]);
}


}  // namespace

namespace ebb {

ebb_status new_internal_field(Ctx* c, ebb_rel rel, const std::string& name, ebb_dtype dt, uint32_t rows,
                              uint32_t cols, ebb_layout layout, ebb_field* out) {
    Relation* R = get_rel(c, rel);
    size_t bytes = (size_t)R->size * rows * cols * dtype_size(dt);
    void* p = nullptr;
    if (bytes) {
        // +64 B tail slack: bulk async copies round segment ends up to 16 B
        EBB_CUDA(c, cudaMalloc(&p, bytes + kFieldSlack));
        EBB_CUDA(c, cudaMemset(p, 0, bytes + kFieldSlack));
    }
    ebb_status st = add_field(c, rel, name.c_str(), dt, rows, cols, layout, p, true, out);
    if (st != EBB_OK && p) cudaFree(p);
    return st;
}

ebb_status index_stats(Ctx* c, const uint32_t* index, uint64_t ns, uint32_t out[3]) {
    unsigned int* d = nullptr;
    EBB_CUDA(c, cudaMalloc(&d, 16));
    cudaError_t e = cudaMemset(d, 0, 16);
    if (e == cudaSuccess && ns) {
        k_index_stats<<<grid_for(ns, 256), 256>>>(index, ns, d);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(out, d, 12, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return cuda_fail(c, e, "index_stats");
    return EBB_OK;
}

void release_plans(Ctx* c) {
    for (SegPlan* P : c->segplans) {
        P->release();
        delete P;
    }
    c->segplans.clear();
    for (ChunkPlan* P : c->chunkplans) {
        P->release();
        delete P;
    }
    c->chunkplans.clear();
    c->auto_map.clear();
    for (ColorPlan* P : c->colorplans) {
        P->release();
        delete P;
    }
    c->colorplans.clear();
    for (UpperCSR* U : c->uppers) {
        U->release();
        delete U;
    }
    c->uppers.clear();
}

// Apply a row permutation to every field of `rel` and remap every key-field
// (anywhere in the context) that targets `rel`.  The paper's licence: the
// runtime may reorder relations and re-encode keys.
ebb_status permute_relation(Ctx* c, ebb_rel rel, const uint32_t* d_new_to_old, const uint32_t* d_old_to_new,
                            cudaStream_t s) {
    Relation* R = get_rel(c, rel);
    uint64_t n = R->size;
    // a grouping is a sorted order of `rel` plus a CSR index on the
    // key's target: permuting either side silently invalidates it
    if (R->grouped_by != EBB_NONE)
        return fail(c, EBB_E_STATE, "relation '%s' is grouped: reorder it before ebb_group_by", R->name.c_str());
    if (R->index != EBB_NONE)
        return fail(c, EBB_E_STATE, "relation '%s' is the target of a grouping (it holds a group index): "
                    "reorder it before ebb_group_by", R->name.c_str());
    release_plans(c);
    for (ebb_field fh : R->fields) {
        Field& F = c->fields[fh];
        if (!F.alive) continue;
        size_t es = dtype_size(F.dtype);
        uint64_t tot = n * F.comps();
        void* np = nullptr;
        EBB_CUDA(c, cudaMalloc(&np, tot * es + kFieldSlack));
        EBB_CUDA(c, cudaMemset(np, 0, tot * es + kFieldSlack));
        unsigned g = grid_for(tot, 256);
        int soa = F.layout == EBB_SOA;
        if (es == 8)
            k_gather_rows<uint64_t><<<g, 256, 0, s>>>((const uint64_t*)F.ptr, (uint64_t*)np, d_new_to_old, n, F.comps(), soa);
        else if (es == 4)
            k_gather_rows<uint32_t><<<g, 256, 0, s>>>((const uint32_t*)F.ptr, (uint32_t*)np, d_new_to_old, n, F.comps(), soa);
        else
            k_gather_rows<uint8_t><<<g, 256, 0, s>>>((const uint8_t*)F.ptr, (uint8_t*)np, d_new_to_old, n, F.comps(), soa);
        EBB_CUDA(c, cudaGetLastError());
        if (F.owned) {
            EBB_CUDA(c, cudaStreamSynchronize(s));
            cudaFree(F.ptr);
            F.ptr = np;
        } else {
            // borrowed memory keeps its address: copy back in place
            EBB_CUDA(c, cudaMemcpyAsync(F.ptr, np, tot * es, cudaMemcpyDeviceToDevice, s));
            EBB_CUDA(c, cudaStreamSynchronize(s));
            cudaFree(np);
        }
    }
    for (Field& F : c->fields) {
        if (!F.alive || F.dtype != EBB_KEY || F.key_target != rel) continue;
        uint64_t tot = c->rels[F.rel].size * F.comps();
        k_remap_keys<<<grid_for(tot, 256), 256, 0, s>>>((uint32_t*)F.ptr, tot, d_old_to_new);
        EBB_CUDA(c, cudaGetLastError());
    }
    // a grouping of rel or an index on rel is no longer valid unless rebuilt
    EBB_CUDA(c, cudaStreamSynchronize(s));
    return EBB_OK;
}

}  // namespace ebb

extern "C" {

const char* ebb_version(void) { return "ebb-b200 0.1 (sm_100a)"; }

ebb_status ebb_ctx_new(int device, ebb_ctx* out) {
    if (!out) return EBB_E_ARG;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
        cudaGetLastError();
        return EBB_E_CUDA;
    }
    Ctx* c = new Ctx();
    c->device = device;
    EBB_DEVICE_GUARD(c);   // allocate on `device`, leave the caller's device current
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (cudaMalloc(&c->d_err, 4 * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMemset(c->d_err, 0, 4 * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&c->d_partials, 8 * 8192 * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&c->d_counter, 64 * sizeof(unsigned int)) != cudaSuccess ||
        cudaMemset(c->d_counter, 0, 64 * sizeof(unsigned int)) != cudaSuccess) {
        delete c;
        return EBB_E_CUDA;
    }
    Relation g;
    g.name = "__globals";
    g.size = 1;
    c->rels.push_back(g);
    c->globals_rel = 0;
    *out = c;
    return EBB_OK;
}

ebb_status ebb_ctx_free(ebb_ctx ctx) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c) return EBB_E_ARG;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    for (Field& F : c->fields)
        if (F.alive && F.owned && F.ptr) cudaFree(F.ptr);
    if (c->scratch) cudaFree(c->scratch);
    for (auto& e : c->ev_pool) cudaEventDestroy(e);
    release_plans(c);
    comm_release(c);
    peer_release(c);
    for (auto& G : c->graphs)
        if (G.exec) cudaGraphExecDestroy(G.exec);
    cudaFree(c->d_err);
    cudaFree(c->d_partials);
    cudaFree(c->d_counter);
    delete c;
    return EBB_OK;
}

const char* ebb_last_error(ebb_ctx ctx) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    return c ? c->err.c_str() : "null context";
}

ebb_status ebb_error_counts(ebb_ctx ctx, uint64_t out[4], int reset) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !out) return EBB_E_ARG;
    EBB_CUDA(c, cudaDeviceSynchronize());
    unsigned long long h[4];
    EBB_CUDA(c, cudaMemcpy(h, c->d_err, sizeof(h), cudaMemcpyDeviceToHost));
    for (int i = 0; i < 4; ++i) out[i] = h[i];
    if (reset) EBB_CUDA(c, cudaMemset(c->d_err, 0, sizeof(h)));
    return EBB_OK;
}

ebb_status ebb_sync(ebb_ctx ctx, ebb_stream s) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c) return EBB_E_ARG;
    EBB_CUDA(c, cudaStreamSynchronize((cudaStream_t)s));
    return EBB_OK;
}

ebb_status ebb_timing_enable(ebb_ctx ctx, int on) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c) return EBB_E_ARG;
    if (on && c->ev_pool.empty()) {
        c->ev_pool.resize(16384);
        for (auto& e : c->ev_pool) EBB_CUDA(c, cudaEventCreate(&e));
    }
    c->timing = on != 0;
    return EBB_OK;
}

ebb_status ebb_timing_read(ebb_ctx ctx, int32_t kernel, double* total_ms, uint64_t* launches, int reset) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !total_ms || !launches) return EBB_E_ARG;
    double tot = 0.0;
    uint64_t n = 0;
    for (auto& t : c->timed) {
        if (t.kernel != kernel) continue;
        EBB_CUDA(c, cudaEventSynchronize(t.b));
        float ms = 0.f;
        EBB_CUDA(c, cudaEventElapsedTime(&ms, t.a, t.b));
        tot += ms;
        ++n;
    }
    *total_ms = tot;
    *launches = n;
    if (reset) {
        EBB_CUDA(c, cudaDeviceSynchronize());
        c->timed.clear();
        c->ev_used = 0;
    }
    return EBB_OK;
}

ebb_status ebb_launch_count(ebb_ctx ctx, uint64_t* out, int reset) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !out) return EBB_E_ARG;
    *out = c->launches;
    if (reset) c->launches = 0;
    return EBB_OK;
}

ebb_status ebb_graph_begin(ebb_ctx ctx, ebb_stream s) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c) return EBB_E_ARG;
    if (!s) return fail(c, EBB_E_ARG, "graph capture needs a non-default stream");
    EBB_CUDA(c, cudaStreamBeginCapture((cudaStream_t)s, cudaStreamCaptureModeThreadLocal));
    c->capture_launch0 = c->launches;
    return EBB_OK;
}

ebb_status ebb_graph_end(ebb_ctx ctx, ebb_stream s, int32_t* graph_out) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !graph_out || !s) return fail(c, EBB_E_ARG, "bad argument");
    cudaGraph_t g = nullptr;
    EBB_CUDA(c, cudaStreamEndCapture((cudaStream_t)s, &g));
    Ctx::GraphRec r;
    cudaError_t e = cudaGraphInstantiate(&r.exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaGraphInstantiate");
    r.launches = c->launches - c->capture_launch0;
    c->graphs.push_back(r);
    *graph_out = (int32_t)(c->graphs.size() - 1);
    return EBB_OK;
}

ebb_status ebb_graph_launch(ebb_ctx ctx, int32_t graph, ebb_stream s) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || graph < 0 || (size_t)graph >= c->graphs.size() || !c->graphs[graph].exec)
        return fail(c, EBB_E_ARG, "bad graph handle");
    EBB_CUDA(c, cudaGraphLaunch(c->graphs[graph].exec, (cudaStream_t)s));
    c->launches += c->graphs[graph].launches;
    return EBB_OK;
}

ebb_status ebb_graph_free(ebb_ctx ctx, int32_t graph) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || graph < 0 || (size_t)graph >= c->graphs.size()) return EBB_E_ARG;
    if (c->graphs[graph].exec) cudaGraphExecDestroy(c->graphs[graph].exec);
    c->graphs[graph].exec = nullptr;
    return EBB_OK;
}

ebb_status ebb_relation_new(ebb_ctx ctx, const char* name, uint64_t size, ebb_rel* out) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !name || !out) return fail(c, EBB_E_ARG, "null argument");
    if (size == 0) return fail(c, EBB_E_SIZE, "relation '%s' has zero size", name);
    for (auto& R : c->rels)
        if (R.alive && R.name == name) return fail(c, EBB_E_DUP, "relation '%s' already exists", name);
    Relation R;
    R.name = name;
    R.size = size;
    c->rels.push_back(R);
    *out = (ebb_rel)(c->rels.size() - 1);
    return EBB_OK;
}

ebb_status ebb_relation_size(ebb_ctx ctx, ebb_rel rel, uint64_t* out) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    Relation* R = get_rel(c, rel);
    if (!R || !out) return fail(c, EBB_E_ARG, "bad relation");
    *out = R->size;
    return EBB_OK;
}

ebb_status ebb_field_new(ebb_ctx ctx, ebb_rel rel, const char* name, ebb_dtype dtype, uint32_t rows, uint32_t cols,
                         ebb_layout layout, const void* host_init, ebb_field* out) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !out) return fail(c, EBB_E_ARG, "null argument");
    if (dtype == EBB_KEY) return fail(c, EBB_E_TYPE, "use ebb_key_field for key-fields");
    ebb_field h;
    EBB_TRY(new_internal_field(c, rel, name ? name : "", dtype, rows, cols, layout, &h));
    Field& F = c->fields[h];
    if (host_init) {
        uint64_t nbytes = c->rels[rel].size * F.comps() * dtype_size(dtype);
        ebb_status st = ebb_field_write(ctx, h, host_init, nbytes, nullptr);
        if (st != EBB_OK) return st;
        EBB_CUDA(c, cudaDeviceSynchronize());
    }
    *out = h;
    return EBB_OK;
}

ebb_status ebb_field_wrap(ebb_ctx ctx, ebb_rel rel, const char* name, ebb_dtype dtype, uint32_t rows, uint32_t cols,
                          ebb_layout layout, void* device_ptr, ebb_field* out) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !out || !device_ptr) return fail(c, EBB_E_ARG, "null argument");
    if (dtype == EBB_KEY) return fail(c, EBB_E_TYPE, "key-fields must be created by ebb_key_field");
    return add_field(c, rel, name, dtype, rows, cols, layout, device_ptr, false, out);
}

ebb_status ebb_field_find(ebb_ctx ctx, ebb_rel rel, const char* name, ebb_field* out) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    Relation* R = get_rel(c, rel);
    if (!R || !name || !out) return fail(c, EBB_E_ARG, "bad argument");
    for (ebb_field f : R->fields)
        if (c->fields[f].alive && c->fields[f].name == name) {
            *out = f;
            return EBB_OK;
        }
    return fail(c, EBB_E_ARG, "no field '%s' on relation '%s'", name, R->name.c_str());
}

ebb_status ebb_field_write(ebb_ctx ctx, ebb_field f, const void* host, uint64_t nbytes, ebb_stream s) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    Field* F = get_field(c, f);
    if (!F || !host) return fail(c, EBB_E_ARG, "bad field or null host pointer");
    uint64_t n = c->rels[F->rel].size;
    uint64_t want = n * F->comps() * dtype_size(F->dtype);
    if (nbytes != want) return fail(c, EBB_E_SIZE, "field '%s': %llu bytes given, %llu expected", F->name.c_str(),
                                    (unsigned long long)nbytes, (unsigned long long)want);
    cudaStream_t st = (cudaStream_t)s;
    if (F->dtype == EBB_KEY) {
        // keys stay in bounds by construction: check the new keys
        // before they replace the old ones; plans built on the old
        // connectivity are dropped; a grouping key cannot be rewritten
        if (c->rels[F->rel].grouped_by == f)
            return fail(c, EBB_E_STATE, "key-field '%s' groups its relation: it cannot be rewritten", F->name.c_str());
        EBB_TRY(scratch_reserve(c, nbytes + 16));
        unsigned long long* bad = (unsigned long long*)((char*)c->scratch + ((nbytes + 7) & ~7ull));
        EBB_CUDA(c, cudaMemcpyAsync(c->scratch, host, nbytes, cudaMemcpyHostToDevice, st));
        EBB_CUDA(c, cudaMemsetAsync(bad, 0, 8, st));
        const uint64_t nk = n * F->comps();
        k_keys_check<<<grid_for(nk, 256), 256, 0, st>>>((const uint32_t*)c->scratch, nk, c->rels[F->key_target].size, bad);
        EBB_CUDA(c, cudaGetLastError());
        unsigned long long hb = 0;
        EBB_CUDA(c, cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, st));
        EBB_CUDA(c, cudaStreamSynchronize(st));
        if (hb) return fail(c, EBB_E_BOUNDS, "key-field '%s': %llu keys out of range of '%s'", F->name.c_str(), hb,
                            c->rels[F->key_target].name.c_str());
        release_plans(c);
        EBB_CUDA(c, cudaMemcpyAsync(F->ptr, c->scratch, nbytes, cudaMemcpyDeviceToDevice, st));
        return EBB_OK;
    }
    if (F->layout == EBB_AOS || F->comps() == 1) {
        EBB_CUDA(c, cudaMemcpyAsync(F->ptr, host, nbytes, cudaMemcpyHostToDevice, st));
        return EBB_OK;
    }
    EBB_TRY(scratch_reserve(c, nbytes));
    EBB_CUDA(c, cudaMemcpyAsync(c->scratch, host, nbytes, cudaMemcpyHostToDevice, st));
    return convert_layout(c, *F, n, c->scratch, F->ptr, true, st);
}

ebb_status ebb_field_read(ebb_ctx ctx, ebb_field f, void* host, uint64_t nbytes, ebb_stream s) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    Field* F = get_field(c, f);
    if (!F || !host) return fail(c, EBB_E_ARG, "bad field or null host pointer");
    uint64_t n = c->rels[F->rel].size;
    uint64_t want = n * F->comps() * dtype_size(F->dtype);
    if (nbytes != want) return fail(c, EBB_E_SIZE, "field '%s': %llu bytes given, %llu expected", F->name.c_str(),
                                    (unsigned long long)nbytes, (unsigned long long)want);
    cudaStream_t st = (cudaStream_t)s;
    if (F->layout == EBB_AOS || F->comps() == 1) {
        EBB_CUDA(c, cudaMemcpyAsync(host, F->ptr, nbytes, cudaMemcpyDeviceToHost, st));
    } else {
        EBB_TRY(scratch_reserve(c, nbytes));
        EBB_TRY(convert_layout(c, *F, n, F->ptr, c->scratch, false, st));
        EBB_CUDA(c, cudaMemcpyAsync(host, c->scratch, nbytes, cudaMemcpyDeviceToHost, st));
    }
    EBB_CUDA(c, cudaStreamSynchronize(st));
    return EBB_OK;
}

ebb_status ebb_field_read_async(ebb_ctx ctx, ebb_field f, void* host, uint64_t nbytes, ebb_stream s) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    Field* F = get_field(c, f);
    if (!F || !host) return fail(c, EBB_E_ARG, "bad field or null host pointer");
    uint64_t n = c->rels[F->rel].size;
    uint64_t want = n * F->comps() * dtype_size(F->dtype);
    if (nbytes != want) return fail(c, EBB_E_SIZE, "field '%s': %llu bytes given, %llu expected", F->name.c_str(),
                                    (unsigned long long)nbytes, (unsigned long long)want);
    if (F->layout != EBB_AOS && F->comps() != 1)
        return fail(c, EBB_E_TYPE, "read_async: '%s' is component-planar (use ebb_field_read)", F->name.c_str());
    EBB_CUDA(c, cudaMemcpyAsync(host, F->ptr, nbytes, cudaMemcpyDeviceToHost, (cudaStream_t)s));
    return EBB_OK;
}

ebb_status ebb_field_fill(ebb_ctx ctx, ebb_field f, double value, ebb_stream s) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    Field* F = get_field(c, f);
    if (!F) return fail(c, EBB_E_ARG, "bad field");
    if (F->dtype == EBB_KEY) return fail(c, EBB_E_TYPE, "cannot fill a key-field");
    uint64_t n = c->rels[F->rel].size * F->comps();
    cudaStream_t st = (cudaStream_t)s;
    unsigned g = grid_for(n, 256);
    switch (F->dtype) {
        case EBB_F32: k_fill<float><<<g, 256, 0, st>>>((float*)F->ptr, n, (float)value); break;
        case EBB_F64: k_fill<double><<<g, 256, 0, st>>>((double*)F->ptr, n, value); break;
        case EBB_I32: k_fill<int32_t><<<g, 256, 0, st>>>((int32_t*)F->ptr, n, (int32_t)value); break;
        case EBB_I64: k_fill<int64_t><<<g, 256, 0, st>>>((int64_t*)F->ptr, n, (int64_t)value); break;
        case EBB_U32: k_fill<uint32_t><<<g, 256, 0, st>>>((uint32_t*)F->ptr, n, (uint32_t)value); break;
        case EBB_U8: k_fill<uint8_t><<<g, 256, 0, st>>>((uint8_t*)F->ptr, n, (uint8_t)value); break;
        default: return fail(c, EBB_E_TYPE, "bad dtype");
    }
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status ebb_field_copy(ebb_ctx ctx, ebb_field dst, ebb_field src, ebb_stream s) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    Field* D = get_field(c, dst);
    Field* S = get_field(c, src);
    if (!D || !S) return fail(c, EBB_E_ARG, "bad field");
    if (D->dtype != S->dtype || D->comps() != S->comps() || D->layout != S->layout ||
        c->rels[D->rel].size != c->rels[S->rel].size)
        return fail(c, EBB_E_TYPE, "field_copy: '%s' and '%s' differ in type/shape/layout", D->name.c_str(),
                    S->name.c_str());
    if (D->dtype == EBB_KEY) {
        if (D->key_target != S->key_target)
            return fail(c, EBB_E_TYPE, "field_copy: key-fields '%s' and '%s' target different relations",
                        D->name.c_str(), S->name.c_str());
        if (c->rels[D->rel].grouped_by == dst)
            return fail(c, EBB_E_STATE, "key-field '%s' groups its relation: it cannot be rewritten", D->name.c_str());
        release_plans(c);
    }
    uint64_t nbytes = c->rels[D->rel].size * D->comps() * dtype_size(D->dtype);
    EBB_CUDA(c, cudaMemcpyAsync(D->ptr, S->ptr, nbytes, cudaMemcpyDeviceToDevice, (cudaStream_t)s));
    return EBB_OK;
}

ebb_status ebb_field_convert(ebb_ctx ctx, ebb_field dst, ebb_field src, ebb_stream s) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    Field* D = get_field(c, dst);
    Field* S = get_field(c, src);
    if (!D || !S) return fail(c, EBB_E_ARG, "bad field");
    bool fl = (D->dtype == EBB_F32 || D->dtype == EBB_F64) && (S->dtype == EBB_F32 || S->dtype == EBB_F64);
    if (!fl || D->comps() != S->comps() || D->layout != S->layout || c->rels[D->rel].size != c->rels[S->rel].size)
        return fail(c, EBB_E_TYPE, "field_convert: '%s' <- '%s' needs float fields of equal shape/layout/size",
                    D->name.c_str(), S->name.c_str());
    if (D->dtype == S->dtype) return ebb_field_copy(ctx, dst, src, s);
    uint64_t n = c->rels[D->rel].size * D->comps();
    if (D->dtype == EBB_F32)
        k_convert<float, double><<<grid_for(n, 256), 256, 0, (cudaStream_t)s>>>((float*)D->ptr, (const double*)S->ptr, n);
    else
        k_convert<double, float><<<grid_for(n, 256), 256, 0, (cudaStream_t)s>>>((double*)D->ptr, (const float*)S->ptr, n);
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status ebb_field_view(ebb_ctx ctx, ebb_field f, ebb_view* out) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    Field* F = get_field(c, f);
    if (!F || !out) return fail(c, EBB_E_ARG, "bad field");
    uint64_t n = c->rels[F->rel].size;
    size_t es = dtype_size(F->dtype);
    out->data = F->ptr;
    out->count = n;
    out->rows = F->rows;
    out->cols = F->cols;
    out->dtype = F->dtype;
    out->layout = F->layout;
    if (F->layout == EBB_AOS) {
        out->elem_stride = es * F->comps();
        out->comp_stride = es;
    } else {
        out->elem_stride = es;
        out->comp_stride = es * n;
    }
    out->rel = F->rel;
    out->key_target = F->key_target;
    return EBB_OK;
}

ebb_status ebb_key_field(ebb_ctx ctx, ebb_rel owner, const char* name, ebb_rel target, uint32_t rows, uint32_t cols,
                         const uint64_t* keys, int keys_on_device, ebb_field* out) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !keys || !out) return fail(c, EBB_E_ARG, "null argument");
    Relation* O = get_rel(c, owner);
    Relation* T = get_rel(c, target);
    if (!O || !T) return fail(c, EBB_E_ARG, "bad relation handle");
    if (T->size > 0xFFFFFFFFull) return fail(c, EBB_E_RANGE, "target relation '%s' exceeds 2^32-1 rows", T->name.c_str());
    ebb_field h;
    EBB_TRY(new_internal_field(c, owner, name ? name : "", EBB_KEY, rows, cols, EBB_AOS, &h));
    c->fields[h].key_target = target;
    uint64_t n = O->size * rows * cols;
    DevBuf in;
    const uint64_t* dkeys = keys;
    if (!keys_on_device) {
        EBB_CUDA(c, cudaMalloc(&in.p, n * 8));
        EBB_CUDA(c, cudaMemcpy(in.p, keys, n * 8, cudaMemcpyHostToDevice));
        dkeys = (const uint64_t*)in.p;
    }
    DevBuf flag;
    EBB_CUDA(c, cudaMalloc(&flag.p, 16));
    unsigned long long init[2] = {0ull, ~0ull};
    EBB_CUDA(c, cudaMemcpy(flag.p, init, 16, cudaMemcpyHostToDevice));
    unsigned long long* fl = (unsigned long long*)flag.p;
    k_keys_narrow<<<grid_for(n, 256), 256>>>(dkeys, (uint32_t*)c->fields[h].ptr, n, T->size, fl, fl + 1);
    EBB_CUDA(c, cudaGetLastError());
    unsigned long long res[2];
    EBB_CUDA(c, cudaMemcpy(res, flag.p, 16, cudaMemcpyDeviceToHost));
    if (res[0]) {
        // drop the field again: a key-field is in bounds by construction
        Field& F = c->fields[h];
        cudaFree(F.ptr);
        F.ptr = nullptr;
        F.alive = false;
        O->fields.pop_back();
        return fail(c, EBB_E_BOUNDS, "key-field '%s': %llu keys out of range of '%s' (size %llu); first at flat index %llu",
                    name, res[0], T->name.c_str(), (unsigned long long)T->size, res[1]);
    }
    *out = h;
    return EBB_OK;
}

ebb_status ebb_global_new(ebb_ctx ctx, const char* name, ebb_dtype dtype, double init, ebb_field* out) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !out) return fail(c, EBB_E_ARG, "null argument");
    if (dtype != EBB_F64 && dtype != EBB_F32 && dtype != EBB_I64 && dtype != EBB_I32)
        return fail(c, EBB_E_TYPE, "globals are scalar numeric");
    ebb_field h;
    EBB_TRY(new_internal_field(c, c->globals_rel, name ? name : "", dtype, 1, 1, EBB_AOS, &h));
    c->fields[h].is_global = true;
    EBB_TRY(ebb_global_set(ctx, h, init, nullptr));
    EBB_CUDA(c, cudaDeviceSynchronize());
    *out = h;
    return EBB_OK;
}

ebb_status ebb_global_get(ebb_ctx ctx, ebb_field g, double* out) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    Field* F = get_field(c, g);
    if (!F || !out || !F->is_global) return fail(c, EBB_E_ARG, "not a global");
    EBB_CUDA(c, cudaDeviceSynchronize());
    union { double d; float f; int64_t l; int32_t i; } u;
    EBB_CUDA(c, cudaMemcpy(&u, F->ptr, dtype_size(F->dtype), cudaMemcpyDeviceToHost));
    switch (F->dtype) {
        case EBB_F64: *out = u.d; break;
        case EBB_F32: *out = u.f; break;
        case EBB_I64: *out = (double)u.l; break;
        default: *out = (double)u.i; break;
    }
    return EBB_OK;
}

ebb_status ebb_global_set(ebb_ctx ctx, ebb_field g, double value, ebb_stream s) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    Field* F = get_field(c, g);
    if (!F || !F->is_global) return fail(c, EBB_E_ARG, "not a global");
    return ebb_field_fill(ctx, g, value, s);
}

ebb_status ebb_group_by(ebb_ctx ctx, ebb_rel rel, ebb_field key) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    Relation* R = get_rel(c, rel);
    Field* K = get_field(c, key);
    if (!R || !K) return fail(c, EBB_E_ARG, "bad handle");
    if (K->dtype != EBB_KEY || K->comps() != 1 || K->rel != rel)
        return fail(c, EBB_E_TYPE, "group_by: '%s' is not a scalar key-field of '%s'", K->name.c_str(), R->name.c_str());
    if (R->grouped_by != EBB_NONE) return fail(c, EBB_E_STATE, "relation '%s' is already grouped", R->name.c_str());
    ebb_rel src = K->key_target;
    uint64_t n = R->size, ns = c->rels[src].size;
    if (n > 0xFFFFFFFFull) return fail(c, EBB_E_RANGE, "relation too large for 32-bit keys");
    DevBuf kout, vin, vout, inv, tmp;
    EBB_CUDA(c, cudaMalloc(&kout.p, n * 4));
    EBB_CUDA(c, cudaMalloc(&vin.p, n * 4));
    EBB_CUDA(c, cudaMalloc(&vout.p, n * 4));
    EBB_CUDA(c, cudaMalloc(&inv.p, n * 4));
    k_iota<<<grid_for(n, 256), 256>>>((uint32_t*)vin.p, n);
    size_t tb = 0;
    int end_bit = 1;
    while (end_bit < 32 && (1ull << end_bit) < ns) ++end_bit;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (const uint32_t*)K->ptr, (uint32_t*)kout.p, (const uint32_t*)vin.p,
                                    (uint32_t*)vout.p, (int)n, 0, end_bit);
    EBB_CUDA(c, cudaMalloc(&tmp.p, tb));
    EBB_CUDA(c, cub::DeviceRadixSort::SortPairs(tmp.p, tb, (const uint32_t*)K->ptr, (uint32_t*)kout.p,
                                                (const uint32_t*)vin.p, (uint32_t*)vout.p, (int)n, 0, end_bit));
    k_invert_perm<<<grid_for(n, 256), 256>>>((const uint32_t*)vout.p, (uint32_t*)inv.p, n);
    EBB_CUDA(c, cudaGetLastError());
    EBB_TRY(permute_relation(c, rel, (const uint32_t*)vout.p, (const uint32_t*)inv.p, nullptr));
    // hidden index on the source relation ("range of rows ... encoded as two indices")
    ebb_field idx;
    Relation* Sr = get_rel(c, src);
    std::string iname = "__index_" + R->name;
    // index has ns+1 entries: allocate on a fresh hidden relation of that size
    ebb_rel irel;
    EBB_TRY(ebb_relation_new(ctx, ("__index_rel_" + R->name).c_str(), ns + 1, &irel));
    EBB_TRY(new_internal_field(c, irel, iname, EBB_U32, 1, 1, EBB_AOS, &idx));
    R = get_rel(c, rel);
    Sr = get_rel(c, src);
    K = get_field(c, key);
    k_lower_bound_index<<<grid_for(ns + 1, 256), 256>>>((const uint32_t*)K->ptr, n, (uint32_t*)c->fields[idx].ptr, ns);
    uint32_t st[3];
    EBB_TRY(index_stats(c, (const uint32_t*)c->fields[idx].ptr, ns, st));
    R->grouped_by = key;
    R->index = idx;
    R->max_group = st[0];
    R->max_chunk16 = st[1];
    R->max_chunk64 = st[2];
    Sr->index = idx;
    Sr->max_group = st[0];
    return EBB_OK;
}

static ebb_status rows_common(Ctx* c, ebb_field f, ebb_field rows, ebb_field buf, Field** F, Field** Rw, Field** B,
                              uint64_t* n, uint32_t* words) {
    *F = get_field(c, f);
    *Rw = get_field(c, rows);
    *B = get_field(c, buf);
    if (!*F || !*Rw || !*B) return fail(c, EBB_E_ARG, "rows_gather/scatter: bad handle");
    if ((*F)->layout != EBB_AOS && (*F)->comps() > 1 && (*F)->dtype != EBB_F32 && (*F)->dtype != EBB_F64)
        return fail(c, EBB_E_TYPE, "component-planar halo fields must be F32 or F64");
    if ((*F)->dtype == EBB_KEY) return fail(c, EBB_E_TYPE, "halo rows of a key-field are not supported");
    if ((*Rw)->dtype != EBB_U32 || (*Rw)->comps() != 1) return fail(c, EBB_E_TYPE, "rows must be a U32 scalar field");
    if ((*B)->dtype != (*F)->dtype || (*B)->comps() != (*F)->comps() || (*B)->rel != (*Rw)->rel)
        return fail(c, EBB_E_TYPE, "buf must match f's dtype/shape on the rows' relation");
    size_t eb = (*F)->comps() * dtype_size((*F)->dtype);
    if (eb % 4) return fail(c, EBB_E_TYPE, "halo element size must be a multiple of 4 bytes");
    *words = (uint32_t)(eb / 4);
    *n = c->rels[(*Rw)->rel].size;
    return EBB_OK;
}

// SOA fields (the edge relation's 3x3 K): gather / scatter (+add) per component
static ebb_status rows_soa(Ctx* c, Field* F, Field* Rw, Field* B, uint64_t n, bool gather, int add,
                           cudaStream_t s) {
    const uint64_t N = c->rels[F->rel].size;
    const uint32_t q = F->comps();
    c->launches++;
    if (n == 0) return EBB_OK;
    const unsigned g = grid_for(n * q, 256);
    if (F->dtype == EBB_F64) {
        if (gather) k_rows_gather_soa<double><<<g, 256, 0, s>>>((const double*)F->ptr, N, (const uint32_t*)Rw->ptr,
                                                               (double*)B->ptr, n, q);
        else k_rows_scatter_soa<double><<<g, 256, 0, s>>>((double*)F->ptr, N, (const uint32_t*)Rw->ptr,
                                                          (const double*)B->ptr, n, q, add);
    } else {
        if (gather) k_rows_gather_soa<float><<<g, 256, 0, s>>>((const float*)F->ptr, N, (const uint32_t*)Rw->ptr,
                                                              (float*)B->ptr, n, q);
        else k_rows_scatter_soa<float><<<g, 256, 0, s>>>((float*)F->ptr, N, (const uint32_t*)Rw->ptr,
                                                         (const float*)B->ptr, n, q, add);
    }
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status ebb_rows_gather(ebb_ctx ctx, ebb_field f, ebb_field rows, ebb_field buf, ebb_stream s) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    Field *F, *Rw, *B;
    uint64_t n;
    uint32_t w;
    EBB_TRY(rows_common(c, f, rows, buf, &F, &Rw, &B, &n, &w));
    if (F->layout == EBB_SOA && F->comps() > 1) return rows_soa(c, F, Rw, B, n, true, 0, (cudaStream_t)s);
    c->launches++;
    k_rows_gather<<<grid_for(n * w, 256), 256, 0, (cudaStream_t)s>>>((const uint32_t*)F->ptr, (const uint32_t*)Rw->ptr,
                                                                     (uint32_t*)B->ptr, n, w);
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status ebb_rows_scatter(ebb_ctx ctx, ebb_field f, ebb_field rows, ebb_field buf, ebb_stream s) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    Field *F, *Rw, *B;
    uint64_t n;
    uint32_t w;
    EBB_TRY(rows_common(c, f, rows, buf, &F, &Rw, &B, &n, &w));
    if (F->layout == EBB_SOA && F->comps() > 1) return rows_soa(c, F, Rw, B, n, false, 0, (cudaStream_t)s);
    c->launches++;
    k_rows_scatter<<<grid_for(n * w, 256), 256, 0, (cudaStream_t)s>>>((uint32_t*)F->ptr, (const uint32_t*)Rw->ptr,
                                                                      (const uint32_t*)B->ptr, n, w);
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status ebb_rows_scatter_add(ebb_ctx ctx, ebb_field f, ebb_field rows, ebb_field buf, ebb_stream s) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    Field *F, *Rw, *B;
    uint64_t n;
    uint32_t w;
    EBB_TRY(rows_common(c, f, rows, buf, &F, &Rw, &B, &n, &w));
    if (F->dtype != EBB_F32 && F->dtype != EBB_F64) return fail(c, EBB_E_TYPE, "scatter_add needs an F32/F64 field");
    if (F->layout == EBB_SOA && F->comps() > 1) return rows_soa(c, F, Rw, B, n, false, 1, (cudaStream_t)s);
    const uint32_t q = F->comps();   // AOS: component k of row r at f[r q + k]
    c->launches++;
    if (n) {
        const unsigned g = grid_for(n * q, 256);
        if (F->dtype == EBB_F64)
            k_rows_add_aos<double><<<g, 256, 0, (cudaStream_t)s>>>((double*)F->ptr, (const uint32_t*)Rw->ptr,
                                                                  (const double*)B->ptr, n, q);
        else
            k_rows_add_aos<float><<<g, 256, 0, (cudaStream_t)s>>>((float*)F->ptr, (const uint32_t*)Rw->ptr,
                                                                 (const float*)B->ptr, n, q);
    }
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status ebb_group_index(ebb_ctx ctx, ebb_rel rel, ebb_field* index_out) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    Relation* R = get_rel(c, rel);
    if (!R || !index_out) return fail(c, EBB_E_ARG, "bad argument");
    if (R->index == EBB_NONE) return fail(c, EBB_E_STATE, "relation '%s' has no group index", R->name.c_str());
    *index_out = R->index;
    return EBB_OK;
}

}  // extern "C"
