// setup.cu -- one-time mesh setup on the device:
// orientation, Morton renumbering, tet sort, edge relation + GroupBy,
// tets.e[4][4], self-loop keys, rest data, partition owner maps.
// All integer results are bit-exact against the oracle (tests/test_gpu_setup.py).
#include <cub/cub.cuh>

#include <cstdio>

#include "ebb_internal.cuh"

using namespace ebb;

namespace {

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

__device__ __forceinline__ double det3(const double a[3][3]) {
    return a[0][0] * (a[1][1] * a[2][2] - a[1][2] * a[2][1]) - a[0][1] * (a[1][0] * a[2][2] - a[1][2] * a[2][0]) +
           a[0][2] * (a[1][0] * a[2][1] - a[1][1] * a[2][0]);
}

__device__ __forceinline__ void load_dm(const double* __restrict__ X, const uint32_t* v, double D[3][3]) {
    for (int k = 0; k < 3; ++k)
        for (int a = 0; a < 3; ++a) D[a][k] = X[3ull * v[k + 1] + a] - X[3ull * v[0] + a];
}

// O1: orientation fix (swap v2, v3 when det(Dm) < 0), degenerate detection
__global__ void k_orient(uint32_t* __restrict__ tv, const double* __restrict__ X, uint64_t nt,
                         unsigned long long* swaps, unsigned long long* degenerate) {
    uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    uint32_t v[4];
    for (int i = 0; i < 4; ++i) v[i] = tv[4 * t + i];
    double D[3][3];
    load_dm(X, v, D);
    double d = det3(D);
    double l = 0.0;
    for (int i = 0; i < 4; ++i)
        for (int j = i + 1; j < 4; ++j) {
            double s = 0.0;
            for (int a = 0; a < 3; ++a) {
                double q = X[3ull * v[j] + a] - X[3ull * v[i] + a];
                s += q * q;
            }
            l = fmax(l, sqrt(s));
        }
    if (fabs(d) <= 1e-12 * l * l * l) {
        atomicAdd(degenerate, 1ull);
        return;
    }
    if (d < 0.0) {
        tv[4 * t + 2] = v[3];
        tv[4 * t + 3] = v[2];
        atomicAdd(swaps, 1ull);
    }
}

// bounding box, pass 1 (per-block min/max per component) and pass 2
__global__ void k_bbox_partial(const double* __restrict__ X, uint64_t n, double* __restrict__ part) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        for (int d = 0; d < 3; ++d) {
            double x = X[3 * i + d];
            lo[d] = fmin(lo[d], x);
            hi[d] = fmax(hi[d], x);
        }
    __shared__ double s[6][256];
    for (int d = 0; d < 3; ++d) {
        s[d][threadIdx.x] = lo[d];
        s[3 + d][threadIdx.x] = hi[d];
    }
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int d = 0; d < 3; ++d) {
                s[d][threadIdx.x] = fmin(s[d][threadIdx.x], s[d][threadIdx.x + w]);
                s[3 + d][threadIdx.x] = fmax(s[3 + d][threadIdx.x], s[3 + d][threadIdx.x + w]);
            }
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int d = 0; d < 6; ++d) part[6 * blockIdx.x + d] = s[d][0];
}

__global__ void k_morton(const double* __restrict__ X, uint64_t n, const double* __restrict__ part, int nparts,
                         uint64_t* __restrict__ code) {
    __shared__ double lo[3], hi[3];
    if (threadIdx.x < 3) {
        double a = INFINITY, b = -INFINITY;
        for (int p = 0; p < nparts; ++p) {
            a = fmin(a, part[6 * p + threadIdx.x]);
            b = fmax(b, part[6 * p + 3 + threadIdx.x]);
        }
        lo[threadIdx.x] = a;
        hi[threadIdx.x] = b;
    }
    __syncthreads();
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t c = 0;
    for (int d = 0; d < 3; ++d) {
        uint64_t q = 0;
        if (hi[d] != lo[d]) {
            // exactly O3's order: subtract, divide, multiply, floor -- no FMA
            double s = __dsub_rn(X[3 * i + d], lo[d]);
            s = __ddiv_rn(s, __dsub_rn(hi[d], lo[d]));
            s = __dmul_rn(s, 2097152.0);
            q = (uint64_t)floor(s);
            if (q > 2097151ull) q = 2097151ull;
        }
        for (int b = 0; b < 21; ++b) c |= ((q >> b) & 1ull) << (3 * b + d);
    }
    code[i] = c;
}

__global__ void k_iota(uint32_t* p, uint64_t n) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = (uint32_t)i;
}

__global__ void k_invert(const uint32_t* __restrict__ n2o, uint32_t* __restrict__ o2n, uint64_t n) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) o2n[n2o[i]] = (uint32_t)i;
}

// sorted 4-tuple component k of tet t (ascending vertex ids), gathered by perm
__global__ void k_tuple_key(const uint32_t* __restrict__ tv, const uint32_t* __restrict__ perm, uint64_t nt, int k,
                            uint32_t* __restrict__ key, int nc) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= nt) return;
    uint64_t t = perm[i];
    uint32_t s[4];
    for (int j = 0; j < nc; ++j) s[j] = tv[(uint64_t)nc * t + j];
    for (int a = 1; a < nc; ++a)
        for (int b = a; b > 0 && s[b - 1] > s[b]; --b) {
            uint32_t q = s[b];
            s[b] = s[b - 1];
            s[b - 1] = q;
        }
    key[i] = s[k];
}

// a1: 16 ordered pairs per tet (incl. i == j) plus a self-loop per vertex
__global__ void k_edge_pairs(const uint32_t* __restrict__ tv, uint64_t nt, uint64_t nv, uint64_t* __restrict__ out) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < nt * 16) {
        uint64_t t = i >> 4;
        int a = (int)((i >> 2) & 3), b = (int)(i & 3);
        out[i] = ((uint64_t)tv[4 * t + a] << 32) | tv[4 * t + b];
    } else if (i < nt * 16 + nv) {
        uint64_t v = i - nt * 16;
        out[i] = (v << 32) | v;
    }
}

__global__ void k_split_pairs(const uint64_t* __restrict__ pairs, uint64_t ne, uint32_t* __restrict__ tail,
                              uint32_t* __restrict__ head) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= ne) return;
    uint64_t p = pairs[i];
    tail[i] = (uint32_t)(p >> 32);
    head[i] = (uint32_t)(p & 0xFFFFFFFFull);
}

__global__ void k_lower_bound(const uint32_t* __restrict__ sorted, uint64_t n, uint32_t* __restrict__ index,
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

__device__ __forceinline__ uint32_t find_row(const uint32_t* __restrict__ index, const uint32_t* __restrict__ head,
                                             uint32_t a, uint32_t b) {
    uint32_t lo = index[a], hi = index[a + 1];
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (head[mid] < b) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// tets.e[t][i][j] = row of (v[i], v[j]) in the grouped edge relation
__global__ void k_tet_edges(const uint32_t* __restrict__ tv, uint64_t nt, const uint32_t* __restrict__ index,
                            const uint32_t* __restrict__ head, uint32_t* __restrict__ e) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= nt * 16) return;
    uint64_t t = i >> 4;
    int a = (int)((i >> 2) & 3), b = (int)(i & 3);
    e[i] = find_row(index, head, tv[4 * t + a], tv[4 * t + b]);
}

__global__ void k_self_edges(uint64_t nv, const uint32_t* __restrict__ index, const uint32_t* __restrict__ head,
                             uint32_t* __restrict__ self) {
    uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (v < nv) self[v] = find_row(index, head, (uint32_t)v, (uint32_t)v);
}


// a3: rest data.  Dminv stored component-planar: plane (3r + c) holds row r col c.
__global__ void k_rest(const uint32_t* __restrict__ tv, const double* __restrict__ X, uint64_t nt, double rho,
                       double* __restrict__ Dminv, double* __restrict__ W, double* __restrict__ mass,
                       unsigned long long* bad) {
    uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    uint32_t v[4];
    for (int i = 0; i < 4; ++i) v[i] = tv[4 * t + i];
    double A[3][3];
    load_dm(X, v, A);
    double d = det3(A);
    double w = d / 6.0;
    if (!(w > 0.0)) atomicAdd(bad, 1ull);
    double C[3][3];
    C[0][0] = A[1][1] * A[2][2] - A[1][2] * A[2][1];
    C[0][1] = -(A[1][0] * A[2][2] - A[1][2] * A[2][0]);
    C[0][2] = A[1][0] * A[2][1] - A[1][1] * A[2][0];
    C[1][0] = -(A[0][1] * A[2][2] - A[0][2] * A[2][1]);
    C[1][1] = A[0][0] * A[2][2] - A[0][2] * A[2][0];
    C[1][2] = -(A[0][0] * A[2][1] - A[0][1] * A[2][0]);
    C[2][0] = A[0][1] * A[1][2] - A[0][2] * A[1][1];
    C[2][1] = -(A[0][0] * A[1][2] - A[0][2] * A[1][0]);
    C[2][2] = A[0][0] * A[1][1] - A[0][1] * A[1][0];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) Dminv[(uint64_t)(3 * r + c) * nt + t] = C[c][r] / d;
    W[t] = w;
    double mv = rho * w / 4.0;
    for (int i = 0; i < 4; ++i) atomicAdd(&mass[v[i]], mv);
}

// consistent (Galerkin) mass of linear tets on the edge relation:
// mass_e[e[i][j]] += rho W (1 + d_ij) / 20 (one fp64 red per (tet, i, j))
__global__ void k_consistent_mass(const uint32_t* __restrict__ te, const double* __restrict__ W, uint64_t nt,
                                  double rho, double* __restrict__ mass_e) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= nt * 16) return;
    const uint64_t t = k >> 4;
    const int i = (int)(k >> 2) & 3, j = (int)k & 3;
    atomicAdd(&mass_e[te[k]], rho * W[t] * (i == j ? 2.0 : 1.0) / 20.0);
}

__global__ void k_first_tet(const uint32_t* __restrict__ tv, uint64_t nt, unsigned int* __restrict__ first) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < nt * 4) atomicMin(&first[tv[i]], (unsigned int)(i >> 2));
}

__global__ void k_owners(const unsigned int* __restrict__ first, uint64_t nv, uint64_t nt, int P,
                         int32_t* __restrict__ owner_v, int32_t* __restrict__ owner_t) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < nt) owner_t[i] = (int32_t)((i * (uint64_t)P) / nt);
    if (i < nv) {
        unsigned int f = first[i];
        owner_v[i] = (f == 0xFFFFFFFFu) ? (int32_t)((i * (uint64_t)P) / nv) : (int32_t)(((uint64_t)f * P) / nt);
    }
}

ebb_status check_tets_v(Ctx* c, ebb_field tets_v, Field** out) {
    Field* F = get_field(c, tets_v);
    if (!F) return fail(c, EBB_E_ARG, "bad tets.v handle");
    if (F->dtype != EBB_KEY || F->comps() != 4 || F->layout != EBB_AOS)
        return fail(c, EBB_E_TYPE, "'%s' must be a 4x1 key-field (tets.v)", F->name.c_str());
    *out = F;
    return EBB_OK;
}

ebb_status check_pos(Ctx* c, ebb_field pos, ebb_rel verts, Field** out) {
    Field* F = get_field(c, pos);
    if (!F) return fail(c, EBB_E_ARG, "bad position field handle");
    if (F->dtype != EBB_F64 || F->comps() != 3 || F->layout != EBB_AOS || F->rel != verts)
        return fail(c, EBB_E_TYPE, "'%s' must be an AOS vec3 F64 field on the vertex relation", F->name.c_str());
    *out = F;
    return EBB_OK;
}

}  // namespace

extern "C" {

ebb_status ebb_tetmesh_orient(ebb_ctx ctx, ebb_field tets_v, ebb_field pos, uint64_t* n_swapped) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c) return EBB_E_ARG;
    Field *V, *X;
    EBB_TRY(check_tets_v(c, tets_v, &V));
    EBB_TRY(check_pos(c, pos, V->key_target, &X));
    uint64_t nt = c->rels[V->rel].size;
    DevBuf cnt;
    EBB_CUDA(c, cudaMalloc(&cnt.p, 16));
    EBB_CUDA(c, cudaMemset(cnt.p, 0, 16));
    unsigned long long* h = (unsigned long long*)cnt.p;
    k_orient<<<grid_for(nt, 256), 256>>>((uint32_t*)V->ptr, (const double*)X->ptr, nt, h, h + 1);
    EBB_CUDA(c, cudaGetLastError());
    unsigned long long r[2];
    EBB_CUDA(c, cudaMemcpy(r, cnt.p, 16, cudaMemcpyDeviceToHost));
    if (n_swapped) *n_swapped = r[0];
    if (r[1]) return fail(c, EBB_E_DEGENERATE, "%llu degenerate tets (|det Dm| <= 1e-12 l^3)", r[1]);
    return EBB_OK;
}

ebb_status ebb_renumber_morton(ebb_ctx ctx, ebb_rel rel, ebb_field pos) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c) return EBB_E_ARG;
    Field* X;
    EBB_TRY(check_pos(c, pos, rel, &X));
    Relation* R = get_rel(c, rel);
    if (R->grouped_by != EBB_NONE) return fail(c, EBB_E_STATE, "renumber a relation before grouping it");
    uint64_t n = R->size;
    const int nb = 256;
    DevBuf part, code, code2, vin, vout, inv, tmp;
    EBB_CUDA(c, cudaMalloc(&part.p, nb * 6 * sizeof(double)));
    k_bbox_partial<<<nb, 256>>>((const double*)X->ptr, n, (double*)part.p);
    EBB_CUDA(c, cudaMalloc(&code.p, n * 8));
    EBB_CUDA(c, cudaMalloc(&code2.p, n * 8));
    k_morton<<<grid_for(n, 256), 256>>>((const double*)X->ptr, n, (const double*)part.p, nb, (uint64_t*)code.p);
    EBB_CUDA(c, cudaMalloc(&vin.p, n * 4));
    EBB_CUDA(c, cudaMalloc(&vout.p, n * 4));
    EBB_CUDA(c, cudaMalloc(&inv.p, n * 4));
    k_iota<<<grid_for(n, 256), 256>>>((uint32_t*)vin.p, n);
    EBB_CUDA(c, cudaGetLastError());
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (const uint64_t*)code.p, (uint64_t*)code2.p, (const uint32_t*)vin.p,
                                    (uint32_t*)vout.p, (int)n, 0, 63);
    EBB_CUDA(c, cudaMalloc(&tmp.p, tb));
    // LSD radix sort is stable: ties keep ascending old id (O3 "(code, old id)")
    EBB_CUDA(c, cub::DeviceRadixSort::SortPairs(tmp.p, tb, (const uint64_t*)code.p, (uint64_t*)code2.p,
                                                (const uint32_t*)vin.p, (uint32_t*)vout.p, (int)n, 0, 63));
    k_invert<<<grid_for(n, 256), 256>>>((const uint32_t*)vout.p, (uint32_t*)inv.p, n);
    EBB_CUDA(c, cudaGetLastError());
    return permute_relation(c, rel, (const uint32_t*)vout.p, (const uint32_t*)inv.p, nullptr);
}

ebb_status ebb_sort_by_key_tuple(ebb_ctx ctx, ebb_rel rel, ebb_field keys) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c) return EBB_E_ARG;
    Field* V = get_field(c, keys);
    if (!V) return fail(c, EBB_E_ARG, "bad key-field handle");
    if (V->dtype != EBB_KEY || V->comps() < 1 || V->comps() > 4 || V->layout != EBB_AOS)
        return fail(c, EBB_E_TYPE, "'%s' must be a key-field of 1..4 keys per row", V->name.c_str());
    const int nc = (int)V->comps();
    if (V->rel != rel) return fail(c, EBB_E_TYPE, "key-field is not on the relation being sorted");
    uint64_t nt = c->rels[rel].size;
    uint64_t ntarget = c->rels[V->key_target].size;
    int end_bit = 1;
    while (end_bit < 32 && (1ull << end_bit) < ntarget) ++end_bit;
    DevBuf perm, perm2, key, key2, inv, tmp;
    EBB_CUDA(c, cudaMalloc(&perm.p, nt * 4));
    EBB_CUDA(c, cudaMalloc(&perm2.p, nt * 4));
    EBB_CUDA(c, cudaMalloc(&key.p, nt * 4));
    EBB_CUDA(c, cudaMalloc(&key2.p, nt * 4));
    EBB_CUDA(c, cudaMalloc(&inv.p, nt * 4));
    k_iota<<<grid_for(nt, 256), 256>>>((uint32_t*)perm.p, nt);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (const uint32_t*)key.p, (uint32_t*)key2.p, (const uint32_t*)perm.p,
                                    (uint32_t*)perm2.p, (int)nt, 0, end_bit);
    EBB_CUDA(c, cudaMalloc(&tmp.p, tb));
    // LSD over the sorted tuple: least significant component first, stable
    for (int k = nc - 1; k >= 0; --k) {
        k_tuple_key<<<grid_for(nt, 256), 256>>>((const uint32_t*)V->ptr, (const uint32_t*)perm.p, nt, k,
                                                (uint32_t*)key.p, nc);
        EBB_CUDA(c, cub::DeviceRadixSort::SortPairs(tmp.p, tb, (const uint32_t*)key.p, (uint32_t*)key2.p,
                                                    (const uint32_t*)perm.p, (uint32_t*)perm2.p, (int)nt, 0, end_bit));
        std::swap(perm.p, perm2.p);
    }
    k_invert<<<grid_for(nt, 256), 256>>>((const uint32_t*)perm.p, (uint32_t*)inv.p, nt);
    EBB_CUDA(c, cudaGetLastError());
    return permute_relation(c, rel, (const uint32_t*)perm.p, (const uint32_t*)inv.p, nullptr);
}

ebb_status ebb_tetmesh_build(ebb_ctx ctx, ebb_field tets_v, const char* edges_name, ebb_tetmesh* out) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !out || !edges_name) return fail(c, EBB_E_ARG, "null argument");
    Field* V;
    EBB_TRY(check_tets_v(c, tets_v, &V));
    ebb_rel tets = V->rel, verts = V->key_target;
    uint64_t nt = c->rels[tets].size, nv = c->rels[verts].size;
    uint64_t np = nt * 16 + nv;
    if (np > 0x7FFFFFFFull) return fail(c, EBB_E_RANGE, "too many edge candidates for one sort (%llu)", np);
    int vbits = 1;
    while (vbits < 32 && (1ull << vbits) < nv) ++vbits;
    DevBuf pairs, pairs2, uniq, nsel, tmp;
    EBB_CUDA(c, cudaMalloc(&pairs.p, np * 8));
    EBB_CUDA(c, cudaMalloc(&pairs2.p, np * 8));
    EBB_CUDA(c, cudaMalloc(&uniq.p, np * 8));
    EBB_CUDA(c, cudaMalloc(&nsel.p, 8));
    k_edge_pairs<<<grid_for(np, 256), 256>>>((const uint32_t*)V->ptr, nt, nv, (uint64_t*)pairs.p);
    EBB_CUDA(c, cudaGetLastError());
    size_t tb1 = 0, tb2 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb1, (const uint64_t*)pairs.p, (uint64_t*)pairs2.p, (int)np, 0, 32 + vbits);
    cub::DeviceSelect::Unique(nullptr, tb2, (const uint64_t*)pairs2.p, (uint64_t*)uniq.p, (int*)nsel.p, (int)np);
    EBB_CUDA(c, cudaMalloc(&tmp.p, tb1 > tb2 ? tb1 : tb2));
    EBB_CUDA(c, cub::DeviceRadixSort::SortKeys(tmp.p, tb1, (const uint64_t*)pairs.p, (uint64_t*)pairs2.p, (int)np, 0,
                                               32 + vbits));
    EBB_CUDA(c, cub::DeviceSelect::Unique(tmp.p, tb2, (const uint64_t*)pairs2.p, (uint64_t*)uniq.p, (int*)nsel.p,
                                          (int)np));
    int ne = 0;
    EBB_CUDA(c, cudaMemcpy(&ne, nsel.p, 4, cudaMemcpyDeviceToHost));
    ebb_rel edges;
    EBB_TRY(ebb_relation_new(ctx, edges_name, (uint64_t)ne, &edges));
    ebb_field tail, head, e, self, idx;
    EBB_TRY(new_internal_field(c, edges, "tail", EBB_KEY, 1, 1, EBB_AOS, &tail));
    EBB_TRY(new_internal_field(c, edges, "head", EBB_KEY, 1, 1, EBB_AOS, &head));
    c->fields[tail].key_target = verts;
    c->fields[head].key_target = verts;
    k_split_pairs<<<grid_for(ne, 256), 256>>>((const uint64_t*)uniq.p, ne, (uint32_t*)c->fields[tail].ptr,
                                              (uint32_t*)c->fields[head].ptr);
    EBB_CUDA(c, cudaGetLastError());
    // GroupBy(tail): rows are already in (tail, head) order -> identity permutation;
    // build the hidden [begin, end) index on verts
    ebb_rel irel;
    EBB_TRY(ebb_relation_new(ctx, (std::string("__index_rel_") + edges_name).c_str(), nv + 1, &irel));
    EBB_TRY(new_internal_field(c, irel, std::string("__index_") + edges_name, EBB_U32, 1, 1, EBB_AOS, &idx));
    k_lower_bound<<<grid_for(nv + 1, 256), 256>>>((const uint32_t*)c->fields[tail].ptr, ne,
                                                  (uint32_t*)c->fields[idx].ptr, nv);
    uint32_t st[3];
    EBB_TRY(index_stats(c, (const uint32_t*)c->fields[idx].ptr, nv, st));
    c->rels[edges].grouped_by = tail;
    c->rels[edges].index = idx;
    c->rels[edges].max_group = st[0];
    c->rels[edges].max_chunk16 = st[1];
    c->rels[edges].max_chunk64 = st[2];
    c->rels[verts].index = idx;
    c->rels[verts].max_group = st[0];
    // tets.e[4][4] and verts.self
    char ename[64];
    snprintf(ename, sizeof(ename), "e_%s", edges_name);
    EBB_TRY(new_internal_field(c, tets, ename, EBB_KEY, 4, 4, EBB_AOS, &e));
    c->fields[e].key_target = edges;
    snprintf(ename, sizeof(ename), "self_%s", edges_name);
    EBB_TRY(new_internal_field(c, verts, ename, EBB_KEY, 1, 1, EBB_AOS, &self));
    c->fields[self].key_target = edges;
    V = get_field(c, tets_v);
    k_tet_edges<<<grid_for(nt * 16, 256), 256>>>((const uint32_t*)V->ptr, nt, (const uint32_t*)c->fields[idx].ptr,
                                                 (const uint32_t*)c->fields[head].ptr, (uint32_t*)c->fields[e].ptr);
    k_self_edges<<<grid_for(nv, 256), 256>>>(nv, (const uint32_t*)c->fields[idx].ptr,
                                             (const uint32_t*)c->fields[head].ptr, (uint32_t*)c->fields[self].ptr);
    EBB_CUDA(c, cudaGetLastError());
    EBB_CUDA(c, cudaDeviceSynchronize());
    out->edges = edges;
    out->tail = tail;
    out->head = head;
    out->e = e;
    out->self = self;
    out->index = idx;
    return EBB_OK;
}

ebb_status ebb_tetmesh_rest(ebb_ctx ctx, ebb_field tets_v, ebb_field pos, double rho, ebb_field Dminv, ebb_field W,
                            ebb_field mass, ebb_stream s) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c) return EBB_E_ARG;
    Field *V, *X;
    EBB_TRY(check_tets_v(c, tets_v, &V));
    EBB_TRY(check_pos(c, pos, V->key_target, &X));
    Field* D = get_field(c, Dminv);
    Field* Wf = get_field(c, W);
    Field* M = get_field(c, mass);
    if (!D || !Wf || !M) return fail(c, EBB_E_ARG, "bad output field handle");
    if (D->dtype != EBB_F64 || D->comps() != 9 || D->layout != EBB_SOA || D->rel != V->rel)
        return fail(c, EBB_E_TYPE, "Dminv must be a SOA 3x3 F64 field on tets");
    if (Wf->dtype != EBB_F64 || Wf->comps() != 1 || Wf->rel != V->rel)
        return fail(c, EBB_E_TYPE, "W must be a scalar F64 field on tets");
    if (M->dtype != EBB_F64 || M->comps() != 1 || M->rel != V->key_target)
        return fail(c, EBB_E_TYPE, "mass must be a scalar F64 field on verts");
    uint64_t nt = c->rels[V->rel].size, nv = c->rels[V->key_target].size;
    cudaStream_t st = (cudaStream_t)s;
    DevBuf bad;
    EBB_CUDA(c, cudaMalloc(&bad.p, 8));
    EBB_CUDA(c, cudaMemsetAsync(bad.p, 0, 8, st));
    EBB_CUDA(c, cudaMemsetAsync(M->ptr, 0, nv * 8, st));
    k_rest<<<grid_for(nt, 256), 256, 0, st>>>((const uint32_t*)V->ptr, (const double*)X->ptr, nt, rho,
                                              (double*)D->ptr, (double*)Wf->ptr, (double*)M->ptr,
                                              (unsigned long long*)bad.p);
    EBB_CUDA(c, cudaGetLastError());
    unsigned long long hb = 0;
    EBB_CUDA(c, cudaMemcpyAsync(&hb, bad.p, 8, cudaMemcpyDeviceToHost, st));
    EBB_CUDA(c, cudaStreamSynchronize(st));
    if (hb) return fail(c, EBB_E_INVERTED, "%llu tets with W <= 0 (orient the mesh first)", hb);
    return EBB_OK;
}

ebb_status ebb_tetmesh_consistent_mass(ebb_ctx ctx, ebb_field tets_e, ebb_field W, double rho, ebb_field mass_e,
                                       ebb_stream s) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c) return EBB_E_ARG;
    Field* E = get_field(c, tets_e);
    Field* Wf = get_field(c, W);
    Field* M = get_field(c, mass_e);
    if (!E || !Wf || !M) return fail(c, EBB_E_ARG, "bad field handle");
    if (E->dtype != EBB_KEY || E->comps() != 16 || E->layout != EBB_AOS)
        return fail(c, EBB_E_TYPE, "'%s' must be the 4x4 key-field tets.e", E->name.c_str());
    if (Wf->dtype != EBB_F64 || Wf->comps() != 1 || Wf->rel != E->rel)
        return fail(c, EBB_E_TYPE, "W must be a scalar F64 field on tets");
    if (M->dtype != EBB_F64 || M->comps() != 1 || M->rel != E->key_target)
        return fail(c, EBB_E_TYPE, "mass_e must be a scalar F64 field on the edge relation tets.e points to");
    if (M->ptr == Wf->ptr) return fail(c, EBB_E_PHASE, "mass_e aliases W");
    const uint64_t nt = c->rels[E->rel].size, ne = c->rels[M->rel].size;
    cudaStream_t st = (cudaStream_t)s;
    EBB_CUDA(c, cudaMemsetAsync(M->ptr, 0, ne * 8, st));
    if (nt) {
        k_consistent_mass<<<grid_for(nt * 16, 256), 256, 0, st>>>((const uint32_t*)E->ptr, (const double*)Wf->ptr,
                                                                  nt, rho, (double*)M->ptr);
        c->launches++;
    }
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status ebb_partition(ebb_ctx ctx, ebb_field tets_v, int32_t nparts, ebb_field owner_t, ebb_field owner_v) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c) return EBB_E_ARG;
    Field* V;
    EBB_TRY(check_tets_v(c, tets_v, &V));
    Field* OT = get_field(c, owner_t);
    Field* OV = get_field(c, owner_v);
    if (!OT || !OV || nparts < 1) return fail(c, EBB_E_ARG, "bad partition arguments");
    if (OT->dtype != EBB_I32 || OT->rel != V->rel || OV->dtype != EBB_I32 || OV->rel != V->key_target)
        return fail(c, EBB_E_TYPE, "owner fields must be I32 on tets / verts");
    uint64_t nt = c->rels[V->rel].size, nv = c->rels[V->key_target].size;
    DevBuf first;
    EBB_CUDA(c, cudaMalloc(&first.p, nv * 4));
    EBB_CUDA(c, cudaMemset(first.p, 0xFF, nv * 4));
    k_first_tet<<<grid_for(nt * 4, 256), 256>>>((const uint32_t*)V->ptr, nt, (unsigned int*)first.p);
    uint64_t n = nt > nv ? nt : nv;
    k_owners<<<grid_for(n, 256), 256>>>((const unsigned int*)first.p, nv, nt, nparts, (int32_t*)OV->ptr,
                                        (int32_t*)OT->ptr);
    EBB_CUDA(c, cudaGetLastError());
    EBB_CUDA(c, cudaDeviceSynchronize());
    return EBB_OK;
}

}  // extern "C"
