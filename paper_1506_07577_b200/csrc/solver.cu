// solver.cu -- edge-relation matvec, Jacobi-PCG, implicit assembly, integrator
// updates and global reductions.
//
// The matvec is the paper's query-loop `for e in v.edges do ... e.head ... end`
// over the edge relation grouped by tail (CSR) with the
// 3x3 stiffness stored per edge.  PCG follows Saad Alg. 9.1
// with the Jacobi preconditioner; alpha and beta stay on the device.
#include "ebb_internal.cuh"
#include "reduce.cuh"

using namespace ebb;

namespace {

enum { S_RHO = 0, S_ALPHA = 1, S_BETA = 2, S_PQ = 3, S_NSCAL = 8 };

// ---------------------------------------------------------------------------
// a10: q_v = sum_{e in row(v)} A_e p_head(e); LPV lanes cooperate on one vertex.
// MODE 0: plain; 1: q *= mask, fused p.q -> pq_out; 2: CG (mask, p.q, alpha).
template <typename R, int LPV, int MODE>
__global__ void __launch_bounds__(256) k_matvec(uint64_t nv, const uint32_t* __restrict__ index,
                                                const uint32_t* __restrict__ head, const R* __restrict__ A, uint64_t ne,
                                                const R* __restrict__ p, R* __restrict__ q,
                                                const uint8_t* __restrict__ mask, double* __restrict__ partials,
                                                unsigned int* __restrict__ counter, double* __restrict__ scal,
                                                double* __restrict__ pq_out, unsigned long long* __restrict__ err) {
    // warp-uniform trip count: the LPV-lane groups of one warp leave together
    const unsigned lane = threadIdx.x % LPV;
    const unsigned gpw = 32 / LPV;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    double pq = 0.0;
    for (uint64_t vb = warp * gpw; vb < nv; vb += nwarps * gpw) {
        const uint64_t v = vb + (threadIdx.x & 31) / LPV;
        const bool valid = v < nv;
        const uint32_t r0 = valid ? index[v] : 0u, r1 = valid ? index[v + 1] : 0u;
        R a0 = 0, a1 = 0, a2 = 0;
        for (uint32_t e = r0 + lane; e < r1; e += LPV) {
            const uint32_t h = head[e];
            const R px = p[3ull * h], py = p[3ull * h + 1], pz = p[3ull * h + 2];
            a0 += A[e] * px + A[ne + e] * py + A[2 * ne + e] * pz;
            a1 += A[3 * ne + e] * px + A[4 * ne + e] * py + A[5 * ne + e] * pz;
            a2 += A[6 * ne + e] * px + A[7 * ne + e] * py + A[8 * ne + e] * pz;
        }
#pragma unroll
        for (int o = LPV / 2; o > 0; o >>= 1) {
            a0 += __shfl_xor_sync(0xffffffffu, a0, o, LPV);
            a1 += __shfl_xor_sync(0xffffffffu, a1, o, LPV);
            a2 += __shfl_xor_sync(0xffffffffu, a2, o, LPV);
        }
        if (lane == 0 && valid) {
            if (MODE >= 1 && mask && !mask[v]) a0 = a1 = a2 = 0;
            q[3 * v] = a0;
            q[3 * v + 1] = a1;
            q[3 * v + 2] = a2;
            if (MODE >= 1) pq += (double)p[3 * v] * a0 + (double)p[3 * v + 1] * a1 + (double)p[3 * v + 2] * a2;
        }
    }
    if (MODE >= 1) {
        double tot;
        if (block_sum_last_done(pq, partials, counter, &tot)) {
            if (MODE == 1) {
                *pq_out = tot;
            } else {
                scal[S_PQ] = tot;
                if (tot < 0.0) atomicAdd(&err[ERR_NOT_SPD], 1ull);
                scal[S_ALPHA] = (tot != 0.0) ? scal[S_RHO] / tot : 0.0;
            }
        }
    }
}

// CG init: x = 0, r = b*m, z = r*dinv, p = z, rho = r.z
template <typename R>
__global__ void k_cg_init(uint64_t ndof, const R* __restrict__ b, const uint8_t* __restrict__ mask,
                          const R* __restrict__ dinv, R* __restrict__ x, R* __restrict__ r, R* __restrict__ z,
                          R* __restrict__ p, double* __restrict__ partials, unsigned int* __restrict__ counter,
                          double* __restrict__ scal, double* __restrict__ rho_user) {
    double acc = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ndof; i += (uint64_t)gridDim.x * blockDim.x) {
        R m = (mask && !mask[i / 3]) ? R(0) : R(1);
        R ri = b[i] * m;
        R zi = ri * dinv[i];
        x[i] = 0;
        r[i] = ri;
        z[i] = zi;
        p[i] = zi;
        acc += (double)ri * zi;
    }
    double tot;
    if (block_sum_last_done(acc, partials, counter, &tot)) {
        scal[S_RHO] = tot;
        scal[S_ALPHA] = 0.0;
        scal[S_BETA] = 0.0;
        if (rho_user) *rho_user = tot;
    }
}

// dinv = 1/diag(A) on free DOFs (Jacobi), 0 on fixed DOFs
template <typename R>
__global__ void k_dinv(uint64_t nv, const uint32_t* __restrict__ self, const R* __restrict__ A, uint64_t ne,
                       const uint8_t* __restrict__ mask, R* __restrict__ dinv) {
    uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (v >= nv) return;
    uint32_t e = self[v];
    bool fr = !mask || mask[v];
#pragma unroll
    for (int a = 0; a < 3; ++a) dinv[3 * v + a] = fr ? R(1) / A[(uint64_t)(4 * a) * ne + e] : R(0);
}

// x += alpha p; r -= alpha q; z = r*dinv; rho' = r.z -> beta = rho'/rho
template <typename R>
__global__ void k_cg_update(uint64_t ndof, const R* __restrict__ p, const R* __restrict__ q, const R* __restrict__ dinv,
                            R* __restrict__ x, R* __restrict__ r, R* __restrict__ z, double* __restrict__ partials,
                            unsigned int* __restrict__ counter, double* __restrict__ scal, double* __restrict__ rho_user) {
    const R alpha = (R)scal[S_ALPHA];
    double acc = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ndof; i += (uint64_t)gridDim.x * blockDim.x) {
        R pi = p[i];
        R ri = r[i] - alpha * q[i];
        R zi = ri * dinv[i];
        x[i] += alpha * pi;
        r[i] = ri;
        z[i] = zi;
        acc += (double)ri * zi;
    }
    double tot;
    if (block_sum_last_done(acc, partials, counter, &tot)) {
        double rho = scal[S_RHO];
        scal[S_BETA] = (rho != 0.0) ? tot / rho : 0.0;
        scal[S_RHO] = tot;
        if (rho_user) *rho_user = tot;
    }
}

// p = z + beta p
template <typename R>
__global__ void k_cg_dir(uint64_t ndof, const R* __restrict__ z, R* __restrict__ p, const double* __restrict__ scal) {
    const R beta = (R)scal[S_BETA];
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ndof; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = z[i] + beta * p[i];
}

// a9: A = M + h (alpha M + beta K) + h^2 K on every row of vertex v (in place ok)
template <typename R, int LPV>
__global__ void k_assemble_A(uint64_t nv, const uint32_t* __restrict__ index, const uint32_t* __restrict__ head,
                             const R* K, R* A, uint64_t ne, const R* __restrict__ mass, R h,
                             R alpha, R beta) {
    const unsigned lane = threadIdx.x % LPV;
    uint64_t v = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / LPV;
    if (v >= nv) return;
    const R m = mass[v];
    for (uint32_t e = index[v] + lane; e < index[v + 1]; e += LPV) {
        const bool diag = head[e] == v;
#pragma unroll
        for (int c = 0; c < 9; ++c) {
            R Me = (diag && (c == 0 || c == 4 || c == 8)) ? m : R(0);
            R Ke = K[(uint64_t)c * ne + e];
            R De = alpha * Me + beta * Ke;
            A[(uint64_t)c * ne + e] = Me + h * De + h * h * Ke;
        }
    }
}

// b = h (f + M g - D v - h K v), D v = alpha M v + beta K v
template <typename R>
__global__ void k_assemble_b(uint64_t nv, const R* __restrict__ f, const R* __restrict__ mass, const R* __restrict__ vel,
                             const R* __restrict__ Kv, R* __restrict__ b, R h, R alpha, R beta, R g0, R g1, R g2) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= 3 * nv) return;
    const R g = (i % 3 == 0) ? g0 : ((i % 3 == 1) ? g1 : g2);
    const R m = mass[i / 3];
    R Mv = m * vel[i];
    R Dv = alpha * Mv + beta * Kv[i];
    b[i] = h * (f[i] + m * g - Dv - h * Kv[i]);
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

template <typename R>
__global__ void k_implicit_update(uint64_t ndof, const R* __restrict__ dv, R h, R* __restrict__ u, R* __restrict__ vel) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= ndof) return;
    R v = vel[i] + dv[i];
    vel[i] = v;
    u[i] += h * v;
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

struct EdgeGraph {
    uint64_t nv = 0, ne = 0;
    const uint32_t* index = nullptr;
    const uint32_t* head = nullptr;
    uint32_t max_group = 0;
    ebb_rel verts = EBB_NONE;
};

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
    return EBB_OK;
}

unsigned vec_grid(Ctx* c, uint64_t n) {
    unsigned g = grid_for(n, 256);
    unsigned cap = (unsigned)c->num_sms * 8;
    return g < cap ? g : cap;
}

template <typename R, int MODE>
ebb_status launch_matvec(Ctx* c, const EdgeGraph& G, const R* A, const R* p, R* q, const uint8_t* mask, double* scal,
                         double* pq_out, unsigned int* counter, cudaStream_t s) {
    KernelTimer kt(c, EBB_K_EDGE_MATVEC, s);
    if (G.max_group <= 16) {
        unsigned grid = vec_grid(c, G.nv * 16);
        k_matvec<R, 16, MODE><<<grid, 256, 0, s>>>(G.nv, G.index, G.head, A, G.ne, p, q, mask, c->d_partials, counter,
                                                   scal, pq_out, c->d_err);
    } else {
        unsigned grid = vec_grid(c, G.nv * 32);
        k_matvec<R, 32, MODE><<<grid, 256, 0, s>>>(G.nv, G.index, G.head, A, G.ne, p, q, mask, c->d_partials, counter,
                                                   scal, pq_out, c->d_err);
    }
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

ebb_status check_mask(Ctx* c, ebb_field m, ebb_rel rel, const uint8_t** out) {
    *out = nullptr;
    if (m == EBB_NONE) return EBB_OK;
    Field* M = get_field(c, m);
    if (!M || M->dtype != EBB_U8 || M->comps() != 1 || M->rel != rel)
        return fail(c, EBB_E_TYPE, "mask must be a U8 scalar field on verts");
    *out = (const uint8_t*)M->ptr;
    return EBB_OK;
}

template <typename R>
ebb_status cg_iterate(Ctx* c, const ebb_cg* cg, const EdgeGraph& G, int iters, cudaStream_t s) {
    const R* A = (const R*)c->fields[cg->A].ptr;
    R* x = (R*)c->fields[cg->x].ptr;
    R* r = (R*)c->fields[cg->r].ptr;
    R* p = (R*)c->fields[cg->p].ptr;
    R* z = (R*)c->fields[cg->z].ptr;
    R* q = (R*)c->fields[cg->q].ptr;
    const R* dinv = (const R*)c->fields[cg->dinv].ptr;
    const uint8_t* mask;
    EBB_TRY(check_mask(c, cg->mask, G.verts, &mask));
    double* scal = (double*)c->fields[cg->scal].ptr;
    double* rho_user = (double*)c->fields[cg->rho].ptr;
    uint64_t ndof = 3 * G.nv;
    unsigned vg = vec_grid(c, ndof);
    for (int k = 0; k < iters; ++k) {
        EBB_TRY((launch_matvec<R, 2>(c, G, A, p, q, mask, scal, nullptr, c->d_counter + 1, s)));
        {
            KernelTimer kt(c, EBB_K_CG_UPDATE, s);
            k_cg_update<R><<<vg, 256, 0, s>>>(ndof, p, q, dinv, x, r, z, c->d_partials, c->d_counter + 2, scal, rho_user);
        }
        {
            KernelTimer kt(c, EBB_K_CG_DIR, s);
            k_cg_dir<R><<<vg, 256, 0, s>>>(ndof, z, p, scal);
        }
    }
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status cg_validate(Ctx* c, const ebb_cg* cg, EdgeGraph* G, ebb_dtype* dt) {
    EBB_TRY(edge_graph(c, cg->edges, G));
    Field* A = get_field(c, cg->A);
    if (!A) return fail(c, EBB_E_ARG, "cg: bad A");
    *dt = A->dtype;
    EBB_TRY(check_mat(c, A, cg->edges, *dt, "A"));
    EBB_TRY(check_vec(c, get_field(c, cg->b), G->verts, *dt, "b"));
    EBB_TRY(check_vec(c, get_field(c, cg->x), G->verts, *dt, "x"));
    return EBB_OK;
}

}  // namespace

extern "C" {

ebb_status ebb_map_edge_matvec(ebb_ctx ctx, ebb_rel edges, ebb_field A, ebb_field p, ebb_field q, ebb_field mask,
                               ebb_field pq_global, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
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
    bool fused = pq || m;
    if (dt == EBB_F64) {
        if (fused) return launch_matvec<double, 1>(c, G, (const double*)Af->ptr, (const double*)P->ptr, (double*)Q->ptr, m,
                                                   nullptr, pq ? pq : (double*)c->d_partials + 8191, c->d_counter + 3, s);
        return launch_matvec<double, 0>(c, G, (const double*)Af->ptr, (const double*)P->ptr, (double*)Q->ptr, nullptr,
                                        nullptr, nullptr, c->d_counter + 3, s);
    }
    if (dt == EBB_F32) {
        if (fused) return launch_matvec<float, 1>(c, G, (const float*)Af->ptr, (const float*)P->ptr, (float*)Q->ptr, m,
                                                  nullptr, pq ? pq : (double*)c->d_partials + 8191, c->d_counter + 3, s);
        return launch_matvec<float, 0>(c, G, (const float*)Af->ptr, (const float*)P->ptr, (float*)Q->ptr, nullptr,
                                       nullptr, nullptr, c->d_counter + 3, s);
    }
    return fail(c, EBB_E_TYPE, "matvec: dtype must be F32 or F64");
}

ebb_status ebb_global_reduce(ebb_ctx ctx, int32_t op, ebb_field a, ebb_field b, ebb_field mask, ebb_field out,
                             ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
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
    unsigned grid = vec_grid(c, n * Af->comps());
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
    if (!M || M->dtype != dt || M->comps() != 1 || M->rel != G.verts)
        return fail(c, EBB_E_TYPE, "assemble: mass must be a scalar field of the map dtype on verts");
    Field* F = get_field(c, d->f);
    Field* V = get_field(c, d->vel);
    Field* B = get_field(c, d->b);
    EBB_TRY(check_vec(c, F, G.verts, dt, "f"));
    EBB_TRY(check_vec(c, V, G.verts, dt, "vel"));
    EBB_TRY(check_vec(c, B, G.verts, dt, "b"));
    if (B->ptr == F->ptr || B->ptr == V->ptr) return fail(c, EBB_E_PHASE, "assemble: b aliases a read field");
    // K v scratch (allocated once per context, on the vertex relation)
    ebb_field kvf = EBB_NONE;
    for (ebb_field f : c->rels[G.verts].fields)
        if (c->fields[f].alive && c->fields[f].name == "__Kv" && c->fields[f].dtype == dt) kvf = f;
    if (kvf == EBB_NONE) EBB_TRY(new_internal_field(c, G.verts, "__Kv", dt, 3, 1, EBB_AOS, &kvf));
    // re-fetch (field table may have grown)
    K = get_field(c, d->K);
    A = get_field(c, d->A);
    M = get_field(c, d->mass);
    F = get_field(c, d->f);
    V = get_field(c, d->vel);
    B = get_field(c, d->b);
    void* kv = c->fields[kvf].ptr;
    cudaStream_t s = (cudaStream_t)stream;
    const int lpv = G.max_group <= 16 ? 16 : 32;
#define EBB_ASM(R)                                                                                                  \
    do {                                                                                                            \
        EBB_TRY((launch_matvec<R, 0>(c, G, (const R*)K->ptr, (const R*)V->ptr, (R*)kv, nullptr, nullptr, nullptr,     \
                                     c->d_counter + 5, s)));                                                        \
        KernelTimer kt(c, EBB_K_ASSEMBLE, s);                                                                       \
        c->launches++;                                                                                              \
        k_assemble_b<R><<<grid_for(3 * G.nv, 256), 256, 0, s>>>(G.nv, (const R*)F->ptr, (const R*)M->ptr,             \
                                                                (const R*)V->ptr, (const R*)kv, (R*)B->ptr, (R)d->h,  \
                                                                (R)d->alpha, (R)d->beta, (R)d->g[0], (R)d->g[1],      \
                                                                (R)d->g[2]);                                          \
        if (lpv == 16)                                                                                              \
            k_assemble_A<R, 16><<<grid_for(G.nv * 16, 256), 256, 0, s>>>(G.nv, G.index, G.head, (const R*)K->ptr,     \
                                                                         (R*)A->ptr, G.ne, (const R*)M->ptr, (R)d->h, \
                                                                         (R)d->alpha, (R)d->beta);                    \
        else                                                                                                        \
            k_assemble_A<R, 32><<<grid_for(G.nv * 32, 256), 256, 0, s>>>(G.nv, G.index, G.head, (const R*)K->ptr,     \
                                                                         (R*)A->ptr, G.ne, (const R*)M->ptr, (R)d->h, \
                                                                         (R)d->alpha, (R)d->beta);                    \
    } while (0)
    if (dt == EBB_F64) EBB_ASM(double);
    else EBB_ASM(float);
#undef EBB_ASM
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status ebb_cg_init(ebb_ctx ctx, ebb_cg* cg, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    if (!c || !cg) return fail(c, EBB_E_ARG, "null argument");
    EdgeGraph G;
    ebb_dtype dt;
    EBB_TRY(cg_validate(c, cg, &G, &dt));
    Field* S = get_field(c, cg->self);
    if (!S || S->dtype != EBB_KEY || S->rel != G.verts || S->key_target != cg->edges)
        return fail(c, EBB_E_TYPE, "cg: self must be the verts -> edges self-loop key");
    const uint8_t* mask;
    EBB_TRY(check_mask(c, cg->mask, G.verts, &mask));
    // allocate work fields that were not supplied
    static int serial = 0;
    int id = serial++;
    char nm[64];
    ebb_field* work[] = {&cg->r, &cg->p, &cg->z, &cg->q, &cg->dinv};
    const char* wn[] = {"r", "p", "z", "q", "dinv"};
    for (int i = 0; i < 5; ++i) {
        if (*work[i] == EBB_NONE) {
            snprintf(nm, sizeof(nm), "__cg%d_%s", id, wn[i]);
            EBB_TRY(new_internal_field(c, G.verts, nm, dt, 3, 1, EBB_AOS, work[i]));
        } else {
            EBB_TRY(check_vec(c, get_field(c, *work[i]), G.verts, dt, wn[i]));
        }
    }
    if (cg->rho == EBB_NONE) {
        snprintf(nm, sizeof(nm), "__cg%d_rho", id);
        EBB_TRY(ebb_global_new(ctx, nm, EBB_F64, 0.0, &cg->rho));
    }
    if (cg->scal == EBB_NONE) {
        snprintf(nm, sizeof(nm), "__cg%d_scal", id);
        ebb_rel sr;
        EBB_TRY(ebb_relation_new(ctx, (std::string(nm) + "_rel").c_str(), S_NSCAL, &sr));
        EBB_TRY(new_internal_field(c, sr, nm, EBB_F64, 1, 1, EBB_AOS, &cg->scal));
    }
    cudaStream_t s = (cudaStream_t)stream;
    uint64_t ndof = 3 * G.nv;
    unsigned vg = vec_grid(c, ndof);
    const uint32_t* self = (const uint32_t*)c->fields[cg->self].ptr;
    double* scal = (double*)c->fields[cg->scal].ptr;
    double* rho = (double*)c->fields[cg->rho].ptr;
#define EBB_INIT(R)                                                                                                 \
    do {                                                                                                            \
        c->launches += 2;                                                                                           \
        k_dinv<R><<<grid_for(G.nv, 256), 256, 0, s>>>(G.nv, self, (const R*)c->fields[cg->A].ptr, G.ne, mask,         \
                                                      (R*)c->fields[cg->dinv].ptr);                                  \
        k_cg_init<R><<<vg, 256, 0, s>>>(ndof, (const R*)c->fields[cg->b].ptr, mask, (const R*)c->fields[cg->dinv].ptr, \
                                        (R*)c->fields[cg->x].ptr, (R*)c->fields[cg->r].ptr, (R*)c->fields[cg->z].ptr,  \
                                        (R*)c->fields[cg->p].ptr, c->d_partials, c->d_counter + 6, scal, rho);         \
    } while (0)
    if (dt == EBB_F64) EBB_INIT(double);
    else EBB_INIT(float);
#undef EBB_INIT
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status ebb_cg_step(ebb_ctx ctx, const ebb_cg* cg, int32_t iters, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    if (!c || !cg) return fail(c, EBB_E_ARG, "null argument");
    if (iters < 0) return fail(c, EBB_E_ARG, "negative iteration count");
    EdgeGraph G;
    ebb_dtype dt;
    EBB_TRY(cg_validate(c, cg, &G, &dt));
    ebb_field w[] = {cg->r, cg->p, cg->z, cg->q, cg->dinv, cg->rho, cg->scal};
    for (ebb_field f : w)
        if (!get_field(c, f)) return fail(c, EBB_E_STATE, "cg: call ebb_cg_init first");
    cudaStream_t s = (cudaStream_t)stream;
    if (dt == EBB_F64) return cg_iterate<double>(c, cg, G, iters, s);
    return cg_iterate<float>(c, cg, G, iters, s);
}

ebb_status ebb_explicit_update(ebb_ctx ctx, const ebb_explicit_desc* d, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
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

ebb_status ebb_implicit_update(ebb_ctx ctx, ebb_field dv, double h, ebb_field u, ebb_field vel, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
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
    if (dt == EBB_F64)
        k_implicit_update<double><<<grid_for(ndof, 256), 256, 0, s>>>(ndof, (const double*)c->fields[dv].ptr, h,
                                                                      (double*)U->ptr, (double*)c->fields[vel].ptr);
    else
        k_implicit_update<float><<<grid_for(ndof, 256), 256, 0, s>>>(ndof, (const float*)c->fields[dv].ptr, (float)h,
                                                                     (float*)U->ptr, (float*)c->fields[vel].ptr);
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

}  // extern "C"
