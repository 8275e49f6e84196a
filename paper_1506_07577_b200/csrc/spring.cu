// spring.cu -- the Fig. 2 spring-mass program:
// a second workload on the same relations, all of it edge query-loops over
// v.edges (the grouped edge relation):
//
//   initLen(e)               rest_len = |head.pos - tail.pos|
//   computeInternalForces(v) for e in v.edges: dq = e.head.q - v.q,
//                            v.force += K (e.rest_len normalize(dq) - dq)
//   applyForces(v)           qdd = force/mass, q += qd dt + qdd dt^2/2,
//                            qd += qdd dt, force = 0
//   measureTotalEnergy(v)    E += mass qd.qd / 2
//
// The force sign is the one printed (DESIGN.md §3 reading 21); normalize(0)
// = 0, so self-loop rows add nothing.  Query-loop layout as the CG matvec:
// LPV lanes per vertex walk its rows (head key + rest length streamed, q
// gathered through head: L2-resident), a shuffle tree sums the lanes.
// ebb_spring_step fuses one whole Fig. 2 iteration (forces in registers,
// then the update) into ONE kernel; q is double-buffered (read q_in,
// write q_out) because neighbours read q while owners would write it -- the
// phase rule of P:443-450 that makes the paper split the two kernels.
#include <algorithm>

#include "ebb_internal.cuh"
#include "reduce.cuh"

namespace ebb {
namespace {

template <typename R>
__global__ void k_spring_init_len(uint64_t ne, const uint32_t* __restrict__ tail, const uint32_t* __restrict__ head,
                                  const R* __restrict__ pos, R* __restrict__ rest) {
    const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (e >= ne) return;
    const uint64_t a = tail[e], b = head[e];
    const R d0 = pos[3 * b] - pos[3 * a], d1 = pos[3 * b + 1] - pos[3 * a + 1], d2 = pos[3 * b + 2] - pos[3 * a + 2];
    rest[e] = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
}

// sum over v's rows of K (rest dir - dq), for the LPV lanes of vertex v
template <typename R, int LPV>
__device__ __forceinline__ void spring_row_sum(uint64_t v, bool live, const uint32_t* __restrict__ index,
                                               const uint32_t* __restrict__ head, const R* __restrict__ q,
                                               const R* __restrict__ rest, R K, R& s0, R& s1, R& s2) {
    const unsigned lane = threadIdx.x % LPV;
    s0 = s1 = s2 = R(0);
    if (live) {
        const R q0 = q[3 * v], q1 = q[3 * v + 1], q2 = q[3 * v + 2];
        for (uint32_t e = index[v] + lane; e < index[v + 1]; e += LPV) {
            const uint64_t h = head[e];
            const R L = rest[e];
            const R d0 = q[3 * h] - q0, d1 = q[3 * h + 1] - q1, d2 = q[3 * h + 2] - q2;
            const R len = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
            const R c = len > R(0) ? L / len : R(0);   // rest * normalize(dq) = (rest/len) dq
            s0 += K * (c * d0 - d0);
            s1 += K * (c * d1 - d1);
            s2 += K * (c * d2 - d2);
        }
    }
#pragma unroll
    for (int o = LPV / 2; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o, LPV);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o, LPV);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o, LPV);
    }
}

template <typename R, int LPV>
__global__ void __launch_bounds__(256) k_spring_forces(uint64_t nv, const uint32_t* __restrict__ index,
                                                       const uint32_t* __restrict__ head, const R* __restrict__ q,
                                                       const R* __restrict__ rest, R K, R* __restrict__ force,
                                                       int accumulate) {
    const uint64_t v = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / LPV;
    const bool live = v < nv;
    R s0, s1, s2;
    spring_row_sum<R, LPV>(v, live, index, head, q, rest, K, s0, s1, s2);
    if (live && threadIdx.x % LPV == 0) {
        if (accumulate) {
            s0 += force[3 * v];
            s1 += force[3 * v + 1];
            s2 += force[3 * v + 2];
        }
        force[3 * v] = s0;
        force[3 * v + 1] = s1;
        force[3 * v + 2] = s2;
    }
}

template <typename R>
__device__ __forceinline__ void spring_update(R f, R m, R dt, R q, R& qd, R& qn) {
    const R qdd = f / m;
    qn = q + (qd * dt + R(0.5) * qdd * dt * dt);
    qd = qd + qdd * dt;
}

template <typename R>
__global__ void k_spring_apply(uint64_t nv, const R* __restrict__ mass, R dt, R* __restrict__ q, R* __restrict__ qd,
                               R* __restrict__ force) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= 3 * nv) return;
    R v = qd[i], qn;
    spring_update(force[i], mass[i / 3], dt, q[i], v, qn);
    q[i] = qn;
    qd[i] = v;
    force[i] = R(0);
}

// one Fig. 2 iteration: forces from q_in (registers), then applyForces into
// q_out / qd; `force` (nullable) receives the forces for inspection
template <typename R, int LPV>
__global__ void __launch_bounds__(256) k_spring_step(uint64_t nv, const uint32_t* __restrict__ index,
                                                     const uint32_t* __restrict__ head, const R* __restrict__ q,
                                                     const R* __restrict__ rest, const R* __restrict__ mass, R K,
                                                     R dt, R* __restrict__ qout, R* __restrict__ qd,
                                                     R* __restrict__ force) {
    const uint64_t v = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / LPV;
    const bool live = v < nv;
    R s[3];
    spring_row_sum<R, LPV>(v, live, index, head, q, rest, K, s[0], s[1], s[2]);
    const unsigned lane = threadIdx.x % LPV;
    if (live && lane < 3) {   // one component per lane
        const R f = lane == 0 ? s[0] : lane == 1 ? s[1] : s[2];
        const uint64_t i = 3 * v + lane;
        R w = qd[i], qn;
        spring_update(f, mass[v], dt, q[i], w, qn);
        qout[i] = qn;
        qd[i] = w;
        if (force) force[i] = f;
    }
}

template <typename R>
__global__ void __launch_bounds__(256) k_kinetic_energy(uint64_t nv, const R* __restrict__ mass,
                                                        const R* __restrict__ qd, double* __restrict__ partials,
                                                        unsigned int* __restrict__ counter, double* __restrict__ out) {
    double acc = 0.0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x) {
        const double a = qd[3 * v], b = qd[3 * v + 1], c = qd[3 * v + 2];
        acc += 0.5 * (double)mass[v] * (a * a + b * b + c * c);
    }
    double tot;
    if (block_sum_last_done(acc, partials, counter, &tot)) *out = tot;
}

ebb_status check_vert_vec(Ctx* c, ebb_field f, ebb_rel verts, ebb_dtype dt, const char* what, Field** out) {
    Field* F = get_field(c, f);
    if (!F) return fail(c, EBB_E_ARG, "spring: bad %s", what);
    if (F->rel != verts || F->comps() != 3 || F->layout != EBB_AOS || F->dtype != dt)
        return fail(c, EBB_E_TYPE, "spring: %s must be an AOS vec3 field of the %s dtype on the vertices", what,
                    dt == EBB_F64 ? "F64" : "F32");
    *out = F;
    return EBB_OK;
}

ebb_status check_scalar(Ctx* c, ebb_field f, ebb_rel rel, ebb_dtype dt, const char* what, Field** out) {
    Field* F = get_field(c, f);
    if (!F) return fail(c, EBB_E_ARG, "spring: bad %s", what);
    if (F->rel != rel || F->comps() != 1 || F->dtype != dt)
        return fail(c, EBB_E_TYPE, "spring: %s must be a scalar field of the position dtype", what);
    *out = F;
    return EBB_OK;
}

ebb_status float_dtype(Ctx* c, Field* F, ebb_dtype* dt) {
    if (F->dtype != EBB_F64 && F->dtype != EBB_F32) return fail(c, EBB_E_TYPE, "spring: fields must be F32 or F64");
    *dt = F->dtype;
    return EBB_OK;
}

int lanes_for(const EdgeGraph& G) { return G.max_group <= 16 ? 16 : 32; }

}  // namespace
}  // namespace ebb

using namespace ebb;

extern "C" {

ebb_status ebb_spring_init_len(ebb_ctx ctx, ebb_rel edges, ebb_field pos, ebb_field rest_len, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    if (!c) return EBB_E_ARG;
    EdgeGraph G;
    EBB_TRY(edge_graph(c, edges, &G));
    Relation* E = get_rel(c, edges);
    Field* P = get_field(c, pos);
    if (!P) return fail(c, EBB_E_ARG, "spring: bad pos");
    ebb_dtype dt;
    EBB_TRY(float_dtype(c, P, &dt));
    Field *Pf, *Lf;
    EBB_TRY(check_vert_vec(c, pos, G.verts, dt, "pos", &Pf));
    EBB_TRY(check_scalar(c, rest_len, edges, dt, "rest_len", &Lf));
    const uint32_t* tail = (const uint32_t*)c->fields[E->grouped_by].ptr;
    cudaStream_t s = (cudaStream_t)stream;
    c->launches++;
    if (G.ne) {
        if (dt == EBB_F64)
            k_spring_init_len<double><<<grid_for(G.ne, 256), 256, 0, s>>>(G.ne, tail, G.head, (const double*)Pf->ptr,
                                                                          (double*)Lf->ptr);
        else
            k_spring_init_len<float><<<grid_for(G.ne, 256), 256, 0, s>>>(G.ne, tail, G.head, (const float*)Pf->ptr,
                                                                         (float*)Lf->ptr);
    }
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status ebb_spring_forces(ebb_ctx ctx, ebb_rel edges, ebb_field q, ebb_field rest_len, double K, ebb_field force,
                             int32_t accumulate, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    if (!c) return EBB_E_ARG;
    EdgeGraph G;
    EBB_TRY(edge_graph(c, edges, &G));
    Field* Q0 = get_field(c, q);
    if (!Q0) return fail(c, EBB_E_ARG, "spring: bad q");
    ebb_dtype dt;
    EBB_TRY(float_dtype(c, Q0, &dt));
    Field *Q, *L, *F;
    EBB_TRY(check_vert_vec(c, q, G.verts, dt, "q", &Q));
    EBB_TRY(check_vert_vec(c, force, G.verts, dt, "force", &F));
    EBB_TRY(check_scalar(c, rest_len, edges, dt, "rest_len", &L));
    if (F->ptr == Q->ptr) return fail(c, EBB_E_PHASE, "spring: force aliases q (read and reduced in one kernel)");
    cudaStream_t s = (cudaStream_t)stream;
    const int lpv = lanes_for(G);
    KernelTimer kt(c, EBB_K_SPRING, s);
    if (G.nv) {
#define EBB_SPF(R)                                                                                                  \
    do {                                                                                                            \
        auto k = lpv == 16 ? k_spring_forces<R, 16> : k_spring_forces<R, 32>;                                       \
        k<<<grid_for(G.nv * lpv, 256), 256, 0, s>>>(G.nv, G.index, G.head, (const R*)Q->ptr, (const R*)L->ptr,      \
                                                    (R)K, (R*)F->ptr, accumulate);                                  \
    } while (0)
        if (dt == EBB_F64) EBB_SPF(double);
        else EBB_SPF(float);
#undef EBB_SPF
    }
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status ebb_spring_apply(ebb_ctx ctx, ebb_field mass, double dt_step, ebb_field q, ebb_field qd, ebb_field force,
                            ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    if (!c) return EBB_E_ARG;
    Field* Q0 = get_field(c, q);
    if (!Q0) return fail(c, EBB_E_ARG, "spring: bad q");
    ebb_dtype dt;
    EBB_TRY(float_dtype(c, Q0, &dt));
    Field *Q, *QD, *F, *M;
    EBB_TRY(check_vert_vec(c, q, Q0->rel, dt, "q", &Q));
    EBB_TRY(check_vert_vec(c, qd, Q0->rel, dt, "qd", &QD));
    EBB_TRY(check_vert_vec(c, force, Q0->rel, dt, "force", &F));
    EBB_TRY(check_scalar(c, mass, Q0->rel, dt, "mass", &M));
    const uint64_t nv = c->rels[Q0->rel].size;
    cudaStream_t s = (cudaStream_t)stream;
    c->launches++;
    if (nv) {
        if (dt == EBB_F64)
            k_spring_apply<double><<<grid_for(3 * nv, 256), 256, 0, s>>>(nv, (const double*)M->ptr, dt_step,
                                                                         (double*)Q->ptr, (double*)QD->ptr,
                                                                         (double*)F->ptr);
        else
            k_spring_apply<float><<<grid_for(3 * nv, 256), 256, 0, s>>>(nv, (const float*)M->ptr, (float)dt_step,
                                                                        (float*)Q->ptr, (float*)QD->ptr,
                                                                        (float*)F->ptr);
    }
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status ebb_spring_step(ebb_ctx ctx, ebb_rel edges, ebb_field q_in, ebb_field q_out, ebb_field qd,
                           ebb_field rest_len, ebb_field mass, double K, double dt_step, ebb_field force,
                           ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    if (!c) return EBB_E_ARG;
    EdgeGraph G;
    EBB_TRY(edge_graph(c, edges, &G));
    Field* Q0 = get_field(c, q_in);
    if (!Q0) return fail(c, EBB_E_ARG, "spring: bad q_in");
    ebb_dtype dt;
    EBB_TRY(float_dtype(c, Q0, &dt));
    Field *Qi, *Qo, *QD, *L, *M, *F = nullptr;
    EBB_TRY(check_vert_vec(c, q_in, G.verts, dt, "q_in", &Qi));
    EBB_TRY(check_vert_vec(c, q_out, G.verts, dt, "q_out", &Qo));
    EBB_TRY(check_vert_vec(c, qd, G.verts, dt, "qd", &QD));
    EBB_TRY(check_scalar(c, rest_len, edges, dt, "rest_len", &L));
    EBB_TRY(check_scalar(c, mass, G.verts, dt, "mass", &M));
    if (force != EBB_NONE) EBB_TRY(check_vert_vec(c, force, G.verts, dt, "force", &F));
    if (Qo->ptr == Qi->ptr || QD->ptr == Qi->ptr || QD->ptr == Qo->ptr || (F && (F->ptr == Qi->ptr || F->ptr == Qo->ptr)))
        return fail(c, EBB_E_PHASE, "spring_step: q_in, q_out, qd and force must be distinct fields");
    cudaStream_t s = (cudaStream_t)stream;
    const int lpv = lanes_for(G);
    KernelTimer kt(c, EBB_K_SPRING, s);
    if (G.nv) {
#define EBB_SPS(R)                                                                                                  \
    do {                                                                                                            \
        auto k = lpv == 16 ? k_spring_step<R, 16> : k_spring_step<R, 32>;                                           \
        k<<<grid_for(G.nv * lpv, 256), 256, 0, s>>>(G.nv, G.index, G.head, (const R*)Qi->ptr, (const R*)L->ptr,     \
                                                    (const R*)M->ptr, (R)K, (R)dt_step, (R*)Qo->ptr, (R*)QD->ptr,   \
                                                    F ? (R*)F->ptr : nullptr);                                      \
    } while (0)
        if (dt == EBB_F64) EBB_SPS(double);
        else EBB_SPS(float);
#undef EBB_SPS
    }
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status ebb_kinetic_energy(ebb_ctx ctx, ebb_field mass, ebb_field qd, ebb_field out, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    if (!c) return EBB_E_ARG;
    Field* QD0 = get_field(c, qd);
    if (!QD0) return fail(c, EBB_E_ARG, "kinetic_energy: bad qd");
    ebb_dtype dt;
    EBB_TRY(float_dtype(c, QD0, &dt));
    Field *QD, *M;
    EBB_TRY(check_vert_vec(c, qd, QD0->rel, dt, "qd", &QD));
    EBB_TRY(check_scalar(c, mass, QD0->rel, dt, "mass", &M));
    Field* O = get_field(c, out);
    if (!O || !O->is_global || O->dtype != EBB_F64)
        return fail(c, EBB_E_TYPE, "kinetic_energy: out must be an F64 global");
    const uint64_t nv = c->rels[QD0->rel].size;
    cudaStream_t s = (cudaStream_t)stream;
    c->launches++;
    const unsigned g = nv ? (unsigned)std::min<uint64_t>(grid_for(nv, 256), 4096) : 1;
    if (dt == EBB_F64)
        k_kinetic_energy<double><<<g, 256, 0, s>>>(nv, (const double*)M->ptr, (const double*)QD->ptr, c->d_partials,
                                                   c->d_counter + 12, (double*)O->ptr);
    else
        k_kinetic_energy<float><<<g, 256, 0, s>>>(nv, (const float*)M->ptr, (const float*)QD->ptr, c->d_partials,
                                                  c->d_counter + 12, (double*)O->ptr);
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

}  // extern "C"
