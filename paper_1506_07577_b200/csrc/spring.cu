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
#include <cstdlib>

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
        const uint32_t e1 = index[v + 1];
#pragma unroll 4
        for (uint32_t e = index[v] + lane; e < e1; e += LPV) {
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
__global__ void k_spring_apply(uint64_t nv, int qs, const R* __restrict__ mass, R dt, R* __restrict__ q,
                               R* __restrict__ qd, R* __restrict__ force) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= (uint64_t)qs * nv || i % qs == 3) return;   // (padding lane of a 4x1 record)
    R v = qd[i], qn;
    spring_update(force[i], mass[i / qs], dt, q[i], v, qn);
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
    const unsigned lane = threadIdx.x % LPV;
    // the update operands do not depend on the forces: load them first so
    // their latency overlaps the row walk (components c = lane, lane + LPV, ..)
    constexpr int NC = LPV >= 3 ? 1 : (3 + LPV - 1) / LPV;
    R w[NC], qi[NC], mv = 1;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        const unsigned c = lane + k * LPV;
        w[k] = qi[k] = 0;
        if (live && c < 3) {
            w[k] = qd[3 * v + c];
            qi[k] = q[3 * v + c];
        }
    }
    if (live && lane < 3) mv = mass[v];
    R s[3];
    spring_row_sum<R, LPV>(v, live, index, head, q, rest, K, s[0], s[1], s[2]);
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        const unsigned c = lane + k * LPV;
        if (live && c < 3) {
            const R f = c == 0 ? s[0] : c == 1 ? s[1] : s[2];
            R qn;
            spring_update(f, mv, dt, qi[k], w[k], qn);
            qout[3 * v + c] = qn;
            qd[3 * v + c] = w[k];
            if (force) force[3 * v + c] = f;
        }
    }
}

// Row-staged variant (the default): a CTA owns SB consecutive vertices, whose
// rows are one contiguous range of the grouped relation: the CTA
// first copies that range of head keys and rest lengths into shared memory
// with coalesced loads, then thread = vertex walks its rows there (only the
// q gathers go to L2).  STEP: the fused iteration (else forces only).
#define SPRING_SB 128
#ifndef SPRING_B
#define SPRING_B 4      // rows gathered together per thread
#endif
template <typename R>
struct SpV4;
template <>
struct SpV4<double> {
    using T = double4;
};
template <>
struct SpV4<float> {
    using T = float4;
};
// QS = record stride of the vertex vectors: 3 (vec3) or 4 (padded: one
// 32-byte fp64 / 16-byte fp32 access per gathered record)
template <typename R, int QS>
__device__ __forceinline__ void ld_rec(const R* __restrict__ p, uint64_t v, R& a, R& b, R& c) {
    if constexpr (QS == 4) {
        const auto r = reinterpret_cast<const typename SpV4<R>::T*>(p)[v];
        a = r.x;
        b = r.y;
        c = r.z;
    } else {
        a = p[3 * v];
        b = p[3 * v + 1];
        c = p[3 * v + 2];
    }
}
template <typename R, bool STEP, int QS>
__global__ void __launch_bounds__(SPRING_SB) k_spring_staged(uint64_t nv, const uint32_t* __restrict__ index,
                                                             const uint32_t* __restrict__ head,
                                                             const R* __restrict__ q, const R* __restrict__ rest,
                                                             const R* __restrict__ mass, R K, R dt,
                                                             R* __restrict__ qout, R* __restrict__ qd,
                                                             R* __restrict__ force, int accumulate) {
    extern __shared__ __align__(16) unsigned char sp_smem[];
    const uint64_t v0 = (uint64_t)blockIdx.x * SPRING_SB;
    const uint64_t v1 = v0 + SPRING_SB < nv ? v0 + SPRING_SB : nv;
    const uint32_t e0 = index[v0], n = index[v1] - e0;
    R* ls = reinterpret_cast<R*>(sp_smem);
    uint32_t* hs = reinterpret_cast<uint32_t*>(ls + ((n + 1) & ~1u));
    // asynchronous copies (cp.async: no registers held while in flight, so
    // every row of the range is requested at once)
    for (uint32_t k = threadIdx.x; k < n; k += SPRING_SB) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(hs + k)),
                     "l"(head + e0 + k)
                     : "memory");
        if constexpr (sizeof(R) == 8)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(ls + k)),
                         "l"(rest + e0 + k)
                         : "memory");
        else
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(ls + k)),
                         "l"(rest + e0 + k)
                         : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    const uint64_t v = v0 + threadIdx.x;
    const bool live = v < v1;
    R w[3], qv[3], mv = 1;
    uint32_t r0 = 0, r1 = 0;
    if (live) {
        ld_rec<R, QS>(q, v, qv[0], qv[1], qv[2]);
        if (STEP) {
            ld_rec<R, QS>(qd, v, w[0], w[1], w[2]);
            mv = mass[v];
        } else {
            w[0] = w[1] = w[2] = R(0);
        }
        r0 = index[v] - e0;
        r1 = index[v + 1] - e0;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (!live) return;
    R s0 = 0, s1 = 0, s2 = 0;
    // batches of SPRING_B rows: every gather of a batch is issued before the
    // first sqrt / division (whose slow-path branches end the scheduler's
    // basic block), so SPRING_B gathers are in flight per thread
    constexpr int B = SPRING_B;
    for (uint32_t rb = r0; rb < r1; rb += B) {
        R qh[B][3], Lb[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const uint32_t r = rb + u < r1 ? rb + u : r1 - 1;   // (a repeated row is masked below)
            Lb[u] = ls[r];
            ld_rec<R, QS>(q, (uint64_t)hs[r], qh[u][0], qh[u][1], qh[u][2]);
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const R d0 = qh[u][0] - qv[0], d1 = qh[u][1] - qv[1], d2 = qh[u][2] - qv[2];
            const R len = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
            const R c = len > R(0) ? Lb[u] / len : R(0);
            if (rb + u < r1) {
                s0 += K * (c * d0 - d0);
                s1 += K * (c * d1 - d1);
                s2 += K * (c * d2 - d2);
            }
        }
    }
    const R f[3] = {s0, s1, s2};
    if (STEP) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            R qn, wc = w[c];
            spring_update(f[c], mv, dt, qv[c], wc, qn);
            qout[QS * v + c] = qn;
            qd[QS * v + c] = wc;
            if (force) force[QS * v + c] = f[c];
        }
    } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) force[QS * v + c] = accumulate ? f[c] + force[QS * v + c] : f[c];
    }
}

template <typename R>
__global__ void __launch_bounds__(256) k_kinetic_energy(uint64_t nv, int qs, const R* __restrict__ mass,
                                                        const R* __restrict__ qd, double* __restrict__ partials,
                                                        unsigned int* __restrict__ counter, double* __restrict__ out) {
    double acc = 0.0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x) {
        const double a = qd[qs * v], b = qd[qs * v + 1], c = qd[qs * v + 2];
        acc += 0.5 * (double)mass[v] * (a * a + b * b + c * c);
    }
    double tot;
    if (block_sum_last_done(acc, partials, counter, &tot)) *out = tot;
}

ebb_status check_vert_vec(Ctx* c, ebb_field f, ebb_rel verts, ebb_dtype dt, const char* what, Field** out) {
    Field* F = get_field(c, f);
    if (!F) return fail(c, EBB_E_ARG, "spring: bad %s", what);
    if (F->rel != verts || (F->comps() != 3 && F->comps() != 4) || F->layout != EBB_AOS || F->dtype != dt)
        return fail(c, EBB_E_TYPE, "spring: %s must be an AOS vec3 (or padded 4x1) field of the %s dtype on the "
                    "vertices", what, dt == EBB_F64 ? "F64" : "F32");
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

// lanes per vertex of the register-path query-loop (EBB_SPRING_LPV = 1..32);
// 0 = the row-staged kernel.  Defaults (measured): the fused
// step and padded records use the staged kernel, vec3 forces-only the
// thread-per-vertex register path.
int lanes_for(const EdgeGraph& G, bool step, int qs) {
    const char* e = getenv("EBB_SPRING_LPV");
    if (e) {
        const int l = atoi(e);
        if (l == 1 || l == 2 || l == 4 || l == 8 || l == 16 || l == 32) return l;
    }
    const size_t smem = (size_t)SPRING_SB * (G.max_group ? G.max_group : 1) * 12 + 16;
    if (qs == 4 || (step && smem <= 160 * 1024)) return 0;
    return 1;
}

template <typename R, bool STEP>
ebb_status launch_staged(Ctx* c, const EdgeGraph& G, int qs, const R* q, const R* rest, const R* mass, R K, R dt,
                         R* qout, R* qd, R* force, int accumulate, cudaStream_t s) {
    const size_t smem = (size_t)SPRING_SB * (G.max_group ? G.max_group : 1) * (sizeof(R) + 4) + 16;
    if (smem > 200 * 1024)
        return fail(c, EBB_E_RANGE, "spring: a vertex with %u edge rows needs %zu B of shared memory for the staged "
                    "kernel (padded records have no register-path fallback; use vec3 fields)", G.max_group, smem);
    auto kern = qs == 4 ? k_spring_staged<R, STEP, 4> : k_spring_staged<R, STEP, 3>;
    if (smem > 48 * 1024)
        EBB_CUDA(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid_for(G.nv, SPRING_SB), SPRING_SB, smem, s>>>(G.nv, G.index, G.head, q, rest, mass, K, dt, qout, qd,
                                                           force, accumulate);
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

}  // namespace
}  // namespace ebb

using namespace ebb;

extern "C" {

ebb_status ebb_spring_init_len(ebb_ctx ctx, ebb_rel edges, ebb_field pos, ebb_field rest_len, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
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
    if (Pf->comps() != 3) return fail(c, EBB_E_TYPE, "spring_init_len: pos must be a vec3 (3x1) field");
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
    EBB_DEVICE_GUARD(c);
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
    const int qs = (int)Q->comps();
    if (F->comps() != Q->comps()) return fail(c, EBB_E_TYPE, "spring: q and force must have the same record shape");
    const int lpv = lanes_for(G, false, qs);
    if (qs == 4 && lpv != 0) return fail(c, EBB_E_TYPE, "spring: padded records need the staged kernel");
    KernelTimer kt(c, EBB_K_SPRING, s);
    if (G.nv && lpv == 0) {
        if (dt == EBB_F64)
            return launch_staged<double, false>(c, G, qs, (const double*)Q->ptr, (const double*)L->ptr, nullptr, K,
                                                0.0, nullptr, nullptr, (double*)F->ptr, accumulate, s);
        return launch_staged<float, false>(c, G, qs, (const float*)Q->ptr, (const float*)L->ptr, nullptr, (float)K,
                                           0.f, nullptr, nullptr, (float*)F->ptr, accumulate, s);
    }
    if (G.nv) {
#define EBB_SPF(R)                                                                                                  \
    do {                                                                                                            \
        auto k = lpv == 1 ? k_spring_forces<R, 1> : lpv == 2 ? k_spring_forces<R, 2>                               \
               : lpv == 4 ? k_spring_forces<R, 4> : lpv == 8 ? k_spring_forces<R, 8>                               \
               : lpv == 16 ? k_spring_forces<R, 16> : k_spring_forces<R, 32>;                                       \
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
    EBB_DEVICE_GUARD(c);
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
    if (QD->comps() != Q->comps() || F->comps() != Q->comps())
        return fail(c, EBB_E_TYPE, "spring_apply: q, qd, force must have the same record shape");
    const uint64_t nv = c->rels[Q0->rel].size;
    cudaStream_t s = (cudaStream_t)stream;
    c->launches++;
    if (nv) {
        if (dt == EBB_F64)
            k_spring_apply<double><<<grid_for(Q->comps() * nv, 256), 256, 0, s>>>(nv, (int)Q->comps(),
                                                                         (const double*)M->ptr, dt_step,
                                                                         (double*)Q->ptr, (double*)QD->ptr,
                                                                         (double*)F->ptr);
        else
            k_spring_apply<float><<<grid_for(Q->comps() * nv, 256), 256, 0, s>>>(nv, (int)Q->comps(),
                                                                        (const float*)M->ptr, (float)dt_step,
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
    EBB_DEVICE_GUARD(c);
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
    const int qs = (int)Qi->comps();
    if (Qo->comps() != Qi->comps() || QD->comps() != Qi->comps() || (F && F->comps() != Qi->comps()))
        return fail(c, EBB_E_TYPE, "spring_step: q_in, q_out, qd, force must have the same record shape");
    const int lpv = lanes_for(G, true, qs);
    if (qs == 4 && lpv != 0) return fail(c, EBB_E_TYPE, "spring: padded records need the staged kernel");
    KernelTimer kt(c, EBB_K_SPRING, s);
    if (G.nv && lpv == 0) {
        if (dt == EBB_F64)
            return launch_staged<double, true>(c, G, qs, (const double*)Qi->ptr, (const double*)L->ptr,
                                               (const double*)M->ptr, K, dt_step, (double*)Qo->ptr,
                                               (double*)QD->ptr, F ? (double*)F->ptr : nullptr, 0, s);
        return launch_staged<float, true>(c, G, qs, (const float*)Qi->ptr, (const float*)L->ptr,
                                          (const float*)M->ptr, (float)K, (float)dt_step, (float*)Qo->ptr,
                                          (float*)QD->ptr, F ? (float*)F->ptr : nullptr, 0, s);
    }
    if (G.nv) {
#define EBB_SPS(R)                                                                                                  \
    do {                                                                                                            \
        auto k = lpv == 1 ? k_spring_step<R, 1> : lpv == 2 ? k_spring_step<R, 2>                                   \
               : lpv == 4 ? k_spring_step<R, 4> : lpv == 8 ? k_spring_step<R, 8>                                   \
               : lpv == 16 ? k_spring_step<R, 16> : k_spring_step<R, 32>;                                           \
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
    EBB_DEVICE_GUARD(c);
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
        k_kinetic_energy<double><<<g, 256, 0, s>>>(nv, (int)QD->comps(), (const double*)M->ptr, (const double*)QD->ptr, c->d_partials,
                                                   c->d_counter + 12, (double*)O->ptr);
    else
        k_kinetic_energy<float><<<g, 256, 0, s>>>(nv, (int)QD->comps(), (const float*)M->ptr, (const float*)QD->ptr, c->d_partials,
                                                  c->d_counter + 12, (double*)O->ptr);
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

}  // extern "C"
