// grid.cu -- the regular 2-D grid domain (P:733-772 affine indexing; Fig. 3,
// P:497-529 particle coupling).  nx x ny unit cells, cell
// (i, j) = [i, i+1) x [j, j+1) with row-major id i + nx j, periodic.  Keys
// between grid elements are computed arithmetically (the affine maps
// {{1,0,dx},{0,1,dy}} of P:757-770), never stored:
//   ebb_grid2_stencil        out[c] = sum_k w_k in[cell(i+dx_k, j+dy_k)]
//   ebb_grid2_point_locate   dual_cell = (floor(x-1/2) mod nx, floor(y-1/2) mod ny)
//   ebb_grid2_particle_vel   Fig. 3 update_particle_vel (bilinear over the
//                            dual cell's four cells)
// Readings: DESIGN.md §3 (22).
#include <cmath>

#include "ebb_internal.cuh"

namespace ebb {
namespace {

struct Stencil {
    int n;
    int dx[EBB_GRID2_MAX_STENCIL], dy[EBB_GRID2_MAX_STENCIL];
    double w[EBB_GRID2_MAX_STENCIL];
};

__device__ __forceinline__ uint32_t wrap(int64_t i, uint32_t n) {
    if (i >= 0 && i < (int64_t)n) return (uint32_t)i;          // the common case: no division
    if (i < 0 && i >= -(int64_t)n) return (uint32_t)(i + n);
    if (i >= (int64_t)n && i < 2 * (int64_t)n) return (uint32_t)(i - n);
    int64_t r = i % (int64_t)n;
    return (uint32_t)(r < 0 ? r + n : r);
}

// thread = ROWS cells of one column (x fastest across the warp: coalesced
// rows; neighbours served by L1/L2); the column offset of each stencil point
// is wrapped once per thread, the rows give independent sums.  ROWS = 4 in
// fp32, 1 in fp64 (measured)
template <typename R>
__host__ __device__ constexpr int grid2_rows() { return sizeof(R) == 4 ? 4 : 1; }
template <typename R, int NC>
__global__ void __launch_bounds__(256) k_grid2_stencil(uint32_t nx, uint32_t ny, const R* __restrict__ in,
                                                       R* __restrict__ out, Stencil st) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t j0 = (blockIdx.y * blockDim.y + threadIdx.y) * grid2_rows<R>();
    if (i >= nx || j0 >= ny) return;
    R acc[grid2_rows<R>()][NC];
#pragma unroll
    for (int r = 0; r < grid2_rows<R>(); ++r)
#pragma unroll
        for (int a = 0; a < NC; ++a) acc[r][a] = R(0);
    // offsets arrive reduced to [0, n) on the host: one add and one
    // conditional subtract per axis, 32-bit indices (cells < 2^32)
    for (int k = 0; k < st.n; ++k) {
        uint32_t i2 = i + (uint32_t)st.dx[k];
        i2 = i2 >= nx ? i2 - nx : i2;
        const R w = (R)st.w[k];
#pragma unroll
        for (int r = 0; r < grid2_rows<R>(); ++r) {
            uint32_t j2 = j0 + r + (uint32_t)st.dy[k];
            j2 = j2 >= ny ? j2 - ny : j2;
            j2 = j2 >= ny ? j2 - ny : j2;      // (j0 + r may itself pass ny on the last rows)
            const uint32_t c = i2 + nx * j2;
#pragma unroll
            for (int a = 0; a < NC; ++a) acc[r][a] += w * in[(size_t)NC * c + a];
        }
    }
#pragma unroll
    for (int r = 0; r < grid2_rows<R>(); ++r) {
        if (j0 + r >= ny) break;
        const size_t c = i + (size_t)nx * (j0 + r);
#pragma unroll
        for (int a = 0; a < NC; ++a) out[NC * c + a] = acc[r][a];
    }
}

template <typename R>
__global__ void k_grid2_point_locate(uint64_t np, uint32_t nx, uint32_t ny, const R* __restrict__ pos,
                                     uint32_t* __restrict__ dual) {
    const uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (p >= np) return;
    const int64_t a = (int64_t)floor((double)pos[3 * p] - 0.5), b = (int64_t)floor((double)pos[3 * p + 1] - 0.5);
    dual[p] = wrap(a, nx) + nx * wrap(b, ny);
}

template <typename R, int NC>
__global__ void k_grid2_particle_vel(uint64_t np, uint32_t nx, uint32_t ny, const R* __restrict__ cell_vel,
                                     const R* __restrict__ pos, const uint32_t* __restrict__ dual,
                                     R* __restrict__ vel) {
    const uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (p >= np) return;
    // the fractional parts in fp64 for both dtypes: the same decision as
    // PointLocate's floor (a particle within an ulp of a cell centre cannot
    // get weights of the neighbouring dual cell)
    const double px = (double)pos[3 * p] - 0.5, py = (double)pos[3 * p + 1] - 0.5;
    const R x1 = (R)(px - floor(px)), y1 = (R)(py - floor(py));
    const R x0 = R(1) - x1, y0 = R(1) - y1;
    const uint32_t d = dual[p], a = d % nx, b = d / nx;
    const uint32_t a1 = a + 1 == nx ? 0 : a + 1, b1 = b + 1 == ny ? 0 : b + 1;
    const uint64_t c00 = a + (uint64_t)nx * b, c10 = a1 + (uint64_t)nx * b;
    const uint64_t c01 = a + (uint64_t)nx * b1, c11 = a1 + (uint64_t)nx * b1;
#pragma unroll
    for (int k = 0; k < NC; ++k)
        vel[NC * p + k] = x0 * y0 * cell_vel[NC * c00 + k] + x1 * y0 * cell_vel[NC * c10 + k] +
                          x0 * y1 * cell_vel[NC * c01 + k] + x1 * y1 * cell_vel[NC * c11 + k];
}

Relation* grid_rel(Ctx* c, ebb_rel r, int kind, const char* what) {
    Relation* R = get_rel(c, r);
    if (!R || R->grid_kind != kind) {
        fail(c, EBB_E_TYPE, "%s must be the %s relation of an ebb_grid2_new grid", what,
             kind == 1 ? "cells" : "dual-cells");
        return nullptr;
    }
    return R;
}

}  // namespace
}  // namespace ebb

using namespace ebb;

extern "C" {

ebb_status ebb_grid2_new(ebb_ctx ctx, const char* name, uint32_t nx, uint32_t ny, ebb_grid2* out) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || !name || !out) return fail(c, EBB_E_ARG, "null argument");
    if (nx == 0 || ny == 0) return fail(c, EBB_E_SIZE, "grid2: zero dimension");
    if ((uint64_t)nx * ny > 0xFFFFFFFFull) return fail(c, EBB_E_RANGE, "grid2: more than 2^32 cells");
    std::string n(name);
    EBB_TRY(ebb_relation_new(ctx, (n + ".cells").c_str(), (uint64_t)nx * ny, &out->cells));
    EBB_TRY(ebb_relation_new(ctx, (n + ".dual_cells").c_str(), (uint64_t)nx * ny, &out->dual_cells));
    for (ebb_rel r : {out->cells, out->dual_cells}) {
        Relation& R = c->rels[r];
        R.dims[0] = nx;
        R.dims[1] = ny;
        R.grid_kind = r == out->cells ? 1 : 2;
        R.grid_peer = r == out->cells ? out->dual_cells : out->cells;
    }
    return EBB_OK;
}

ebb_status ebb_grid2_stencil(ebb_ctx ctx, ebb_rel cells, ebb_field in, ebb_field out, int32_t npts,
                             const int32_t* offsets, const double* weights, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c || (npts > 0 && (!offsets || !weights))) return fail(c, EBB_E_ARG, "null argument");
    Relation* G = grid_rel(c, cells, 1, "cells");
    if (!G) return EBB_E_TYPE;
    if (npts < 1 || npts > EBB_GRID2_MAX_STENCIL) return fail(c, EBB_E_ARG, "grid2_stencil: 1..%d points", EBB_GRID2_MAX_STENCIL);
    Field* I = get_field(c, in);
    Field* O = get_field(c, out);
    if (!I || !O) return fail(c, EBB_E_ARG, "grid2_stencil: bad field");
    if (I->rel != cells || O->rel != cells || I->dtype != O->dtype || I->comps() != O->comps() ||
        (I->dtype != EBB_F32 && I->dtype != EBB_F64) || I->comps() > 4 || (I->comps() > 1 && (I->layout != EBB_AOS || O->layout != EBB_AOS)))
        return fail(c, EBB_E_TYPE, "grid2_stencil: in, out must be F32/F64 AOS fields of the same shape (<= 4 "
                                   "components) on the cells");
    if (I->ptr == O->ptr) return fail(c, EBB_E_PHASE, "grid2_stencil: out aliases in (neighbours read it)");
    Stencil st;
    st.n = npts;
    const uint32_t nx = G->dims[0], ny = G->dims[1];
    for (int k = 0; k < npts; ++k) {   // periodic: reduce each offset to [0, n)
        st.dx[k] = (int)((offsets[2 * k] % (int64_t)nx + nx) % nx);
        st.dy[k] = (int)((offsets[2 * k + 1] % (int64_t)ny + ny) % ny);
        st.w[k] = weights[k];
    }
    cudaStream_t s = (cudaStream_t)stream;
    KernelTimer kt(c, EBB_K_GRID, s);
#define EBB_GS(R, NC)                                                                                               \
    k_grid2_stencil<R, NC><<<dim3((nx + 31) / 32, (ny + 8 * grid2_rows<R>() - 1) / (8 * grid2_rows<R>())),       \
                             dim3(32, 8), 0, s>>>(nx, ny, (const R*)I->ptr, (R*)O->ptr, st)
#define EBB_GSD(R)                            \
    do {                                      \
        switch (I->comps()) {                 \
            case 1: EBB_GS(R, 1); break;      \
            case 2: EBB_GS(R, 2); break;      \
            case 3: EBB_GS(R, 3); break;      \
            default: EBB_GS(R, 4); break;     \
        }                                     \
    } while (0)
    if (I->dtype == EBB_F64) EBB_GSD(double);
    else EBB_GSD(float);
#undef EBB_GSD
#undef EBB_GS
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status ebb_grid2_point_locate(ebb_ctx ctx, ebb_field pos, ebb_field dual_cell, ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c) return EBB_E_ARG;
    Field* P = get_field(c, pos);
    Field* K = get_field(c, dual_cell);
    if (!P || !K) return fail(c, EBB_E_ARG, "grid2_point_locate: bad field");
    if (K->dtype != EBB_KEY || K->comps() != 1 || K->rel != P->rel)
        return fail(c, EBB_E_TYPE, "grid2_point_locate: dual_cell must be a scalar key-field on the particles");
    Relation* D = grid_rel(c, K->key_target, 2, "dual_cell's target");
    if (!D) return EBB_E_TYPE;
    if (P->comps() != 3 || P->layout != EBB_AOS || (P->dtype != EBB_F32 && P->dtype != EBB_F64))
        return fail(c, EBB_E_TYPE, "grid2_point_locate: pos must be an AOS vec3 F32/F64 field");
    const uint64_t np = c->rels[P->rel].size;
    cudaStream_t s = (cudaStream_t)stream;
    c->launches++;
    if (P->dtype == EBB_F64)
        k_grid2_point_locate<double><<<grid_for(np, 256), 256, 0, s>>>(np, D->dims[0], D->dims[1],
                                                                       (const double*)P->ptr, (uint32_t*)K->ptr);
    else
        k_grid2_point_locate<float><<<grid_for(np, 256), 256, 0, s>>>(np, D->dims[0], D->dims[1],
                                                                      (const float*)P->ptr, (uint32_t*)K->ptr);
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

ebb_status ebb_grid2_particle_vel(ebb_ctx ctx, ebb_field dual_cell, ebb_field cell_vel, ebb_field pos, ebb_field vel,
                                  ebb_stream stream) {
    Ctx* c = (Ctx*)ctx;
    EBB_DEVICE_GUARD(c);
    if (!c) return EBB_E_ARG;
    Field* K = get_field(c, dual_cell);
    Field* CV = get_field(c, cell_vel);
    Field* P = get_field(c, pos);
    Field* V = get_field(c, vel);
    if (!K || !CV || !P || !V) return fail(c, EBB_E_ARG, "grid2_particle_vel: bad field");
    if (K->dtype != EBB_KEY || K->comps() != 1) return fail(c, EBB_E_TYPE, "grid2_particle_vel: bad dual_cell key");
    Relation* D = grid_rel(c, K->key_target, 2, "dual_cell's target");
    if (!D) return EBB_E_TYPE;
    const ebb_dtype dt = CV->dtype;
    if ((dt != EBB_F32 && dt != EBB_F64) || CV->rel != D->grid_peer || CV->comps() < 1 || CV->comps() > 4 ||
        (CV->comps() > 1 && CV->layout != EBB_AOS))
        return fail(c, EBB_E_TYPE, "grid2_particle_vel: cell_vel must be an AOS F32/F64 field on the grid's cells");
    if (P->rel != K->rel || P->comps() != 3 || P->dtype != dt || P->layout != EBB_AOS)
        return fail(c, EBB_E_TYPE, "grid2_particle_vel: pos must be an AOS vec3 field of cell_vel's dtype on the "
                                   "particles");
    if (V->rel != K->rel || V->comps() != CV->comps() || V->dtype != dt || (V->comps() > 1 && V->layout != EBB_AOS))
        return fail(c, EBB_E_TYPE, "grid2_particle_vel: vel must have cell_vel's shape, on the particles");
    if (V->ptr == P->ptr) return fail(c, EBB_E_PHASE, "grid2_particle_vel: vel aliases pos");
    const uint64_t np = c->rels[K->rel].size;
    const uint32_t nx = D->dims[0], ny = D->dims[1];
    cudaStream_t s = (cudaStream_t)stream;
    KernelTimer kt(c, EBB_K_GRID, s);
#define EBB_PV(R, NC)                                                                                               \
    k_grid2_particle_vel<R, NC><<<grid_for(np, 256), 256, 0, s>>>(np, nx, ny, (const R*)CV->ptr, (const R*)P->ptr,  \
                                                                  (const uint32_t*)K->ptr, (R*)V->ptr)
#define EBB_PVD(R)                        \
    do {                                  \
        switch (CV->comps()) {            \
            case 1: EBB_PV(R, 1); break;  \
            case 2: EBB_PV(R, 2); break;  \
            case 3: EBB_PV(R, 3); break;  \
            default: EBB_PV(R, 4); break; \
        }                                 \
    } while (0)
    if (dt == EBB_F64) EBB_PVD(double);
    else EBB_PVD(float);
#undef EBB_PVD
#undef EBB_PV
    EBB_CUDA(c, cudaGetLastError());
    return EBB_OK;
}

}  // extern "C"
