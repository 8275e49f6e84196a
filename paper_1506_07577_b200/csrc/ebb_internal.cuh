// ebb_internal.cuh -- runtime state behind the C ABI (include/ebb.h).
// Relations and fields follow the paper's relational model (P:405-420,
// P:663-690).  Everything here is host C++ plus small device
// helpers; kernels live in the *.cu files next to this header.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/ebb.h"

struct ebb_ctx_s {};

namespace ebb {

constexpr size_t kFieldSlack = 64;  // bytes past the end of every library-owned column

struct Field {
    std::string name;
    ebb_rel rel = EBB_NONE;
    ebb_dtype dtype = EBB_F64;
    uint32_t rows = 1, cols = 1;
    ebb_layout layout = EBB_AOS;
    void* ptr = nullptr;
    bool owned = false;
    bool alive = false;
    ebb_rel key_target = EBB_NONE;  // key-fields only
    bool is_global = false;
    uint32_t comps() const { return rows * cols; }
};

struct Relation {
    std::string name;
    uint64_t size = 0;
    std::vector<ebb_field> fields;
    ebb_field grouped_by = EBB_NONE;   // key-field this relation is grouped by
    ebb_field index = EBB_NONE;        // hidden CSR index on the source
    uint32_t max_group = 0;            // longest range of an index on this relation
    uint32_t max_chunk16 = 0;          // most rows of 16 consecutive sources (a TMA matvec chunk)
    uint32_t max_chunk64 = 0;          // most rows of 64 consecutive sources (register matvec chunk)
    // regular 2-D grid (ebb_grid2_new): dims, kind (1 = cells, 2 = dual cells)
    // and the other relation of the same grid
    uint32_t dims[2] = {0, 0};
    int grid_kind = 0;
    ebb_rel grid_peer = EBB_NONE;
    bool alive = true;                 // false after ebb_relation_free
};

// Plan of the SEGMENTED element map (seg_map.cu, built once per mesh on the
// host): variable vertex tiles (consecutive SFC-ordered vertices) grown until
// the tets touching them ("instances") reach `ni`, so one tile is one pass of
// the kernel.  Per tile: its instance tet ids; per canonical edge row (tail <=
// head) owned by the tile a "slot" (global row and transpose row); its phase-2
// work as "items" = chunks of at most `chunk` entries of one slot's (or one
// vertex's force) contribution list, the chunks of a list in consecutive lanes
// of one warp (combined by shuffles), every tile's items padded to whole warps.
struct SegPlan {
    ebb_field v = EBB_NONE, e = EBB_NONE;
    int ni = 0;                       // instance cap per tile (= threads per CTA)
    uint32_t ntiles = 0, max_ent = 0, max_items = 0;
    uint64_t ninst = 0, nslots = 0, nent = 0, nitems = 0;
    double host_ms = 0;               // plan build time (host)
    unsigned host_threads = 1;        // host threads of the per-tile build
    uint4* tdesc = nullptr;           // ntiles + 1: {first vertex, instance offset, item offset
                                      //   (multiple of 32), entry offset (multiple of 4)}
    uint32_t run = 1;                 // consecutive tiles per CTA run (state of shared tets carried)
    uint2* inst = nullptr;            // ninst: each tile's NEW instances (tet, state slot | own << 16)
    uint4* items = nullptr;           // nitems: {meta, row, transpose row | vertex, 0}; meta =
                                      //   begin[0:16) count[16:23) pos[23:26) last[26:29) kind[29:31)
                                      //   kind 0 off-diagonal row, 1 self row + vertex force; row ~0 = padding
    uint32_t* ents = nullptr;         // nent: block entries oi | oj << 13 | pair << 26 (oi, oj =
                                      //   3 i NT + lr, 3 j NT + lr: state word offsets of k_i, k_j),
                                      //   force entries 3 corner NT + lr (offset of f_corner)
    void release() {
        cudaFree(tdesc); cudaFree(inst); cudaFree(items); cudaFree(ents);
        ents = nullptr;
        inst = nullptr;
        tdesc = items = nullptr;
    }
};

// Plan of the CHUNK element map (chunk_map.cu, built on the device once per
// mesh): tiles of NT consecutive tets, each computed once; per tile its items
// (chunks of segments = the blocks of the tile's tets summed into one row),
// outgoing segments first; message slots; (sender -> receiver) tile lists.
struct ChunkPlan {
    ebb_field v = EBB_NONE, e = EBB_NONE;
    int nt_tile = 0;                  // tets per tile = threads per CTA
    uint32_t ntiles = 0;
    uint64_t nseg = 0, nmsg = 0, npair = 0, nitems = 0, nzrows = 0, nzverts = 0;
    double build_ms = 0;
    uint4* tdesc = nullptr;           // ntiles + 1: {item0, outgoing items, owned items, receiver list offset}
    uint32_t* expect = nullptr;       // ntiles: sender tiles of each tile
    uint32_t* recv = nullptr;         // receiver tiles, CSR by sender
    uint32_t* cnt = nullptr;          // ntiles: arrivals (reset by the receiver)
    uint32_t* ticket = nullptr;       // [1] CTAs done (last one reduces the energy)
    double* tile_e = nullptr;         // ntiles: energy of each tile
    uint4* items = nullptr;           // nitems
    uint32_t* ents = nullptr;         // 10 NT per tile: block entries in segment order
    void* msg = nullptr;              // nmsg x 128 B
    uint32_t* zrows = nullptr;        // rows no tet contributes to
    uint32_t* zverts = nullptr;       // vertices in no tet
    uint32_t* srows = nullptr;        // canonical rows fed by more than one tile (zeroed before a RED-mode map)
    uint64_t nsrows = 0;
    void release();
};

// Plan of the COLOURED element map (color_map.cu): tets grouped by colour
// (no two tets of a colour share a vertex).
struct ColorPlan {
    ebb_field v = EBB_NONE;
    int ncolors = 0;
    double host_ms = 0;
    std::vector<uint32_t> offsets;    // ncolors + 1 (host)
    uint32_t* order = nullptr;        // nt: tet ids by colour
    void release() {
        cudaFree(order);
        order = nullptr;
    }
};

// Upper-triangle view of a grouped edge relation (rows tail <= head), used by
// the symmetric-storage PCG (solver.cu): CSR offsets per vertex, head and
// source (full) row of each upper row, and the compressed system matrices.
struct UpperCSR {
    ebb_rel edges = EBB_NONE;
    uint64_t nu = 0;
    uint32_t max_group = 0;
    uint32_t max_chunk16 = 0;   // rows of the largest 16-vertex chunk of the upper triangle
    uint32_t* uptr = nullptr;   // nverts + 1
    uint32_t* uhead = nullptr;  // nu
    uint32_t* usrc = nullptr;   // nu: row of the full relation
    std::vector<std::pair<ebb_field, void*>> ahalf;   // per system matrix: 9 planes of nu (+ slack)
    void release() {
        cudaFree(uptr); cudaFree(uhead); cudaFree(usrc);
        for (auto& a : ahalf) cudaFree(a.second);
        ahalf.clear();
        uptr = uhead = usrc = nullptr;
    }
};

struct Ctx : ebb_ctx_s {
    int device = 0;
    std::vector<Relation> rels;
    std::vector<Field> fields;
    std::string err;
    ebb_rel globals_rel = EBB_NONE;
    unsigned long long* d_err = nullptr;   // device error word [4]
    // reusable scratch (grown on demand, never shrunk)
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    double* d_partials = nullptr;          // per-block reduction partials
    unsigned int* d_counter = nullptr;     // last-block-done tickets
    int num_sms = 148;
    // instrumentation
    unsigned long long launches = 0;
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    struct TimedLaunch { int kernel; cudaEvent_t a, b; };
    std::vector<TimedLaunch> timed;
    std::vector<SegPlan*> segplans; // invalidated by any relation permutation
    std::vector<ChunkPlan*> chunkplans; // (same)
    struct AutoMap { ebb_field v, e; int strategy; };
    std::vector<AutoMap> auto_map;      // AUTO's strategy per (v, e) mesh (same lifetime as the plans)
    std::vector<ColorPlan*> colorplans; // (same)
    std::vector<UpperCSR*> uppers;      // (same)
    void* comm = nullptr;               // ncclComm_t (comm.cu)
    std::vector<void*> peer_groups;     // launch groups of ebb_cg_peer_bind (solver.cu)
    int comm_size = 1, comm_rank = 0;
    struct GraphRec {
        cudaGraphExec_t exec = nullptr;
        unsigned long long launches = 0;
    };
    std::vector<GraphRec> graphs;
    unsigned long long capture_launch0 = 0;
};

// Brackets one hot-kernel launch with events on its stream when timing is on.
struct KernelTimer {
    Ctx* c;
    int kernel;
    cudaStream_t s;
    cudaEvent_t a = nullptr, b = nullptr;
    unsigned int flags = cudaEventRecordDefault;
    KernelTimer(Ctx* c_, int k, cudaStream_t s_) : c(c_), kernel(k), s(s_) {
        c->launches++;
        if (c->timing && c->ev_used + 2 <= c->ev_pool.size()) {
            // under stream capture the records must be external event nodes so
            // that every replay re-records them (host-visible, timeable)
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            if (s && cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
                flags = cudaEventRecordExternal;
            a = c->ev_pool[c->ev_used++];
            b = c->ev_pool[c->ev_used++];
            cudaEventRecordWithFlags(a, s, flags);
        }
    }
    ~KernelTimer() {
        if (a) {
            cudaEventRecordWithFlags(b, s, flags);
            c->timed.push_back({kernel, a, b});
        }
    }
};

// a grouped edge relation seen by a query-loop over v.edges:
// CSR index (V+1), head keys, longest group, source relation
struct EdgeGraph {
    uint64_t nv = 0, ne = 0;
    const uint32_t* index = nullptr;
    const uint32_t* head = nullptr;
    uint32_t max_group = 0;
    uint32_t max_chunk16 = 0, max_chunk64 = 0;   // rows of the largest 16- / 64-source chunk
    ebb_rel verts = EBB_NONE;
};
ebb_status edge_graph(Ctx* c, ebb_rel edges, EdgeGraph* g);   // solver.cu
// longest group, and most rows of any 16 / 64 consecutive groups of a CSR
// index with ns groups (synchronous; abi_core.cu)
ebb_status index_stats(Ctx* c, const uint32_t* index, uint64_t ns, uint32_t out[3]);

size_t dtype_size(ebb_dtype d);
ebb_status fail(Ctx* c, ebb_status code, const char* fmt, ...);
ebb_status cuda_fail(Ctx* c, cudaError_t e, const char* where);
Field* get_field(Ctx* c, ebb_field f);
Relation* get_rel(Ctx* c, ebb_rel r);
ebb_status scratch_reserve(Ctx* c, size_t bytes);
ebb_status new_internal_field(Ctx* c, ebb_rel rel, const std::string& name, ebb_dtype dt, uint32_t rows,
                              uint32_t cols, ebb_layout layout, ebb_field* out);
void release_plans(Ctx* c);
void comm_release(Ctx* c);
void peer_release(Ctx* c);   // solver.cu: frees the ebb_cg_peer_bind groups
// seg_map.cu: the SEGMENTED element map (builds its plan on first use)
ebb_status seg_map_launch(Ctx* c, ebb_field vf, ebb_field ef, int model, bool want_e, int accumulate, uint64_t nt,
                          const Field* V, const Field* U, const Field* D, const Field* W, const Field* MU,
                          const Field* LA, const Field* Fo, const Field* Ko, uint64_t ne, const Field* En,
                          cudaStream_t s);
// seg_plan.cu: the SEGMENTED plan built on the device (identical to the host
// builder's); tiles never cross a block of kSegBlock consecutive vertices
constexpr uint32_t kSegBlock = 2048;
ebb_status build_seg_plan_device(Ctx* c, const uint32_t* tv, uint64_t nt, const uint32_t* index, const uint32_t* head,
                                 uint64_t nv, int ni, SegPlan* P);
// chunk_map.cu: the CHUNK element map (builds its plan on the device on first use)
ebb_status build_chunk_plan(Ctx* c, ebb_field vf, ebb_field ef, int NT, ChunkPlan** out);
ebb_status chunk_map_launch(Ctx* c, ebb_field vf, ebb_field ef, int model, bool want_e, int accumulate, uint64_t nt,
                            const Field* V, const Field* U, const Field* D, const Field* W, const Field* MU,
                            const Field* LA, const Field* Fo, const Field* Ko, uint64_t ne, const Field* En,
                            cudaStream_t s, bool red);
// build the SEGMENTED / CHUNK plan for (v, e) if absent (EBB_E_RANGE: refused)
ebb_status seg_plan_probe(Ctx* c, ebb_field vf, ebb_field ef, ebb_dtype dt, int model);
ebb_status chunk_plan_probe(Ctx* c, ebb_field vf, ebb_field ef, ebb_dtype dt, int model);
// color_map.cu: the COLOURED element map (builds its colouring on first use)
ebb_status color_map_launch(Ctx* c, ebb_field vf, int model, bool want_e, uint64_t nt, const Field* V,
                            const Field* Ef, const Field* U, const Field* D, const Field* W, const Field* MU,
                            const Field* LA, const Field* Fo, const Field* Ko, uint64_t ne, const Field* En,
                            cudaStream_t s);
int color_plan_colors(Ctx* c, ebb_field vf);
ebb_status permute_relation(Ctx* c, ebb_rel rel, const uint32_t* d_new_to_old, const uint32_t* d_old_to_new,
                            cudaStream_t s);

#define EBB_CUDA(c, call)                                               \
    do {                                                                \
        cudaError_t _e = (call);                                        \
        if (_e != cudaSuccess) return ::ebb::cuda_fail((c), _e, #call); \
    } while (0)

// A context is bound to one CUDA device (include/ebb.h): every ABI entry
// point makes that device current for its duration and restores the
// caller's device on return (a process may hold contexts on several GPUs).
constexpr int kMaxDevices = 64;
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(const Ctx* c) {
        if (!c) return;
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != c->device && cudaSetDevice(c->device) == cudaSuccess)
            prev = cur;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};
// NVTX range around every C-ABI call (the runtime reports where time
// goes; SURVEY §5 tracing), named after the entry point: nvtxRangePushA is a
// null-pointer check unless a tool (nsys, ncu --nvtx) injects itself.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
#define EBB_DEVICE_GUARD(c)                          \
    ::ebb::NvtxRange _ebb_nvtx_range(__func__);      \
    ::ebb::DeviceGuard _ebb_device_guard(c)

#define EBB_TRY(call)                  \
    do {                               \
        ebb_status _s = (call);        \
        if (_s != EBB_OK) return _s;   \
    } while (0)

// Grid for a grid-stride kernel: exactly the number of CTAs that are resident
// at once (occupancy API x SM count), never more than the work needs.  A grid
// larger than one resident wave leaves a partial tail wave.
template <typename K>
inline unsigned occ_grid(const Ctx* c, K kernel, int block, size_t smem, uint64_t work_threads) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, block, smem) != cudaSuccess || nb < 1) {
        cudaGetLastError();
        nb = 1;
    }
    uint64_t full = (uint64_t)nb * (uint64_t)c->num_sms;
    uint64_t need = (work_threads + block - 1) / block;
    if (need == 0) need = 1;
    return (unsigned)(need < full ? need : full);
}

inline unsigned grid_for(uint64_t n, unsigned block) {
    uint64_t g = (n + block - 1) / block;
    return (unsigned)(g == 0 ? 1 : g);
}

// error word slots
enum { ERR_INVERTED = 0, ERR_NOT_SPD = 1, ERR_BOUNDS = 2, ERR_PEER = 3 };

}  // namespace ebb
