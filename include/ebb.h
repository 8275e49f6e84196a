/*
 * ebb.h -- C ABI of the B200-native Ebb tet-FEM hot path (libebb_b200.so).
 *
 * Paper: Bernstein et al., "Ebb: A DSL for Physical Simulation on CPUs and
 * GPUs", arXiv 1506.07577.  P:<n> = line n of the paper's PAPER.md, S:<n> =
 * line n of SPEC.md.  The calls follow the paper's relational model:
 * relations, fields in a column store, key-fields
 * (stored as uint64 in the paper P:854 -- here uint32,
 * which "Ebb is subsequently free to ... encode" P:674-677), GroupBy /
 * query-loops, field and global reductions.
 * The one hot path is the FEM element map over tets and the CG solve over the
 * edge relation; see DESIGN.md.
 *
 * Conventions for every call
 *   - Returns EBB_OK (0) or a negative ebb_status; never throws.  The text of
 *     the last error of a context is in ebb_last_error(ctx) (valid until the
 *     next call on that context).
 *   - A context is bound to one CUDA device and is single-entrant:
 *     no two calls on the same context may run concurrently.
 *   - ebb_stream is a cudaStream_t (NULL = the legacy default stream).  Kernel
 *     launching calls are asynchronous and stream-ordered; calls documented as
 *     "synchronous" block the host until the stream is idle.
 *   - Handles (ebb_rel, ebb_field) are small integers owned by the context and
 *     valid until ebb_ctx_free.  EBB_NONE marks an absent optional field.
 *   - Keys are opaque row references.  They cross the ABI as
 *     uint64 and are bounds-checked on entry.
 *   - Device memory of library-allocated fields is owned by the context;
 *     ebb_field_wrap borrows caller memory that must outlive the context.
 *   - Kernel-side failures (inverted elements, non-SPD CG, key out of range)
 *     increment a device error word read by ebb_error_counts (synchronous).
 */
#ifndef EBB_H
#define EBB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t ebb_status;
#define EBB_OK 0
#define EBB_E_ARG (-1)          /* bad handle, NULL pointer, bad enum        */
#define EBB_E_DUP (-2)          /* duplicate relation/field name      */
#define EBB_E_SIZE (-3)         /* zero size / byte count mismatch */
#define EBB_E_BOUNDS (-4)       /* key out of range of its target     */
#define EBB_E_TYPE (-5)         /* dtype/shape/relation mismatch  */
#define EBB_E_STATE (-6)        /* double grouping, missing prerequisite      */
#define EBB_E_PHASE (-7)        /* a field in two phases of one map  */
#define EBB_E_INVERTED (-8)     /* tet with W <= 0 at rest                   */
#define EBB_E_NOT_SPD (-9)      /* CG found p.q <= 0                          */
#define EBB_E_CUDA (-10)        /* CUDA runtime failure                       */
#define EBB_E_RANGE (-11)       /* value does not fit the 32-bit key storage  */
#define EBB_E_NOMEM (-12)       /* device allocation failed                   */
#define EBB_E_DEGENERATE (-13)  /* |det Dm| <= 1e-12 l^3 (O1)                  */
#define EBB_E_NCCL (-14)        /* NCCL missing or failed                      */

typedef struct ebb_ctx_s* ebb_ctx;
typedef uint32_t ebb_rel;
typedef uint32_t ebb_field;
typedef void* ebb_stream; /* cudaStream_t */
#define EBB_NONE 0xFFFFFFFFu

typedef enum {
    EBB_F32 = 1, EBB_F64 = 2, EBB_I32 = 3, EBB_I64 = 4, EBB_U8 = 5, EBB_U32 = 6,
    EBB_KEY = 7 /* key-field: uint32 storage, typed by its target relation */
} ebb_dtype;

/* Storage layout of a rows x cols field.  AOS: element-major (the 9 entries
 * of a 3x3 block are contiguous).  SOA: component-planar -- one contiguous
 * column per component, the paper's column store applied per
 * component; used for tet rest data and the edge stiffness so that a warp's
 * loads coalesce.  Host-side data crossing the ABI is always element-major. */
typedef enum { EBB_AOS = 0, EBB_SOA = 1 } ebb_layout;

typedef struct {
    void* data;               /* device pointer                               */
    uint64_t count;           /* rows of the owning relation                  */
    uint32_t rows, cols;      /* per-element shape (vec3 = 3x1, mat3 = 3x3)   */
    int32_t dtype;            /* ebb_dtype                                    */
    int32_t layout;           /* ebb_layout                                   */
    uint64_t elem_stride;     /* bytes between consecutive elements           */
    uint64_t comp_stride;     /* bytes between consecutive components         */
    ebb_rel rel;              /* owning relation                              */
    ebb_rel key_target;       /* target relation of a key-field, else NONE    */
} ebb_view;

const char* ebb_version(void);

/* ---- context -------------------------------------------------------- */
ebb_status ebb_ctx_new(int device, ebb_ctx* out);
ebb_status ebb_ctx_free(ebb_ctx ctx);
const char* ebb_last_error(ebb_ctx ctx);
/* Kernel-side error counters (synchronous; optionally reset) -- the device
 * error word of SURVEY §8(b) "Errors" (EBB_E_INVERTED, EBB_E_NOT_SPD,
 * EBB_E_BOUNDS classes): out[0] inverted elements (J<=0, the NH reading of
 * DESIGN.md §3 (15)), out[1] CG p.q<=0 events, out[2] key out of range
 * (S:87), out[3] peer waits abandoned by the fused multi-GPU PCG
 * (ebb_cg_peer_step).  EBB_E_ARG on a bad context. */
ebb_status ebb_error_counts(ebb_ctx ctx, uint64_t out[4], int reset);
/* Wait for every call issued on stream s (NULL: the whole device); the
 * synchronising point of SURVEY §8(b) "Asynchrony".  EBB_E_CUDA on a
 * failed kernel. */
ebb_status ebb_sync(ebb_ctx ctx, ebb_stream s);
/* Instrumentation ("we instrument Ebb directly").  When enabled,
 * every launch of a hot kernel is bracketed by CUDA events recorded on the
 * launching stream.  kernel ids: EBB_K_TET_MAP, EBB_K_EDGE_MATVEC,
 * EBB_K_CG_UPDATE, EBB_K_CG_DIR, EBB_K_ASSEMBLE.  timing_read is synchronous
 * and returns the summed device time (ms) and the number of timed launches. */
#define EBB_K_TET_MAP 0
#define EBB_K_EDGE_MATVEC 1
#define EBB_K_CG_UPDATE 2
#define EBB_K_CG_DIR 3
#define EBB_K_ASSEMBLE 4
#define EBB_K_CG_SOLVE 5   /* persistent single-launch PCG (all iterations) */
#define EBB_K_SPRING 6     /* Fig. 2 spring forces / fused spring step         */
#define EBB_K_EBE_MATVEC 7 /* matrix-free element-by-element matvec            */
#define EBB_K_GRID 8       /* regular-grid stencil / particle interpolation    */
ebb_status ebb_timing_enable(ebb_ctx ctx, int on);
ebb_status ebb_timing_read(ebb_ctx ctx, int32_t kernel, double* total_ms, uint64_t* launches, int reset);
/* Number of kernels this context has launched (all entry points). */
ebb_status ebb_launch_count(ebb_ctx ctx, uint64_t* out, int reset);

/* CUDA-graph capture of a sequence of stream-ordered calls (e.g. one implicit
 * step: map, assemble, cg_init, cg_step, implicit_update; SURVEY §8(e) "the
 * whole iteration captured in a CUDA graph").  s must be a
 * non-default stream; calls between begin and end must not allocate or
 * synchronise (run the sequence once eagerly first: first calls build plans
 * and work fields).  Kernel timers recorded during capture become graph
 * event nodes: after a launch + ebb_sync, ebb_timing_read(.., reset=0)
 * returns that replay's per-kernel times.  Launch counts of a replay are the
 * captured ones. */
ebb_status ebb_graph_begin(ebb_ctx ctx, ebb_stream s);
ebb_status ebb_graph_end(ebb_ctx ctx, ebb_stream s, int32_t* graph_out);
ebb_status ebb_graph_launch(ebb_ctx ctx, int32_t graph, ebb_stream s);
ebb_status ebb_graph_free(ebb_ctx ctx, int32_t graph);

/* ---- relations and fields ----------- */
ebb_status ebb_relation_new(ebb_ctx ctx, const char* name, uint64_t size, ebb_rel* out);
ebb_status ebb_relation_size(ebb_ctx ctx, ebb_rel rel, uint64_t* out);
/* Library-allocated field; host_init (element-major, rows*cols per element)
 * or NULL for zeros.  Shapes: rows, cols <= 4, or a column of up to 32 rows
 * (per-element state records); EBB_E_SIZE otherwise.  Synchronous. */
ebb_status ebb_field_new(ebb_ctx ctx, ebb_rel rel, const char* name, ebb_dtype dtype,
                         uint32_t rows, uint32_t cols, ebb_layout layout,
                         const void* host_init, ebb_field* out);
/* Borrowed device memory (e.g. a torch tensor's data_ptr) in the given layout. */
ebb_status ebb_field_wrap(ebb_ctx ctx, ebb_rel rel, const char* name, ebb_dtype dtype,
                          uint32_t rows, uint32_t cols, ebb_layout layout,
                          void* device_ptr, ebb_field* out);
ebb_status ebb_field_find(ebb_ctx ctx, ebb_rel rel, const char* name, ebb_field* out);
/* Host <-> device copies of the whole column, element-major host order.
 * nbytes must equal count*rows*cols*sizeof(dtype).  write is stream-ordered
 * (host buffer must stay valid until the stream reaches it; pinned memory
 * makes it asynchronous); read is synchronous. */
ebb_status ebb_field_write(ebb_ctx ctx, ebb_field f, const void* host, uint64_t nbytes, ebb_stream s);
ebb_status ebb_field_read(ebb_ctx ctx, ebb_field f, void* host, uint64_t nbytes, ebb_stream s);
/* Stream-ordered read of an element-major (AOS or scalar) field: the host
 * buffer (pinned for a truly asynchronous copy) is complete once the stream
 * reaches this point (an event / ebb_sync).  EBB_E_TYPE for component-planar
 * fields.  (The pipelined end-to-end step of SURVEY §8(d): the read of step k
 * overlaps step k+1.) */
ebb_status ebb_field_read_async(ebb_ctx ctx, ebb_field f, void* host, uint64_t nbytes, ebb_stream s);
ebb_status ebb_field_fill(ebb_ctx ctx, ebb_field f, double value, ebb_stream s);
ebb_status ebb_field_copy(ebb_ctx ctx, ebb_field dst, ebb_field src, ebb_stream s);
/* dst = (dtype of dst) src for F32/F64 fields of equal relation, shape, layout. */
ebb_status ebb_field_convert(ebb_ctx ctx, ebb_field dst, ebb_field src, ebb_stream s);
/* Zero-copy raw view; invalidated by group_by/renumber. */
ebb_status ebb_field_view(ebb_ctx ctx, ebb_field f, ebb_view* out);

/* Key-field: rows x cols keys per element of `owner`, each a row
 * of `target`.  keys are uint64 (host, or device if keys_on_device);
 * EBB_E_BOUNDS if any key >= size(target); EBB_E_RANGE if a target is
 * larger than 2^32-1 rows.  Synchronous. */
ebb_status ebb_key_field(ebb_ctx ctx, ebb_rel owner, const char* name, ebb_rel target,
                         uint32_t rows, uint32_t cols, const uint64_t* keys, int keys_on_device,
                         ebb_field* out);

/* ---- globals ----------------------- */
ebb_status ebb_global_new(ebb_ctx ctx, const char* name, ebb_dtype dtype, double init, ebb_field* out);
ebb_status ebb_global_get(ebb_ctx ctx, ebb_field g, double* out);   /* synchronous */
ebb_status ebb_global_set(ebb_ctx ctx, ebb_field g, double value, ebb_stream s);

/* ---- GroupBy ------------------------- */
/* Stably sorts `rel` by the scalar key-field `key`, permutes every field of
 * rel, remaps every key-field in the context that targets rel, and builds the
 * hidden index on the source relation: a U32 field "__index" of size+1 rows
 * (CSR offsets; row s owns [index[s], index[s+1])).  EBB_E_STATE if rel is
 * already grouped; EBB_E_TYPE if key is not a scalar key-field of rel.
 * Synchronous. */
ebb_status ebb_group_by(ebb_ctx ctx, ebb_rel rel, ebb_field key);
ebb_status ebb_group_index(ebb_ctx ctx, ebb_rel rel, ebb_field* index_out);

/* ---- locality renumbering (licence P:674-677) -------- */
/* Morton order of the quantised rows of `pos` (vec3 F64 on rel): q_d =
 * min(2^21-1, floor((x_d-lo_d)/(hi_d-lo_d) 2^21)), x bit at 3b, y at 3b+1,
 * z at 3b+2; stable by old id.  Permutes rel's fields, remaps inbound keys.
 * Synchronous. */
ebb_status ebb_renumber_morton(ebb_ctx ctx, ebb_rel rel, ebb_field pos);
/* Sort `rel` lexicographically by the ascending-sorted tuple of its rows x 1
 * key-field `keys` (1..4 keys per row: tets by their vertex ids, particles by
 * their dual cell), stable.  Permutes rel's fields, remaps inbound keys.
 * Synchronous. */
ebb_status ebb_sort_by_key_tuple(ebb_ctx ctx, ebb_rel rel, ebb_field keys);

/* ---- tetrahedral mesh domain --------- */
typedef struct {
    ebb_rel edges;   /* relation of ordered vertex pairs + one self-loop per vertex */
    ebb_field tail;  /* edges -> verts key, grouped (edges sorted by (tail, head)) */
    ebb_field head;  /* edges -> verts key                                         */
    ebb_field e;     /* tets 4x4 key -> edges; tail(e[i][j]) = v[i], head = v[j]   */
    ebb_field self;  /* verts -> edges key of the self-loop (diagonal block)       */
    ebb_field index; /* verts U32 (V+1) CSR offsets of the grouping                */
} ebb_tetmesh;
/* O1: swap v[2], v[3] of tets with det(Dm) < 0 (pos: verts vec3 F64).
 * EBB_E_DEGENERATE if |det| <= 1e-12 l^3.  Synchronous. */
ebb_status ebb_tetmesh_orient(ebb_ctx ctx, ebb_field tets_v, ebb_field pos, uint64_t* n_swapped);
/* a1: build the edge relation named edges_name from tets.v (4x1 keys) and
 * group it by tail.  Synchronous. */
ebb_status ebb_tetmesh_build(ebb_ctx ctx, ebb_field tets_v, const char* edges_name, ebb_tetmesh* out);
/* a3: Dminv (tets 3x3, rows g_1..g_3), W = det(Dm)/6 (tets 1x1), lumped mass
 * m_v = sum rho W / 4 (verts 1x1), all F64.  EBB_E_INVERTED if some W <= 0. */
ebb_status ebb_tetmesh_rest(ebb_ctx ctx, ebb_field tets_v, ebb_field pos, double rho,
                            ebb_field Dminv, ebb_field W, ebb_field mass, ebb_stream s);

/* Consistent (Galerkin) mass of linear tets on the edge relation (SURVEY
 * §8(c) "Mass matrix" reading: consistent mass on edges is the NEXT option
 * beside the lumped one; §8(f) 1; the paper names only a "mass" field,
 * P:354-355): M_ij = rho W (1 + d_ij)/20 I_3, i.e.
 * mass_e[e[i][j]] += rho W (1 + d_ij)/20 over every tet and (i, j).
 * tets_e: the 4x4 key-field tets.e; W: F64 scalar on tets (ebb_tetmesh_rest);
 * mass_e: F64 scalar on the edge relation (written; zeroed first).  Row sums
 * equal the lumped mass.  fp64 atomic accumulation (like the lumped mass):
 * equal to the oracle within round-off, not bitwise run-to-run.
 * Stream-ordered. */
ebb_status ebb_tetmesh_consistent_mass(ebb_ctx ctx, ebb_field tets_e, ebb_field W, double rho,
                                       ebb_field mass_e, ebb_stream s);

/* ---- the element map (hot path a4-a8) --------------------------------- */
#define EBB_STVK 0
#define EBB_NH 1
#define EBB_SCATTER_AUTO 0      /* the measured fastest: SEGMENTED (f + K);
                                   force-only maps use ATOMIC.
                                   A mesh whose SEGMENTED plan is refused
                                   (EBB_E_RANGE: a vertex in more tets than a
                                   tile holds) runs CHUNK, else ATOMIC; the
                                   choice is made once per (v, e).           */
#define EBB_SCATTER_ATOMIC 1    /* per-tet red.global.add              */
#define EBB_SCATTER_TILED 2     /* retired in round 2 (owner tiles with
                                   shared-memory atomics; measured slower than
                                   SEGMENTED at every size): EBB_E_ARG        */
#define EBB_SCATTER_GATHER 3    /* retired in round 2 (warp-specialized owner
                                   tiles; measured slower): EBB_E_ARG         */
#define EBB_SCATTER_SEGMENTED 4 /* single-pass owner tiles (device-built plan):
                                   every thread computes one instance's
                                   compact element state, then every owned
                                   edge row sums its blocks rebuilt from the
                                   states (segmented reduction over the
                                   row's incident (tet, i, j), in
                                   place of the `+=` of P:885; no atomics,
                                   bitwise run-to-run deterministic).  The
                                   plan is built on the device at the first
                                   call for a (v, e) pair (synchronous; freed by
                                   any relation permutation or ctx_free).
                                   EBB_E_RANGE if one vertex lies in more tets
                                   than the per-tile instance cap (256; 384
                                   for StVK fp64; EBB_SEG_NT overrides).       */
#define EBB_SCATTER_COLOR 5     /* tets greedily coloured (no two tets of a
                                   colour share a vertex), one launch per
                                   colour, plain read-modify-write reductions
                                   (deterministic; EBB_E_RANGE beyond 64
                                   colours).                                  */
#define EBB_SCATTER_CHUNK 6     /* non-redundant tet chunks (device-built plan):
                                   tiles of NT consecutive (SFC-ordered) tets,
                                   each tet's element state computed ONCE;
                                   every canonical row is summed by the last
                                   tile touching it from its own blocks plus
                                   the partial sums earlier tiles leave in
                                   L2 message slots (release/acquire tile
                                   counters; no atomics on f or K; bitwise
                                   run-to-run deterministic).  The plan is
                                   built on the device at the first call for
                                   a (v, e) pair (synchronous; freed by any
                                   relation permutation or ctx_free).
                                   EBB_E_RANGE if one row gets blocks from
                                   more than 128 tiles or more than 248
                                   blocks from one tile.                     */
#define EBB_SCATTER_CHUNK_RED 7 /* SURVEY §8(a) "+=" strategy (i): the CHUNK
                                   tiles (each tet once, rows summed on chip
                                   per tile), rows only one tile feeds stored
                                   once, rows several tiles feed zeroed first
                                   and then added to with red.global.add
                                    -- no messages, no waits between
                                   tiles; not bitwise run-to-run
                                   deterministic (RED order).               */
typedef struct {
    int32_t model;         /* EBB_STVK | EBB_NH                                */
    int32_t scatter;       /* EBB_SCATTER_*                                    */
    int32_t zero_outputs;  /* 1: f, K, energy are zeroed first                 */
    int32_t reserved;
    ebb_field v;           /* tets.v   4x1 key -> verts      (read)            */
    ebb_field e;           /* tets.e   4x4 key -> edges      (read; iff K)     */
    ebb_field u;           /* verts    vec3 displacement     (read)            */
    ebb_field Dminv;       /* tets     3x3 (rows g_1..g_3)   (read)            */
    ebb_field W;           /* tets     rest volume           (read)            */
    ebb_field mu, lam;     /* tets     Lame parameters       (read)     */
    ebb_field f;           /* verts    vec3 force            (reduce +)        */
    ebb_field K;           /* edges    3x3 stiffness         (reduce +) / NONE */
    ebb_field energy;      /* global   strain energy sum WΨ  (reduce +) / NONE */
} ebb_tet_map_desc;
/* For each tet: H = Du Dminv, F = I + H; StVK or
 * compressible neo-Hookean first Piola stress P; f_i = -W P g_i, f_0 =
 * -sum f_i; K_ij = d^2(WΨ)/dx_i dx_j (closed rank-1 forms);
 * f[v[i]] += f_i, K[e[i][j]] += K_ij, energy += WΨ.  All float fields share
 * one dtype (F32 or F64) and the documented layouts: u, f AOS; Dminv, K SOA.
 * EBB_E_PHASE if u aliases f or K, or f aliases K. */
ebb_status ebb_map_tet_forces(ebb_ctx ctx, const ebb_tet_map_desc* d, ebb_stream s);
/* Statistics of the SEGMENTED map plan built for (v, e) (0 if none yet):
 * out = {tiles, instances, instances / tets (redundancy), entries, items,
 *        instance cap per tile, plan build ms (on the device; on the host
 *        with EBB_SEG_PLAN=host), largest tile's entries}.
 * Host-only; no device work. */
ebb_status ebb_map_plan_stats(ebb_ctx ctx, ebb_field v, ebb_field e, double out[8]);
/* Statistics of the CHUNK map plan built for (v, e) (0 if none yet; the
 * most recent plan if several tile sizes were built):
 * out = {tiles, tets per tile, segments, messages (partial row sums sent to
 *        a later tile), items, device build ms, plan bytes per tet resident
 *        on the device (entries, items, descriptors, message slots, lists),
 *        rows no tet contributes to}.  Host-only; no device work. */
ebb_status ebb_map_chunk_stats(ebb_ctx ctx, ebb_field v, ebb_field e, double out[8]);

/* a10: q_v = sum_{e in [index[v], index[v+1])} A_e p_head(e)  (query-loop over
 * v.edges), q *= mask (optional U8 on verts), and optionally
 * pq_global = p.q (fused, deterministic two-pass).  `edges` must be
 * grouped by a key into verts and carry a scalar key-field named "head"
 * (the e.head of the query-loop); A is SOA 3x3, p and q AOS vec3, one dtype. */
ebb_status ebb_map_edge_matvec(ebb_ctx ctx, ebb_rel edges, ebb_field A, ebb_field p, ebb_field q,
                               ebb_field mask, ebb_field pq_global, ebb_stream s);

/* a8: global reductions over every component of `a`:
 * SUM a, DOT a.b, MAX a, MIN a, optionally masked per element by a U8 field
 * (masked-out elements contribute the identity). out is an F64 global. */
#define EBB_RED_SUM 0
#define EBB_RED_DOT 1
#define EBB_RED_MAX 2
#define EBB_RED_MIN 3
ebb_status ebb_global_reduce(ebb_ctx ctx, int32_t op, ebb_field a, ebb_field b, ebb_field mask,
                             ebb_field out, ebb_stream s);

/* ---- integrators (Fig. 2) ---------------------- */
typedef struct {
    ebb_rel edges;
    ebb_field K;      /* edges 3x3 stiffness (read)                          */
    ebb_field A;      /* edges 3x3 system matrix (write; may equal K)        */
    ebb_field self;   /* verts -> edges self-loop key                        */
    ebb_field mass;   /* verts (lumped) or edges (consistent) scalar (read)  */
    ebb_field f, vel; /* verts (read)                                        */
    ebb_field b;      /* verts vec3 rhs (write)                              */
    double h, alpha, beta;    /* step, Rayleigh damping D = alpha M + beta K */
    double g[3];              /* gravity                                     */
    int32_t rhs_form;         /* EBB_RHS_LINEARISED (0): b = h (f + M g - D v
                                 - h K v), v = vel, the one-linearisation step
                                 (O9).  EBB_RHS_NEWTON (1): a later Newton
                                 iteration of the same backward-Euler step,
                                 vel = the velocity iterate w (u = u_n + h w),
                                 vel0 = v_n: b = h (f + M g - D w) + M (v_n - w);
                                 A is the same.  SURVEY §8(f) 1.             */
    ebb_field vel0;           /* verts vec3 v_n (EBB_RHS_NEWTON only)          */
} ebb_implicit_desc;
#define EBB_RHS_LINEARISED 0
#define EBB_RHS_NEWTON 1
/* a9: A = M + h D + h^2 K, b = h (f + M g - D v - h K v).  `mass` is either
 * a scalar field on verts (lumped M = diag(m_v) I_3) or a scalar field on
 * the edge relation (consistent M_r = mass_e[r] I_3 per edge row, from
 * ebb_tetmesh_consistent_mass; M v and M g are then edge query-loops),
 * in the map dtype. */
ebb_status ebb_implicit_assemble(ebb_ctx ctx, const ebb_implicit_desc* d, ebb_stream s);

typedef struct {
    ebb_rel edges;
    ebb_field A, b, x;   /* system (read, library-allocated), rhs, solution   */
    ebb_field self;      /* verts -> edges self-loop key (Jacobi diagonal)    */
    ebb_field mask;      /* verts U8, 1 = free, or EBB_NONE (a12)  */
    /* work fields: EBB_NONE = allocated by ebb_cg_init and written back; a
     * supplied work field must be an AOS 4x1 field on verts (vec3 padded to
     * one 32-byte / 16-byte record so that a vertex is a single access)     */
    ebb_field r, p, z, q, dinv;
    ebb_field rho;       /* F64 global r.z (allocated if NONE)                */
    ebb_field scal;      /* internal device scalars rho, p.q, r.z             */
    ebb_field p2;        /* second direction buffer (p is double-buffered)    */
    int32_t variant;     /* EBB_CG_AUTO | EBB_CG_SAAD | EBB_CG_SINGLE_REDUCTION;
                            fixed from ebb_cg_init to the end of the solve    */
    ebb_field s, y, w, u, u2;     /* single-reduction work vectors: s = A p,
                            y = A D s, w = A z, u = D w (double-buffered with
                            u2; D = diag(A)^-1); EBB_NONE = allocated          */
    double tol;          /* 0 = exactly `iters` iterations (the parity mode,
                            SURVEY O10).  > 0: ebb_cg_step stops, on the
                            device, after the first iteration k with
                            r_k.z_k <= tol^2 r_0.z_0 (Jacobi-preconditioned
                            residual relative to the start; SURVEY §8(f) 1
                            "tolerance-based PCG"); every later ebb_cg_step
                            is a no-op until ebb_cg_init.  The iterations run
                            are read by ebb_cg_iterations.  ebb_cg_phase
                            ignores tol (the multi-GPU driver decides).     */
} ebb_cg;
#define EBB_CG_AUTO 0              /* the measured faster          */
#define EBB_CG_SAAD 1              /* Saad Alg. 9.1: two reductions per iteration    */
#define EBB_CG_SYMMETRIC 3         /* Saad Alg. 9.1 with the matvec over the upper
                                      triangle only (A = A^T: half of A
                                      streamed per iteration); the transposed
                                      blocks reach their rows by red.global.add
                                      (P:885), so iterates agree to round-off but
                                      are not bitwise run-to-run reproducible    */
#define EBB_CG_SINGLE_REDUCTION 2  /* Chronopoulos-Gear with the matvec moved onto
                                      u = D w: one fused reduction (r.z, w.z) and
                                      one gathered vector per iteration, same
                                      iterates in exact arithmetic; ebb_cg_step
                                      only (the per-phase multi-GPU path is Saad) */
/* a11: x = 0, r = b*mask, z = r/diag(A), p = z, rho = r.z.  Stream-ordered.
 * Per iteration: beta = rho'/rho, p = z + beta p fused into q = (A p)*mask
 * with p.q; then alpha = rho/p.q, x += alpha p, r -= alpha q, z = r/diag(A),
 * rho' = r.z.  ebb_cg_step runs all `iters` iterations in ONE persistent
 * cooperative kernel (grid barriers between the phases, deterministic dots);
 * ebb_cg_phase launches the phases separately (multi-GPU). No host sync. */
ebb_status ebb_cg_init(ebb_ctx ctx, ebb_cg* cg, ebb_stream s);
/* Iterations run since ebb_cg_init and whether the tolerance was met
 * (converged = 1).  Synchronises the stream `s` (reads two device scalars);
 * either output may be NULL. */
ebb_status ebb_cg_iterations(ebb_ctx ctx, const ebb_cg* cg, ebb_stream s, int32_t* iters, int32_t* converged);
/* The variant ebb_cg_step runs for this system (AUTO resolved). Host-only. */
ebb_status ebb_cg_variant(ebb_ctx ctx, const ebb_cg* cg, int32_t* out);
/* a10-a12: `iters` Jacobi-PCG iterations (Saad Alg. 9.1), alpha/beta kept
 * on the device (no host sync); p.q <= 0 counts in error word [1]. */
ebb_status ebb_cg_step(ebb_ctx ctx, const ebb_cg* cg, int32_t iters, ebb_stream s);
/* One phase of an iteration, for callers that interleave communication
 * (multi-GPU: allreduce the scal slot after MATVEC (p.q, slot 1) and after
 * UPDATE (r.z, slot 2), and refresh ghost rows of z after UPDATE and after
 * ebb_cg_init).  ebb_cg_step(n) == n x (DIR, MATVEC, UPDATE); DIR is a no-op
 * kept for callers -- the direction update is fused into MATVEC. */
#define EBB_CG_DIR 0
#define EBB_CG_MATVEC 1
#define EBB_CG_UPDATE 2
/* Single-reduction PCG in phase mode ("one fused 2-scalar
 * allreduce if a single-reduction CG variant is adopted"): each call runs one
 * phase of the Chronopoulos-Gear recurrences (the first call after
 * ebb_cg_init forms w_0 = A z_0) and leaves the rank-local w.z and r.z in
 * scal slots 10 and 11; the caller allreduces those two slots and refreshes
 * the ghost rows of both u buffers (ebb_cg.u, ebb_cg.u2) -- and of z before
 * the first call -- then calls again: iters iterations = iters + 1 calls.
 * Needs ebb_cg_init with EBB_CG_SINGLE_REDUCTION.  The tolerance (ebb_cg.tol)
 * is honoured once the initial r.z (slots 0-2 and 7) has been summed. */
#define EBB_CG_SR_PHASE 3
ebb_status ebb_cg_phase(ebb_ctx ctx, const ebb_cg* cg, int32_t phase, ebb_stream s);

/* ---- halo support ------------------------------------- */
/* pack:   buf[k] = f[rows[k]]      unpack: f[rows[k]] = buf[k]
 * f: AOS field of any dtype, or a component-planar (SOA) F32/F64 field;
 * rows: U32 field (row ids of f's relation) on a list relation; buf: AOS
 * field of f's dtype and shape on the list relation. */
ebb_status ebb_rows_gather(ebb_ctx ctx, ebb_field f, ebb_field rows, ebb_field buf, ebb_stream s);
ebb_status ebb_rows_scatter(ebb_ctx ctx, ebb_field f, ebb_field rows, ebb_field buf, ebb_stream s);
/* f[rows[k]] += buf[k] (F32/F64; f AOS or SOA, buf AOS): the reverse add of
 * partial force / stiffness rows into their owners (SURVEY §8(e) "halo
 * exchange ... of the partial force sums").  rows must be distinct within
 * one call; calls are stream-ordered, so several peers' lists may overlap. */
ebb_status ebb_rows_scatter_add(ebb_ctx ctx, ebb_field f, ebb_field rows, ebb_field buf, ebb_stream s);

/* ---- NCCL inside the library ("NCCL over NVLink carries the
 * halo exchange ... and the allreduce of CG scalars"; not in the paper,
 * P:1014).  libnccl.so.2 is opened at run time (the copy the process already
 * uses).  One communicator per context (one process per GPU); every call is
 * stream-ordered, nothing synchronises the host.  EBB_E_NCCL if NCCL is
 * missing or fails, EBB_E_STATE before ebb_comm_init. */
typedef struct { char internal[128]; } ebb_nccl_id;
/* rank 0 creates the id and shares it out of band (e.g. torch.distributed). */
ebb_status ebb_comm_unique_id(ebb_nccl_id* out);
ebb_status ebb_comm_init(ebb_ctx ctx, int32_t nranks, int32_t rank, const ebb_nccl_id* id);
/* in-place sum over ranks of `count` F64 values in device memory (the PCG
 * scalar slots of ebb_cg.scal: p.q, r.z). */
ebb_status ebb_comm_allreduce_sum(ebb_ctx ctx, double* dev_buf, uint64_t count, ebb_stream s);
/* grouped exchange with `npeers` ranks: send_bufs[k] (send_bytes[k]) to
 * peers[k], recv_bufs[k] (recv_bytes[k]) from peers[k]; device buffers, as
 * packed by ebb_rows_gather and unpacked by ebb_rows_scatter. */
ebb_status ebb_comm_halo(ebb_ctx ctx, int32_t npeers, const int32_t* peers, void* const* send_bufs,
                         const uint64_t* send_bytes, void* const* recv_bufs, const uint64_t* recv_bytes,
                         ebb_stream s);

/* ---- fused multi-GPU PCG over peer memory ("the halo
 * exchange of vertex positions ... and the allreduce of CG scalars", here
 * without NCCL on the iteration path; the paper is single-device).
 * The PCG of every rank runs as ONE persistent kernel for all iterations,
 * with one of two bodies (ebb_cg.variant at the bind): single-reduction
 * (EBB_CG_SINGLE_REDUCTION, Chronopoulos-Gear; one exchange of the fused
 * (w.z, r.z) per iteration, halo of the gathered operand u and of x) or
 * Saad (EBB_CG_SAAD; exchanges of p.q and r.z, halo of z and x).  Each owner
 * stores the halo rows that peers hold as ghosts straight into the peers'
 * buffers as it finishes them (P2P stores over NVLink; for ranks emulated
 * on one device, plain stores), and the scalars go through per-rank
 * mailboxes (release/acquire at system scope), summed in rank order on
 * every rank (bitwise the same alpha, beta everywhere).  The z_0 halo and
 * the initial r.z sum are done in the same launch; the x halo lands before
 * the kernel ends, so ebb_implicit_update can follow directly.
 * Decomposition: EBB_PART_OVERLAP (ebb_partition_local): local vertices
 * [0, n_owned) are owned, the rest ghosts; rows of ghosts are not solved.
 * A wait that exceeds ~20 s (a peer that never arrives) counts in error word
 * [3] and is abandoned (results then invalid) instead of hanging the GPU. */
#define EBB_MAX_RANKS 16
#define EBB_PEER_MBOX_WORDS 160   /* F64 rows of a mailbox field (see below)  */
typedef struct {
    int32_t nranks, rank;     /* P <= EBB_MAX_RANKS, 0 <= rank < P            */
    uint64_t n_owned;         /* local verts [0, n_owned) are owned            */
    ebb_field send_off;       /* from ebb_peer_send_csr: U32 CSR offsets (n_owned + 1)  */
    ebb_field send_dst;       /* U32 2x1 (peer rank, row in the peer's local numbering) */
    ebb_field mbox;           /* this rank's mailbox: F64 field of >= EBB_PEER_MBOX_WORDS
                                 rows, all zero before the first step (ebb_field_fill 0) */
    /* device addresses, valid on THIS rank's device, of rank q's cg.u, cg.u2,
     * cg.x, cg.z and mailbox (IPC-mapped with ebb_ipc_open on multi-GPU, the
     * fields' own addresses for ranks emulated on one device); [rank] unused */
    uint64_t peer_u[EBB_MAX_RANKS], peer_u2[EBB_MAX_RANKS], peer_x[EBB_MAX_RANKS],
             peer_z[EBB_MAX_RANKS], peer_mbox[EBB_MAX_RANKS];
} ebb_peer_cg;
/* Mailbox layout (u64 words): [slot 0..1][sender rank 0..15][4] = (d, g,
 * sequence, unused), then word 128 = this rank's exchange count (epoch).
 * Exchange k of a rank writes slot k & 1 of every peer's mailbox and
 * releases its sequence word with k + 1. */
/* Per-source-row send lists for the fused PCG and the peer halos, built on
 * the device: for each peer k (npeers of them, ranks peers[k]) send_rows[k]
 * (U32 local rows, all < n_src -- the source rows: owned vertices for the
 * PCG and COPY halos, every row of the relation for an ADD halo --, e.g.
 * ebb_partition_local's send rows of that peer) and
 * remote_rows[k] (U32, the same length: the row of each of them in the
 * peer's local numbering, i.e. the peer's recv rows from this rank, which
 * list the same vertices in the same order), each < peer_nv[k].  Creates
 * relations <name>.off (n_src + 1 rows, U32 "off") and <name>.dst (one row
 * per entry, U32 2x1 "dst" = (peer, remote row)), entries of a vertex in
 * peers[] order.  EBB_E_RANGE on a row out of bounds.  Synchronous.
 * (SURVEY §8(e) halo lists; P:1014 for the paper's single device) */
ebb_status ebb_peer_send_csr(ebb_ctx ctx, uint64_t n_src, int32_t npeers, const int32_t* peers,
                             const ebb_field* send_rows, const ebb_field* remote_rows, const uint64_t* peer_nv,
                             const char* name, ebb_field* send_off, ebb_field* send_dst);
/* CUDA IPC of a library-allocated field (one process per GPU): the 64-byte
 * handle of the field's allocation; open maps a peer's handle into this
 * context's device (peer access enabled) and returns its device address;
 * close unmaps it.  EBB_E_TYPE for borrowed (wrapped) fields.  (SURVEY §8(e):
 * one process per GPU over NVLink) */
ebb_status ebb_ipc_handle(ebb_ctx ctx, ebb_field f, void* handle64);
ebb_status ebb_ipc_open(ebb_ctx ctx, const void* handle64, uint64_t* dev_addr);
ebb_status ebb_ipc_close(ebb_ctx ctx, uint64_t dev_addr);
/* Bind `nlocal` ranks whose systems live on this context's device (1 per
 * process on a multi-GPU node; P for ranks emulated on one device) into a
 * launch group: cgs[i] (after ebb_cg_init with EBB_CG_SAAD or
 * EBB_CG_SINGLE_REDUCTION, the same on every rank; its fields must outlive
 * the group; the single-reduction body also reads peer_u / peer_u2) and
 * peers[i].  Validates and uploads the
 * per-rank launch records once (synchronous, not capturable); *group_out is
 * the group id.  ebb_cg.tol is taken here.  EBB_E_SIZE if the ranks' CTAs
 * cannot all be resident or a rank's TMA ring (sized by its largest
 * 16-vertex chunk of edge rows) does not fit in shared memory -- hub meshes
 * then use the per-phase driver (ebb_cg_phase), which has unstaged paths.
 * (the PCG of P:946, Jacobi-preconditioned) */
ebb_status ebb_cg_peer_bind(ebb_ctx ctx, int32_t nlocal, const ebb_cg* cgs, const ebb_peer_cg* peers,
                            int32_t* group_out);
/* `iters` PCG iterations (the bound body) of every rank of the group in one
 * cooperative launch (the first call after ebb_cg_init adds the r.z sum and
 * the z_0 halo, and for the single-reduction body the w_0 = A z_0
 * prologue).  Every rank of the job must
 * call it with the same iters, in the same order.  Stream-ordered,
 * graph-capturable; the bound tol is honoured (the same stop on every
 * rank).  EBB_E_STATE if a field of the group was freed since the bind.
 * */
ebb_status ebb_cg_peer_step(ebb_ctx ctx, int32_t group, int32_t iters, ebb_stream s);

/* Halo of a field over peer memory ("halo exchange of vertex
 * positions and of the partial force sums", without NCCL).  Two modes:
 *   EBB_HALO_COPY  owners store the rows [0, n_src) that peers hold as
 *                  ghosts into the peers' copies of `field` (positions:
 *                  owners -> ghosts; send lists of ebb_peer_send_csr);
 *   EBB_HALO_ADD   each rank adds the partial rows it computed for rows
 *                  another rank owns into the owners' rows with
 *                  red.global.add over peer memory (the reverse add of
 *                  partial f / K rows; lists of ebb_partition_reverse made
 *                  into a send CSR over all rows, n_src = the relation's
 *                  rows); F32 / F64 fields.
 * One mailbox exchange first (every rank has reached the push: no peer still
 * reads a ghost row a COPY overwrites, every owner has written the rows an
 * ADD adds into), then the stores / REDs, one exchange more: when
 * ebb_peer_halo_push ends on a rank (stream order) its rows are current.
 * The mailbox may be the one of the rank's fused PCG group (one epoch
 * counter; every rank issues the same sequence of pushes and PCG steps).
 * field: any non-key dtype of 4 / 8-byte elements, element-major or
 * component-planar (SOA: one element per plane; peer_rows[q] = rank q's
 * relation rows, its plane stride).  peer_field[q]: device address, valid
 * on this rank's device, of rank q's copy; [rank] unused.  bind:
 * synchronous, validates; push: stream-ordered, graph-capturable, a
 * cooperative launch (no launch for a one-rank job). */
#define EBB_HALO_COPY 0
#define EBB_HALO_ADD 1
typedef struct {
    int32_t nranks, rank;
    uint64_t n_src;           /* source rows [0, n_src) (owned vertices for COPY) */
    ebb_field field, send_off, send_dst, mbox;
    int32_t mode;             /* EBB_HALO_COPY | EBB_HALO_ADD                    */
    uint64_t peer_field[EBB_MAX_RANKS], peer_mbox[EBB_MAX_RANKS], peer_rows[EBB_MAX_RANKS];
} ebb_peer_halo;
/* (the field reductions of P:885 across ranks) */
ebb_status ebb_peer_halo_bind(ebb_ctx ctx, int32_t nlocal, const ebb_peer_halo* descs, int32_t* group_out);
ebb_status ebb_peer_halo_push(ebb_ctx ctx, int32_t group, ebb_stream s);

typedef struct {
    ebb_field f, mass, mask;  /* mask: verts U8 (1 = free) or EBB_NONE        */
    ebb_field u, vel;         /* verts vec3 (read-write)                      */
    double h;
    double g[3];
} ebb_explicit_desc;
/* O8 (the update of P:376-377): a = (f + m g)/m;
 * u += v h + a h^2/2; v += a h on free vertices. */
ebb_status ebb_explicit_update(ebb_ctx ctx, const ebb_explicit_desc* d, ebb_stream s);
/* O9 implicit state update (P:941 backward Euler):
 * vel += dv; u += h vel.  dv, u, vel: AOS vec3 fields of one dtype on the
 * same relation (EBB_E_TYPE otherwise).  Stream-ordered. */
ebb_status ebb_implicit_update(ebb_ctx ctx, ebb_field dv, double h, ebb_field u, ebb_field vel, ebb_stream s);
/* Newton iteration update (DESIGN.md §3 (19)), after an
 * EBB_RHS_NEWTON solve: vel += dv; u += h dv (keeps u = u_n + h vel).
 * Fields as ebb_implicit_update.  Stream-ordered. */
ebb_status ebb_newton_update(ebb_ctx ctx, ebb_field dv, double h, ebb_field u, ebb_field vel, ebb_stream s);

/* ---- regular 2-D grid domain (Fig. 3)
 * nx x ny unit cells, cell (i, j) = [i, i+1) x [j, j+1), row-major id
 * i + nx j, periodic.  Keys between grid elements are affine maps of the
 * indices ({{1,0,dx},{0,1,dy}}), computed, never stored.  Dual
 * cell (a, b) spans the cell centres a+1/2..a+3/2, b+1/2..b+3/2 and its
 * cell(dx, dy) is cell (a+dx, b+dy).  Readings: DESIGN.md §3 (22). */
typedef struct { ebb_rel cells, dual_cells; } ebb_grid2;
#define EBB_GRID2_MAX_STENCIL 16
/* two relations of nx*ny rows: <name>.cells and <name>.dual_cells */
ebb_status ebb_grid2_new(ebb_ctx ctx, const char* name, uint32_t nx, uint32_t ny, ebb_grid2* out);
/* out[c] = sum_k weights[k] in[cell(i + offsets[2k], j + offsets[2k+1])]
 * (periodic), per component; in, out: F32/F64 AOS fields of the same shape
 * (<= 4 components) on `cells`, distinct (EBB_E_PHASE).  1..16 points.
 * offsets/weights are host arrays (copied into the launch). */
ebb_status ebb_grid2_stencil(ebb_ctx ctx, ebb_rel cells, ebb_field in, ebb_field out, int32_t npts,
                             const int32_t* offsets, const double* weights, ebb_stream s);
/* PointLocate: dual_cell[p] = (floor(x - 1/2) mod nx)
 * + nx (floor(y - 1/2) mod ny), decided in fp64; pos: AOS vec3 F32/F64 on the
 * particles (z ignored); dual_cell: scalar key-field particles -> dual cells. */
ebb_status ebb_grid2_point_locate(ebb_ctx ctx, ebb_field pos, ebb_field dual_cell, ebb_stream s);
/* Fig. 3 update_particle_vel: x1 = frac(x - 1/2), y1 = frac(y - 1/2),
 * vel = x0 y0 c(0,0) + x1 y0 c(1,0) + x0 y1 c(0,1) + x1 y1 c(1,1) with c the
 * dual cell's cells' cell_vel (AOS, 1..4 components, on the grid's cells);
 * vel: same shape on the particles. */
ebb_status ebb_grid2_particle_vel(ebb_ctx ctx, ebb_field dual_cell, ebb_field cell_vel, ebb_field pos,
                                  ebb_field vel, ebb_stream s);

/* ---- matrix-free element-by-element matvec -----------
 * q = sum_t K_t p_t, the product with the stiffness the element map would
 * assemble (K = sum_t K_t on e[i][j]), from a compact per-tet state
 * instead of the edge-relation matrix.  `d` supplies model, v, Dminv (and,
 * for the state, u, W, mu, lam); f, K, e, energy, scatter are ignored.
 * state: SOA field on tets, dtype of the map, 15x1 (NH: k_i = F^-T g_i,
 * W mu, W c1, W lam) or 26x1 (StVK: h_i = F g_i, W S, W mu F F^T, W mu,
 * W lam).  The matvec zeroes q and adds each element's 4 vec3 rows with
 * red.global.add: equal to the assembled product up to summation
 * order, not bitwise run-to-run.  Stream-ordered. */
ebb_status ebb_tet_stiffness_state(ebb_ctx ctx, const ebb_tet_map_desc* d, ebb_field state, ebb_stream s);
ebb_status ebb_ebe_matvec(ebb_ctx ctx, const ebb_tet_map_desc* d, ebb_field state, ebb_field p, ebb_field q,
                          ebb_stream s);

/* ---- Fig. 2 spring-mass program ------------
 * Query-loops over v.edges of a grouped edge relation (`edges`, grouped by
 * tail, with a `head` key-field, e.g. the tetmesh edges).  All fields F32
 * or F64 (one dtype per call): q, qd, force, pos AOS vec3 on the vertices,
 * mass scalar on the vertices, rest_len scalar on the edges.  The force is
 * the printed one, v.force += K (rest_len normalize(dq) - dq) with
 * dq = e.head.q - v.q and normalize(0) = 0 (DESIGN.md §3 reading 21: a
 * restoring spring has K < 0).  Stream-ordered; EBB_E_PHASE when a field
 * is both read and reduced/written where the paper's phase rules forbid it
 * (P:443-450). */
/* initLen: rest_len[e] = |pos[head] - pos[tail]| */
ebb_status ebb_spring_init_len(ebb_ctx ctx, ebb_rel edges, ebb_field pos, ebb_field rest_len, ebb_stream s);
/* computeInternalForces: force (+)= K sum_{e in v.edges} (rest_len dir - dq);
 * accumulate = 0 overwrites force (Fig. 2's force is zero on entry). */
ebb_status ebb_spring_forces(ebb_ctx ctx, ebb_rel edges, ebb_field q, ebb_field rest_len, double K,
                             ebb_field force, int32_t accumulate, ebb_stream s);
/* applyForces: qdd = force/mass; q += qd dt + qdd dt^2/2; qd += qdd dt; force = 0 */
ebb_status ebb_spring_apply(ebb_ctx ctx, ebb_field mass, double dt, ebb_field q, ebb_field qd, ebb_field force,
                            ebb_stream s);
/* One whole Fig. 2 iteration in ONE kernel: forces from q_in kept in
 * registers, then applyForces writing q_out (q double-buffered: neighbours
 * read q while its owner would write it) and qd; force (nullable) receives
 * the forces.  q_in, q_out, qd, force distinct.  Records are vec3 (3x1) or
 * padded (4x1); padded records need the row-staged kernel, which refuses
 * (EBB_E_RANGE) a vertex with more edge rows than fit shared memory. */
ebb_status ebb_spring_step(ebb_ctx ctx, ebb_rel edges, ebb_field q_in, ebb_field q_out, ebb_field qd,
                           ebb_field rest_len, ebb_field mass, double K, double dt, ebb_field force,
                           ebb_stream s);
/* measureTotalEnergy: out (F64 global) = sum mass qd.qd / 2 (deterministic) */
ebb_status ebb_kinetic_energy(ebb_ctx ctx, ebb_field mass, ebb_field qd, ebb_field out, ebb_stream s);

/* ---- multi-GPU partition ----------------------------- */
/* owner_t(t) = floor(t P / T); owner_v(v) = owner_t(min tet containing v),
 * floor(v P / V) if isolated.  Outputs are I32 fields on tets / verts.
 * Synchronous. */
ebb_status ebb_partition(ebb_ctx ctx, ebb_field tets_v, int32_t nparts,
                         ebb_field owner_t, ebb_field owner_v);

/* The local problem of rank `rank` of an nparts-way decomposition (SURVEY
 * §8(e): "vertex-owned shards with ghost layers"; O4 and its overlapping
 * reading), built on the device from the owner maps of
 * ebb_partition (owner_t, owner_v: I32 on tets / verts of tets_v):
 *   mode EBB_PART_OVERLAP  local tets = every tet with a vertex the rank owns
 *                          (ghost tets: every block of every owned edge row
 *                          is local, so the element map needs no reverse add);
 *   mode EBB_PART_OWN      local tets = the tets the rank owns (O4).
 * Local vertices: the owned ones ascending (global id), then the ghosts
 * (vertices of local tets owned elsewhere) ascending; local tets ascending.
 * Halo lists: send to peer q = owned vertices that are ghosts on q, recv from
 * q = ghosts owned by q, both as local rows in ascending global id (the two
 * ends of a pair derive the same order).  Creates relations name.ltets,
 * name.lverts, name.send, name.recv (the last two only if non-empty) with
 * U32 fields "gid" (global ids), the 4x1 key-field ltets."v" -> lverts, and
 * U32 "rows" (local vertex rows) on send / recv grouped by peer: rows of peer
 * q are [send_ptr[q], send_ptr[q+1]) (host arrays of nparts+1 entries, filled
 * here; same for recv_ptr).  EBB_E_SIZE if the rank's local mesh is empty.
 * Synchronous. */
#define EBB_PART_OVERLAP 0
#define EBB_PART_OWN 1
typedef struct {
    ebb_rel ltets, lverts, send, recv;   /* created relations (send/recv NONE if empty) */
    ebb_field tet_gid, vert_gid;         /* U32: global id of each local tet / vertex   */
    ebb_field v;                         /* ltets 4x1 key -> lverts (local tets.v)      */
    ebb_field send_rows, recv_rows;      /* U32 local vertex rows, grouped by peer      */
    uint64_t n_ltets, n_lverts, n_owned; /* lverts [0, n_owned) are the owned vertices  */
} ebb_partition_info;
/* (SURVEY §8(e) "vertex-owned shards with ghost layers"; O4) */
ebb_status ebb_partition_local(ebb_ctx ctx, ebb_field tets_v, ebb_field owner_t, ebb_field owner_v,
                               int32_t nparts, int32_t rank, int32_t mode, const char* name,
                               ebb_partition_info* out, uint64_t* send_ptr, uint64_t* recv_ptr);

/* Reverse-add lists of rank `rank` on its EBB_PART_OVERLAP local mesh
 * ("halo exchange of vertex positions and of the partial force
 * sums"): every tet is computed by exactly ONE rank, the owner of its
 * lowest-gid vertex (so it is local there); rows whose tail a rank does not
 * own get partial sums from its tets, which are added into the owner's rows.
 *   tets_v, tets_e: 4x1 / 4x4 key-fields of the local tets (-> local verts,
 *   -> the local grouped edge relation); vert_gid: U32 global id and
 *   owner_lv: I32 owner rank of every local vertex.
 * Creates U8 "<name>_own" on the tets (1: this rank computes the tet) and the
 * relations <name>.fsend / .frecv (local vertex rows: forces) and .ksend /
 * .krecv (local edge rows: stiffness), each with a U32 field "rows" grouped
 * by peer, rows of a peer in (tail gid, head gid) order so both ends agree;
 * ptrs (host, 4 x (nparts+1)): the CSR offsets by peer of fsend, frecv,
 * ksend, krecv in that order.  Empty lists leave the relation NONE.
 * Synchronous. */
typedef struct {
    ebb_field own;                            /* U8 on tets                   */
    ebb_rel fsend, frecv, ksend, krecv;       /* list relations (or NONE)      */
    ebb_field fsend_rows, frecv_rows, ksend_rows, krecv_rows;
} ebb_reverse_info;
ebb_status ebb_partition_reverse(ebb_ctx ctx, ebb_field tets_v, ebb_field tets_e, ebb_field vert_gid,
                                 ebb_field owner_lv, int32_t nparts, int32_t rank, const char* name,
                                 ebb_reverse_info* out, uint64_t* ptrs);

/* Lifetime (a rank frees the global mesh it partitioned).  field_free: frees
 * the column (borrowed memory is left alone); EBB_E_STATE if the field groups
 * or indexes a relation.  relation_free: frees every field of the relation
 * and its hidden group index; EBB_E_STATE while a key-field of another live
 * relation targets it.  Both drop every cached plan.  The handles become
 * invalid (EBB_E_ARG on use).  Synchronous.  (Relations and fields: P:405-420,
 * P:663-667; the per-rank global mesh of SURVEY §8(e).) */
ebb_status ebb_field_free(ebb_ctx ctx, ebb_field f);
ebb_status ebb_relation_free(ebb_ctx ctx, ebb_rel rel);

#ifdef __cplusplus
}
#endif
#endif /* EBB_H */
