/*
 * alsub.h -- C ABI of the B200-native AlSub uniform-refinement library (arXiv 1809.06047).
 *
 * One uniform refinement level of a polygon mesh (Catmull-Clark primary; Loop and sqrt3
 * variants), split as in the paper into a topology "build" step and a vertex-data "eval" step
 * (Fig. module_core), repeated `levels` times:
 *   - build: the mesh matrix M, its adjacency E = M M^T{Q_c+Q_c^{c-1}}[lambda]
 *     and F = M M^T{Q_c}[gamma] with edge ids from the upper triangle of E, the refined
 *     M_{i+1}, and the inherited crease matrix C_{i+1};
 *   - eval: face points f = M^T P, edge points, vertex points
 *     S = s1 + s2 + s3, boundary repair and crease overrides
 *     (P:L410-457), Loop and sqrt3 variants.
 *
 * Conventions (binding):
 *   - Child vertex numbering: CC [old V | face points F | edge points E]; Loop [old | edges];
 *     sqrt3 [old | faces].
 *   - Edge id = rank of the undirected edge (max, min) in ascending lexicographic order
 *     (upper triangle of E enumerated column-major, P:L312 + P:L574).
 *   - CC child face off_r + t = (v_t, ep(v_t,v_t+1), fp_r, ep(v_t-1,v_t)); Loop child faces
 *     4r+t; sqrt3 child face 3i+t = (v_t, fp_F(v_t+1,v_t), fp_i).
 *   - Boundary edges are infinitely sharp creases; vertex rules smooth / crease / corner with
 *     semi-sharp blending; Chaikin-style sharpness inheritance (readings R6-R9).
 *   - Positions are fp32 [V][3]; sharpness fp32 (+inf allowed).
 *
 * Pointers: every array argument may be a HOST or a DEVICE pointer (the library asks the CUDA
 * driver which); host inputs are copied on `stream`, host outputs are written by a copy on
 * `stream` followed by a stream synchronisation.  `stream` is a cudaStream_t (NULL = legacy).
 * Errors: every call returns an alsub_status; alsub_last_error() gives a thread-local message.
 * Concurrency: one handle must not be used from two threads at once; handles are independent.
 */
#ifndef ALSUB_H
#define ALSUB_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct alsub_mesh alsub_mesh; /* opaque; owns every internal device table */

typedef enum { ALSUB_CATMULL_CLARK = 0, ALSUB_LOOP = 1, ALSUB_SQRT3 = 2 } alsub_scheme;

typedef enum {
    ALSUB_OK = 0,
    ALSUB_E_ARG = 1,         /* null pointer, negative count, unknown scheme, bad level            */
    ALSUB_E_MESH = 2,        /* face order < 3, repeated vertex in a face, vertex id outside [0,V) */
    ALSUB_E_NONMANIFOLD = 3, /* edge in > 2 faces, directed edge twice (orientation), or a vertex
                                whose interior faces form more than one closed fan                */
    ALSUB_E_SCHEME = 4,      /* Loop/sqrt3 on non-triangles; sqrt3 with boundary or creases        */
    ALSUB_E_CREASE = 5,      /* crease pair not an edge, duplicate pair, sigma < 0 or NaN          */
    ALSUB_E_OVERFLOW = 6,    /* a refined count or slot offset would exceed INT32_MAX              */
    ALSUB_E_NOMEM = 7,       /* device allocation failed                                           */
    ALSUB_E_CUDA = 8         /* any other CUDA runtime error                                       */
} alsub_status;

/* Optional device allocator (e.g. the PyTorch caching allocator).  NULL -> cudaMallocAsync. */
typedef struct {
    void *(*alloc)(size_t bytes, void *stream, void *ctx);
    void (*free)(void *ptr, size_t bytes, void *stream, void *ctx);
    void *ctx;
} alsub_allocator;

typedef struct {
    int64_t verts, faces, edges, boundary_edges, face_slots;
    int64_t creases_upper_bound; /* capacity of the crease list at this level (exact count is on
                                    the device: see alsub_level_topology)                         */
    int32_t face_order;          /* 3 or 4 when uniform, 0 = mixed                                */
    int32_t edges_valid;         /* 1 if `edges` is known for this level (sqrt3 levels >= 1: 0)  */
} alsub_counts;

/* Build a handle from a control mesh (P:L224-226 mesh matrix in CSC form).
 *   face_off     [num_faces+1] int32  exclusive offsets into face_vtx, face_off[0] = 0
 *   face_vtx     [face_off[F]] int32  vertex ids in cyclic CCW order per face
 *   pos          [num_verts][3] fp32
 *   crease_pairs [num_creases][2] int32 vertex pairs (nullable if num_creases == 0)
 *   crease_sigma [num_creases] fp32, >= 0, +inf allowed; 0 entries are ignored
 *   alloc        nullable
 * Copies every input (they may be freed on return), runs the whole level-0 build on `stream`
 * and synchronises `stream` once, after it, to read E_0, the validation flags and the special-
 * list sizes together (edge arrays are sized by the bound E_0 <= S_0 until then).  Device-
 * resident face_off adds one earlier read of the offsets (S_0, face orders) on `stream`.
 * Errors: E_ARG, E_MESH, E_NONMANIFOLD, E_CREASE, E_OVERFLOW, E_NOMEM, E_CUDA (no handle). */
alsub_status alsub_mesh_create(const int32_t *face_off, const int32_t *face_vtx, int32_t num_faces,
                               const float *pos, int32_t num_verts,
                               const int32_t *crease_pairs, const float *crease_sigma, int32_t num_creases,
                               const alsub_allocator *alloc, void *stream, alsub_mesh **out);

/* Replace the level-0 positions (host or device [V][3] fp32). Stream-ordered. */
alsub_status alsub_set_positions(alsub_mesh *mesh, const float *pos, void *stream);

/* Dynamic mode: rebuild everything from the level-0 mesh matrix (a1-a3 of
 * SURVEY.md 8(a)) and run `levels` build+eval iterations of `scheme`.  Fully asynchronous on
 * `stream` (no host synchronisation); the first call per (scheme, levels) allocates the level
 * tables and launches eagerly, the second records a CUDA graph that later calls replay
 * (env ALSUB_NO_GRAPH=1 disables graphs).
 * levels = 0 returns the input.  Errors: E_ARG, E_SCHEME, E_OVERFLOW, E_NOMEM, E_CUDA. */
alsub_status alsub_refine(alsub_mesh *mesh, alsub_scheme scheme, int32_t levels, void *stream);

/* Per-kernel timing of one eager refine (instrumentation; the paper reports "the sum of all
 * kernel timings").  A CUDA event is recorded after every kernel launch on `stream`;
 * entry i is the time between event i-1 (or the start event) and event i, i.e. the kernel plus
 * any memset issued just before it.  Synchronises `stream`.  *n_out = number of kernels
 * (entries beyond `cap` are dropped).  level = -1 for the level-0 build. */
typedef struct {
    char name[32];
    int32_t level;
    float ms;
} alsub_kernel_time;
alsub_status alsub_refine_profile(alsub_mesh *mesh, alsub_scheme scheme, int32_t levels, void *stream,
                                  alsub_kernel_time *out, int32_t cap, int32_t *n_out);

/* Host-only: counts of level `level` of the last refine (level 0 always available). */
alsub_status alsub_level_counts(const alsub_mesh *mesh, int32_t level, alsub_counts *out);

/* Export the topology of level `level` (0 .. last refine's levels).  Every output is nullable.
 *   face_vtx     [face_slots]       face_off [faces+1]
 *   edge_vtx     [edges][2] (lo,hi) in edge-id order      (levels < last refined level)
 *   edge_face    [edges][2] face of lo->hi, face of hi->lo, -1 = none
 *   crease_pairs [creases_upper_bound][2] (lo,hi) ascending edge id; crease_sigma [...]
 *   num_creases  [1] int32: the exact number written (boundary edges are not listed)
 * Errors: E_ARG (level out of range, edges requested where not available). */
alsub_status alsub_level_topology(const alsub_mesh *mesh, int32_t level, int32_t *face_vtx, int32_t *face_off,
                                  int32_t *edge_vtx, int32_t *edge_face, int32_t *crease_pairs,
                                  float *crease_sigma, int32_t *num_creases, void *stream);

/* Export the positions of level `level` ([verts][3] fp32). */
alsub_status alsub_level_positions(const alsub_mesh *mesh, int32_t level, float *pos, void *stream);

/* Static mode (Fig. CC_singleSpMV top): evaluate `num_frames` frames of level-0
 * vertex data through the topology of the last alsub_refine (same scheme, `levels` <= its
 * levels) -- only the eval half of every module runs.
 *   frames_in  [num_frames][V0][3] fp32,  frames_out [num_frames][V_levels][3] fp32
 * Frames are processed in batches that share each topology read.  Stream-ordered.
 * Errors: E_ARG (no prior refine / levels too large), E_NOMEM, E_CUDA. */
alsub_status alsub_eval_frames(alsub_mesh *mesh, int32_t levels, const float *frames_in, int32_t num_frames,
                               float *frames_out, void *stream);

/* Extra vertex channels (uv, colours, any per-vertex linear data):
 * refine `channels` values per control vertex with the same stencils as the positions (same
 * smooth / boundary / crease rules, reading R22) through the topology of the last alsub_refine.
 *   attr_in [V0][channels] fp32, attr_out [V_levels][channels] fp32 (host or device pointers;
 *   host output synchronises `stream`).  Channels are packed three at a time into frames of
 *   alsub_eval_frames by a device kernel and unpacked the same way.
 * Errors: E_ARG (channels < 0, null pointers, levels beyond the last refine), E_NOMEM, E_CUDA. */
alsub_status alsub_eval_attributes(alsub_mesh *mesh, int32_t levels, const float *attr_in, int32_t channels,
                                   float *attr_out, void *stream);

/* Hierarchical edits / displacement ("we have access to the vertex data after each
 * iteration and can arbitrarily modify it").  alsub_level_positions_ptr returns the handle-owned
 * device array [V_level][3] fp32 of level `level` of the last refine (level 0 = the control
 * positions); it stays valid until the next alsub_refine with a different level count or
 * alsub_mesh_destroy.  The caller may write it (stream-ordered), then alsub_reevaluate
 * recomputes the positions of levels from_level+1 .. levels from it over the stored topology
 * (static mode; topology and crease sharpness unchanged).  A later alsub_refine recomputes
 * everything from the level-0 positions.
 * Errors: E_ARG (null pointers, level / from_level outside 0 .. levels of the last refine). */
alsub_status alsub_level_positions_ptr(alsub_mesh *mesh, int32_t level, float **pos_dev);
alsub_status alsub_reevaluate(alsub_mesh *mesh, int32_t from_level, void *stream);

/* The refinement matrix R = R_{L-1} ... R_0:
 * P_L = R P_0 for the topology of the last alsub_refine (CC or Loop).  Built by probing: each
 * control face f owns the level-`levels` vertices of its descendant faces (smallest f wins), a row
 * is supported on the 1-ring vertex set of its owner, and a colouring of the control vertices with
 * no repeated colour inside any 1-ring lets ceil(colours / 3) probe frames through the static path
 * (alsub_eval_frames) read every weight exactly once.  Rows in CSR, exact zeros dropped.
 * Errors: E_ARG (levels outside 1 .. last refine), E_SCHEME (sqrt3), E_NOMEM, E_CUDA. */
alsub_status alsub_build_refinement_matrix(alsub_mesh *mesh, int32_t levels, void *stream);
/* levels, rows (= V_levels) and non-zeros of the built matrix; any pointer may be NULL. */
alsub_status alsub_refinement_matrix_info(const alsub_mesh *mesh, int32_t *levels, int64_t *rows, int64_t *nnz);
/* The blocked form alsub_eval_frames_matrix evaluates: `chunks` = F0 + the isolated control
 * vertices (one per owner face, then one identity row per isolated vertex); `weights` = floats of
 * the dense per-chunk blocks W_c [|S_c|][rows_c rounded up to 64] (zeros included).  Either
 * pointer may be NULL.  Errors: E_ARG (no matrix built). */
alsub_status alsub_refinement_matrix_blocks(const alsub_mesh *mesh, int64_t *chunks, int64_t *weights);
/* CSR export: row_off [rows+1], cols [nnz] (control vertex ids, ascending per row), vals [nnz];
 * host or device pointers, any may be NULL; synchronises `stream`. */
alsub_status alsub_refinement_matrix_csr(const alsub_mesh *mesh, int32_t *row_off, int32_t *cols, float *vals,
                                         void *stream);
/* Static evaluation by the single SpMM P_L = R P_0: frames_in [num_frames][V0][3],
 * frames_out [num_frames][V_levels][3], DEVICE pointers; batches of 32 frames.  R is applied in
 * its blocked form: the rows owned by one control face share that face's 1-ring support S_c, so
 * each chunk is a dense |S_c| x rows_c product (weights in registers, the batch's positions of S_c
 * staged in shared memory).  Asynchronous (stream-ordered).
 * Errors: E_ARG (no matrix built -- also after a refine with another scheme or level count --,
 * host pointers).  alsub_build_refinement_matrix additionally returns E_OVERFLOW when R has more
 * than 2^31 - 1 non-zeros (its CSR export uses int32 offsets). */
alsub_status alsub_eval_frames_matrix(alsub_mesh *mesh, const float *frames_in, int32_t num_frames, float *frames_out,
                                      void *stream);
/* The same evaluation, and every output frame's summary record (the alsub_frame_summary layout:
 * int32 [num_frames][8] = bbox lo.xyz, hi.xyz as float bits, then the uint64 checksum) folded in
 * as the frame is written -- identical bit for bit to alsub_frame_summary of frames_out, without
 * reading the frames back.  summary: DEVICE pointer.  Errors: as alsub_eval_frames_matrix; E_ARG
 * for a null summary. */
alsub_status alsub_eval_frames_matrix_summary(alsub_mesh *mesh, const float *frames_in, int32_t num_frames,
                                              float *frames_out, int32_t *summary, void *stream);

/* Selective / feature-adaptive subdivision, the extraction module (
 * P:L459-499, Fig. module_selective).  From level `level` of `mesh` (0, or 1 .. levels of its
 * last alsub_refine):
 *   x_0 = vsel [V_level] uint8 (host or device; nonzero = selected), or NULL = the extraordinary
 *         vertices, valence n = M 1 != 4 (Eq. vo)
 *   `rings` >= 1 propagation steps q_i = M^T x_i (faces with a selected vertex), x_{i+1} = M q_i
 *   M' = X M X̊, P' = X P: the selected faces and their vertices, both in ascending original order,
 *   plus the level's live creases whose two vertices are selected (pairs that are not an edge of
 *   an extracted face are dropped, reading R25)
 * become the control mesh (level 0) of a new handle *out (same allocator); refine it as usual.
 * Synchronises `stream` once (to size the new mesh).  Errors: E_ARG (null pointers, rings < 1,
 * level out of range), E_NOMEM, E_CUDA, and the alsub_mesh_create errors of the extracted mesh. */
alsub_status alsub_mesh_extract(const alsub_mesh *mesh, int32_t level, const uint8_t *vsel, int32_t rings,
                                void *stream, alsub_mesh **out);
/* Original ids of an extracted handle's control mesh: vtx_map [V0] and face_map [F0] (counts
 * from alsub_level_counts(extracted, 0)); either may be NULL; host or device pointers.
 * Errors: E_ARG (null mesh, or a handle not made by alsub_mesh_extract). */
alsub_status alsub_extract_maps(const alsub_mesh *mesh, int32_t *vtx_map, int32_t *face_map, void *stream);

/* Reverse Cuthill-McKee ordering of a control mesh (RCM on the
 * graph Laplacian of the mesh, rows of M permuted, columns sorted by their first non-zero).
 * Host pointers, host computation (an offline preprocess; no handle, no GPU needed).
 *   face_off [num_faces+1], face_vtx [face_off[num_faces]]: the mesh as for alsub_mesh_create
 *   perm_vtx [num_verts]  out: perm_vtx[new] = old vertex id
 *   perm_face [num_faces] out: perm_face[new] = old face id (faces by min new vertex id, stable)
 * Tie breaking is fixed (degree, then id) -- see paper_1809_06047_b200/csrc/reorder.cpp.
 * Relabel the mesh with these permutations before alsub_mesh_create.
 * Errors: E_ARG (null pointers, negative counts), E_MESH (vertex index out of range). */
alsub_status alsub_rcm_order(const int32_t *face_off, const int32_t *face_vtx, int32_t num_faces, int32_t num_verts,
                             int32_t *perm_vtx, int32_t *perm_face);

/* Kernel probe (measurement): time ONE kernel inside every replayed refine.
 * Arms a probe on the first launch named `kernel` ("cc_face", "cc_edge", "cc_vertex", "crease",
 * "s3_face", ...; the names alsub_refine_profile reports) at refinement level `level` (0-based
 * parent level, -1 = the level-0 build).  The next alsub_refine re-captures its CUDA graph with two
 * external event-record nodes around that launch; replay i < steps records into event pair i, so
 * the kernel is timed on its own stream inside the caller's timed region at no host sync.
 * Re-arming with the same level/kernel only resets the pair counter (no re-capture); steps = 0
 * disarms (and drops the graph).  Host-side; synchronises the device once.
 * Errors: E_ARG (null mesh, steps < 0 or > 2^20, null name with steps > 0), E_CUDA. */
alsub_status alsub_probe(alsub_mesh *mesh, int32_t level, const char *kernel, int32_t steps);

/* Durations (ms, host array of `cap`) of the probed kernel in the replays since alsub_probe, in
 * order; *count = number of replays recorded (<= steps).  Waits for the last one.
 * Errors: E_ARG (null mesh/count, or the probe matched no launch of the captured refine), E_CUDA. */
alsub_status alsub_probe_read(alsub_mesh *mesh, float *ms, int32_t cap, int32_t *count);

/* Offsets of the probed kernel inside replay i (measurement: the level timeline of DESIGN.md §12):
 * start_ms[i] / stop_ms[i] = ms from the caller's event ref_events[i] (a cudaEvent_t with timing,
 * recorded on the refine's stream before replay i) to the probe's start / stop record.  The start
 * record follows the kernel's predecessors, so it is the time the kernel could start.  Host arrays
 * of `cap`; *count as alsub_probe_read.  Waits for the last replay.
 * Errors: E_ARG (null mesh/arrays/count, no matching launch), E_CUDA (e.g. an event without timing). */
alsub_status alsub_probe_read_offsets(alsub_mesh *mesh, void *const *ref_events, float *start_ms, float *stop_ms,
                                      int32_t cap, int32_t *count);

/* Per-frame result summary of a batch of frames (what the sharded config-5 job
 * gathers over NCCL -- 32 B per frame instead of the frame).  frames: DEVICE fp32 [num_frames]
 * [num_verts][3] (e.g. the output of alsub_eval_frames); summary: DEVICE, num_frames records of
 * 32 bytes = { float lo[3], hi[3]; uint64_t sum; } with lo/hi the bounding box (exact fp32 min /
 * max; -0 orders below +0) and sum = sum_i bits(x_i) * (2 i + 1) mod 2^64 over the frame's 3V
 * floats in memory order (exact and order-independent, so the record is deterministic).
 * Stream-ordered, no host sync.  Errors: E_ARG (negative counts, null or host pointers,
 * num_frames > 65535), E_CUDA. */
alsub_status alsub_frame_summary(const float *frames, int32_t num_frames, int64_t num_verts, void *summary,
                                 void *stream);

/* Number of kernel launches issued by the last alsub_refine / alsub_eval_frames call
 * (a graph replay counts the kernels inside it). */
int64_t alsub_last_launch_count(const alsub_mesh *mesh);

void alsub_mesh_destroy(alsub_mesh *mesh);
const char *alsub_last_error(void);
const char *alsub_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ALSUB_H */
