// internal.h -- host-side declarations shared by the AlSub CUDA translation units.
#pragma once
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>
#include <vector>

#include "common.cuh"

namespace alsub {

// Counts kernel launches issued into a stream (reported by alsub_last_launch_count).
struct Launches {
    int64_t n = 0;
    // optional second stream for independent kernels of a level (forked / joined with events;
    // inside stream capture this becomes parallel graph branches)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // level-0 build: the special-list chain runs on the side stream beside the level-0 face kernel;
    // build_open = that branch is not joined yet (ev_build marks its end); the level-0 vertex
    // kernel (which reads the lists) waits for it
    cudaEvent_t ev_build = nullptr;
    cudaEvent_t ev_aux = nullptr;  // Loop: end of the vertex kernel, for the crease pass on the side branch
    bool build_open = false;
    bool can_fork() const { return side != nullptr && !timing && !no_fork(); }
    static bool no_fork() {  // ALSUB_NO_FORK=1: one branch (experiments)
        static const bool v = [] { const char *e = getenv("ALSUB_NO_FORK"); return e && e[0] == '1'; }();
        return v;
    }
    // optional per-kernel timing (alsub_refine_profile): an event after every launch
    bool timing = false;
    int level = -1;
    std::vector<cudaEvent_t> ev;
    std::vector<const char *> name;
    std::vector<int> lvl;
    // optional probe (alsub_probe): external event records around the first launch named
    // probe_name at level probe_level; captured into the CUDA graph as event-record nodes
    const char *probe_name = nullptr;
    int probe_level = -2;
    cudaEvent_t probe_ev[2] = {nullptr, nullptr};
    // the probe's event records hang off the main chain on their own stream (forked before and
    // after the kernel, joined at the end of the refine), so the kernel keeps its programmatic
    // launch edges to its neighbours
    cudaStream_t probe_stream = nullptr;
    cudaEvent_t probe_dep[3] = {nullptr, nullptr, nullptr};
    bool probe_hit = false;
    bool probing(const char *kname) const;
    void done(const char *kname, cudaStream_t s) {
        ++n;
        if (timing) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            cudaEventRecord(e, s);
            ev.push_back(e);
            name.push_back(kname);
            lvl.push_back(level);
        }
    }
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Programmatic dependent launch (sm_90+): every kernel starts with griddepcontrol.wait, so it may
// be launched while its predecessor drains; inside the CUDA graph this overlaps the launch latency
// of each level kernel with the tail of the previous one.  ALSUB_NO_PDL=1 disables it.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void launch(Launches &L, const char *name, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                   cudaStream_t s, Args &&...args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    const bool probe = L.probing(name);
    if (probe) {
        cudaEventRecord(L.probe_dep[0], s);
        cudaStreamWaitEvent(L.probe_stream, L.probe_dep[0], 0);
        cudaEventRecordWithFlags(L.probe_ev[0], L.probe_stream, cudaEventRecordExternal);
    }
    cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
    if (probe) {
        cudaEventRecord(L.probe_dep[1], s);
        cudaStreamWaitEvent(L.probe_stream, L.probe_dep[1], 0);
        cudaEventRecordWithFlags(L.probe_ev[1], L.probe_stream, cudaEventRecordExternal);
        L.probe_hit = true;
    }
    L.done(name, s);
}
inline unsigned grid_for(int64_t n, int threads = kThreads) {
    int64_t g = ceil_div(n > 0 ? n : 1, threads);
    return (unsigned)g;
}

// ---------------- primitives (prims.cu) ----------------
// Device-wide exclusive scan of int32 (decoupled look-back, one pass).  `total` (nullable)
// receives the sum.  `scratch` must hold scan_scratch_bytes(n) bytes.
size_t scan_scratch_bytes(int64_t n);
void scan_exclusive(const int32_t *in, int32_t *out, int64_t n, int32_t *total, void *scratch,
                    cudaStream_t s, Launches &L, bool prezeroed = false);
// two independent exclusive scans in one launch (the level-0 build's special-edge flags and
// special-vertex counts)
void scan_exclusive2(const int32_t *ina, int32_t *outa, int64_t na, int32_t *tota, void *scra,
                     const int32_t *inb, int32_t *outb, int64_t nb, int32_t *totb, void *scrb, cudaStream_t s,
                     Launches &L, bool prezeroed);
// initialise up to kZeroSegs int32 arrays in one launch (the level-0 build's ~11 plus up to 3 per
// refined level: boundary words, special words, Loop scan status)
constexpr int kZeroSegs = 64;
struct ZeroSegs {
    int n = 0;
    int32_t *ptr[kZeroSegs];
    int64_t words[kZeroSegs];
    int32_t value[kZeroSegs];
    void add(void *p, int64_t w, int32_t v = 0) {
        if (p && w > 0 && n < kZeroSegs) { ptr[n] = (int32_t *)p; words[n] = w; value[n] = v; ++n; }
    }
};
void zero_segments(const ZeroSegs &z, cudaStream_t s, Launches &L);
// [V][C] vertex channels <-> ceil(C/3) frames of [V][3] (alsub_eval_attributes)
void pack_channels(const float *in, int64_t V, int32_t C, float *out, cudaStream_t s, Launches &L);
void unpack_channels(const float *in, int64_t V, int32_t C, float *out, cudaStream_t s, Launches &L);

// ---------------- level-0 build (build0.cu) ----------------
struct Build0 {
    // inputs
    int32_t V, F, S, K_in;
    int order;  // 0 mixed, 3, 4
    const int32_t *face_off, *face_vtx, *crease_in;
    const float *sigma_in;
    // outputs / work
    int32_t *slot_face;           // [S] (all orders: used for validation & mixed topology)
    int32_t *vtx_off, *vtx_slot;  // [V+1], [S] (M^T in CSR, rows ascending by slot)
    int32_t *vtx_cnt;             // [V+1] row lengths of M^T
    int32_t *vtx_cur;             // [V] scatter cursors of the M^T counting sort
    int32_t *edge_cnt, *edge_off; // [V], [V]
    int32_t *face_edge, *face_twin, *vtx_slot0;  // [S], [S], [V]
    int2 *edge_hh;                // [E] (smallest slot of the edge, the other slot or -1)
    int32_t *vbnd;                // [V] 1 = vertex on a boundary edge
    uint32_t *bnd_word;           // [ceil(E/32)]
    int32_t *bnd_wcnt, *bnd_wpre; // [ceil(E/32)]
    float *edge_sigma;            // [E]
    int32_t *edge_cidx;           // [E] crease index claiming the edge, -1
    int32_t *sp_flag, *sp_off;    // [E]
    SpEdge *sp;                   // [cap] special edges
    int32_t *sv_vtx;              // [cap] special vertices
    int32_t *sv_cnt, *sv_off, *sv_list;  // special-vertex CSR (level 0)
    uint32_t *spw;                // [ceil(E/32)] special-edge bitmask (level 0)
    int32_t *spwpre;              // [ceil(E/32)] its per-word prefix (= sp_off at the word start)
    int32_t *flags;               // device status flags
    int32_t *scalars;             // device scalars: [0] E, [1] B, [2] K special, [3] NSV, [5] long rows
    int32_t *long_list;           // [V] vertices with > 16 incident slots (k_long_rows)
    uint64_t *long_keys;          // [4 S] sort keys of rows longer than the shared-memory cap
    int32_t nlong = -1;           // number of long rows (-1: not known yet, i.e. inside create)
    int32_t E;                    // host-known after the count pass (create) or plan (refine)
    void *scratch;
    bool zeroed = false;          // refine: every work array and scan region pre-initialised by k_zero
    bool no_special = false;      // refine of a closed, crease-free mesh: skip boundary/crease tables
    int32_t crease_lenient = 0;   // 1: crease pairs that are not edges are dropped (extracted meshes)
};
size_t build0_scratch_bytes(int32_t V, int32_t S);
// refine: add the level-0 work arrays / scan regions to z (one k_zero launch instead of memsets)
void build0_zero_segments(Build0 &b, ZeroSegs &z);

// ---- refinement matrix R (rmatrix.cu, NEXT-1) ----
constexpr int kRmLanes = 32;  // frames per SpMM batch (= lanes)
void rm_owner(const int32_t *face_vtx, int32_t FL, int order, int shift, const int32_t *slot_face, int32_t *owner,
              cudaStream_t s, Launches &L);
void rm_probes(int32_t V0, const int32_t *colour, int32_t nprobe, float *out, cudaStream_t s, Launches &L);
void rm_assemble(int32_t VL, const int32_t *owner, const int32_t *sup_off, const int32_t *sup, const int32_t *colour,
                 const float *probe, int64_t probe_stride, bool fill, int32_t *row_len, const int32_t *row_off,
                 int2 *ent, int64_t *nnz64, cudaStream_t s, Launches &L);
// per-frame summary records (summary.cu): init (empty bbox, zero sum) and decode (ordered ints ->
// float bits) of records accumulated by a producer kernel
void summary_init(SummaryRec *rec, int32_t nb, cudaStream_t s, Launches &L);
void summary_decode(SummaryRec *rec, int32_t nb, cudaStream_t s, Launches &L);
// blocked R (chunk = owner face / isolated control vertex; rmatrix.cu)
void rb_hist(int32_t VL, const int32_t *owner, const int32_t *iso_chunk, int32_t *chunk, int32_t *cnt, cudaStream_t s,
             Launches &L);
void rb_scatter(int32_t VL, const int32_t *chunk, const int32_t *row_off, int32_t *cur, int32_t *rows, cudaStream_t s,
                Launches &L);
void rb_sort(int32_t C, const int32_t *row_off, const int32_t *sup_off, int32_t *rows, int32_t *pos, int64_t *wlen,
             int64_t *w_off, cudaStream_t s, Launches &L);
void rb_fill(int32_t VL, const int32_t *chunk, const int32_t *pos, const int32_t *row_off, const int32_t *sup_off,
             const int32_t *sup, const int64_t *w_off, const int32_t *colour, const float *probe, int64_t probe_stride,
             float *W, cudaStream_t s, Launches &L);
void rb_eval(int32_t C, const int32_t *row_off, const int32_t *sup_off, const int64_t *w_off, const int32_t *rows,
             const int32_t *sup, const float *W, const float *in, int32_t V0, int32_t nb, float *XT, int64_t VL,
             float *out, SummaryRec *rec, cudaStream_t s, Launches &L);

// ---- selective subdivision: extraction (extract.cu) ----
struct ExSrcHost {
    int32_t V, F, S, order;  // order 3 / 4 (face r = slots [order r, ...)) or 0 (face_off)
    const int32_t *face_off, *face_vtx;
    const float *pos;        // [V][3]
    const SpEdge *sp;        // the level's special-edge list (creases + boundary)
    int32_t nsp;
};
// device work arrays: n, x, vid [V]; q, fid, fo, foff [F]; cflag, cid [nsp]; tot [4] (V', F',
// S', K'); scratch of scan_scratch_bytes(max(V, F, nsp))
struct ExWork {
    int32_t *n, *x, *vid, *q, *fid, *fo, *foff, *cflag, *cid, *tot;
    void *scratch;
};
// device outputs sized V, F + 1, S, V, F, 2 nsp, 3 V, nsp
struct ExOutHost {
    int32_t *face_off, *face_vtx, *vmap, *fmap, *crease;
    float *pos, *sigma;
};
void extract_level(const ExSrcHost &h, const uint8_t *vsel, int32_t rings, ExWork &w, ExOutHost &out, cudaStream_t s,
                   Launches &L);
void build0_validate(Build0 &b, cudaStream_t s, Launches &L);
void build0_count_edges(Build0 &b, cudaStream_t s, Launches &L);  // through edge_off + scalars[0]
void build0_fill(Build0 &b, bool check_fans, cudaStream_t s, Launches &L);  // needs b.E

// ---------------- per-level kernels ----------------
struct LevelDev {
    int32_t V, F, S, E, B;  // parent counts
    int order;              // 0, 3, 4
    const int32_t *face_off, *slot_face;  // order 0
    const int32_t *face_vtx, *face_edge, *face_twin, *vtx_slot0;
    const int2 *edge_hh;       // [E] (owner slot = smallest, twin slot or -1)
    const uint32_t *bnd_word;
    const int32_t *bnd_wpre;
    const int32_t *loop_base;  // Loop: [E] exclusive scan of child-edge counts
    // special lists of the parent level (host-known sizes)
    const SpEdge *sp;
    int32_t nsp;
    const int32_t *sv_vtx, *sv_off, *sv_list;
    int32_t nsv;
    // CC: edge e is special iff bit e of spw; its list index = spwpre[e/32] + popcount (fused crease)
    const uint32_t *spw;
    const int32_t *spwpre;
    int32_t crease;   // 1 = apply boundary/crease rules inside the level kernels (CC)
    int32_t inherit;  // 1 = also build the child special lists
};
struct ChildDev {
    int32_t V, F, S, E;  // child counts
    int32_t *face_vtx, *face_edge, *face_twin, *vtx_slot0;
    int2 *edge_hh;
    uint32_t *bnd_word;
    int32_t *bnd_wpre;
    SpEdge *sp;
    int32_t *sv_vtx, *sv_off, *sv_list;
    uint32_t *spw;
    int32_t *spwpre;
};

// positions: P [nb][V][3] (frame stride Pstride floats), Pn [nb][V'][3]
struct Frames {
    const float *P;
    float *Pn;
    int64_t Pstride, Pnstride;
    int nb;
    // CC levels >= 2: half ring sums of the edge points born at this level, one per parent slot
    // (= per face of this level), written by the face kernel, read by the vertex kernel
    float *hs = nullptr;
    int64_t hsstride = 0;
    // CC levels >= 1: per-face contribution to its corner-0 vertex, c0[q] = p(corner 1) + f_q,
    // written by the face kernel; every vertex born before this level sums its faces' c0
    float *c0 = nullptr;
    int64_t c0stride = 0;
    // the last refined level (>= 3) keeps only the corner sums it reads -- faces r = 0 mod 4, whose
    // corner 0 is a vertex born before level l-1 -- compacted at r >> 2 (c0shift = 2): full 96-B
    // runs per warp instead of 12-B stores of every face
    int32_t c0shift = 0;
    // last level: the ring terms of the edge-point groups that straddle two blocks of the
    // grandparent edge kernel, [edge block][4][3], and an arrival counter per block boundary (gcnt,
    // zero between launches): the second of the two blocks finishes the group
    float *gside = nullptr;
    int32_t *gcnt = nullptr;
    int64_t gsidestride = 0;
    // per-frame views ([V][3], vertex stride 3)
    ALSUB_HD PR rd(int f) const { return PR{P + f * Pstride, 3}; }
    ALSUB_HD PW wr(int f) const { return PW{Pn + f * Pnstride, 3}; }
    ALSUB_HD PW hsw(int f) const { return PW{hs + f * hsstride, 3}; }
    ALSUB_HD PR hsr(int f) const { return PR{hs + f * hsstride, 3}; }
    ALSUB_HD PW c0w(int f) const { return PW{c0 + f * c0stride, 3}; }
    ALSUB_HD PR c0r(int f) const { return PR{c0 + f * c0stride, 3}; }
};

// Vertex-id segments of a CC level: level-l vertex ids are
// [orig V0 | fp(1) F0 | ep(1) E0 | fp(2) F1 | ep(2) E1 | ... | fp(l) F_{l-1} | ep(l) E_{l-1}].
// A vertex born at level m has its level-l incident slots = 4^(l-m) x its level-m slots, which
// are closed-form in the level-(m-1) tables.  The vertex kernel interleaves all segments so a
// block touches one spatial band of the mesh.
constexpr int kMaxLevels = 16;
constexpr int kMaxSeg = 2 * kMaxLevels + 1;
struct VSegs {
    int32_t nseg, level;
    int32_t start[kMaxSeg], len[kMaxSeg];
    int8_t type[kMaxSeg];   // 0 = level-0 vertex, 1 = face point, 2 = edge point
    int8_t birth[kMaxSeg];  // level m at which the vertex was created
    const int2 *ehh[kMaxLevels];  // ehh[m-1] = edge pairs of level m-1
    const int32_t *vtx_off0, *vtx_list0, *face_off0, *slot_face0, *vbnd0;
    // level-0 vertices with long M^T rows (> kLongRow slots; the build's list): CC sums their rings
    // in k_cc_vertex_long
    const int32_t *long_list = nullptr;
    int32_t nlong = 0;
    int32_t hs_seg;  // segment whose vertex points come from the half sums (-1 = none)
    // sqrt3: slot multiplier 3^(l-m) per segment and the level m-1 face rows
    int32_t mult[kMaxSeg];
    const int32_t *fvx[kMaxLevels], *ftw[kMaxLevels];
    // CC fused crease: special bitmask / prefix and special-vertex count of level m-1 per birth
    const uint32_t *spw[kMaxLevels];
    const int32_t *spwpre[kMaxLevels];
    int32_t nsvb[kMaxLevels];
    // boundary words / per-word prefix of level m (for the structured child-edge ids 4e - bprefix)
    const uint32_t *bw[kMaxLevels];
    const int32_t *bwp[kMaxLevels];
    // last refined level: segment of the edge points born at level l-1 whose vertex points the
    // grandparent edge kernel already wrote (those whose 4 child edges fall in one of its blocks)
    int32_t gp_skip_seg = -1;
};

// mode: adj = emit child adjacency (not the last level); topo = emit child faces;
//       acc = accumulate crease valency/sharpness (refine) vs reuse stored (eval_frames)
// The child boundary words (c.bnd_word) must be zero on entry when adj && p.B > 0.
// gp (nullable) = the grandparent level: at the last refined level (>= 2) the face kernel
// recomputes its edge ids from gp's rows and the edge kernel iterates gp's edges
void cc_level(const LevelDev &p, const ChildDev &c, const Frames &fr, bool topo, bool adj, const VSegs &segs,
              const LevelDev *gp, cudaStream_t s, Launches &L);
// crease >= 0: also run the crease module (crease_level with ep_base = V, scheme 1, inherit =
// crease == 1) inside the level, on the side branch after the edge kernel once the vertex kernel
// is done, i.e. beside the face kernel
void loop_level(const LevelDev &p, const ChildDev &c, const Frames &fr, bool topo, bool adj, int32_t *stat,
                int32_t *base, const VSegs &g, cudaStream_t s, Launches &L, int crease = -1);
void sqrt3_level(const LevelDev &p, const ChildDev &c, const Frames &fr, bool topo, bool adj, const VSegs &g,
                 cudaStream_t s, Launches &L);
// crease / boundary module (crease.cu): ONE kernel per level -- edge and vertex overrides and
// (inherit) the child special lists.  ep_base = first edge-point id; scheme 0 CC, 1 Loop.
void crease_level(const LevelDev &p, const ChildDev &c, const Frames &fr, int32_t ep_base, int scheme, bool inherit,
                  cudaStream_t s, Launches &L);
// Loop child-edge counts -> loop_base (scan); cnt [E] scratch
void loop_edge_base(const LevelDev &p, int32_t *stat, int32_t *base, cudaStream_t s, Launches &L);
// topology export helper: edge_vtx / edge_face from the edge pairs
void export_edges(const LevelDev &p, int32_t *edge_vtx, int32_t *edge_face, cudaStream_t s, Launches &L);

}  // namespace alsub
