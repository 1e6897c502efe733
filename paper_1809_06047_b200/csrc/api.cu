// api.cu -- the C ABI (include/alsub.h): handle lifetime, level plans, the level loop and its
// CUDA-graph capture, static-mode frame evaluation and topology/position export.
//
// The host side only computes closed-form level counts and launches
// kernels; every step of the refinement runs on the device.  One device->host read happens per
// handle (at create: E_0, validation flags and special-list sizes); alsub_refine is fully
// asynchronous and replayable as a CUDA graph.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/alsub.h"
#include "internal.h"

namespace alsub {
void init_scheme_tables(cudaStream_t s);
}

using namespace alsub;

static thread_local std::string g_err;

static alsub_status fail(alsub_status st, const std::string &msg) {
    g_err = msg;
    return st;
}
namespace alsub {
alsub_status set_error(alsub_status st, const char *msg) { return fail(st, msg); }
}  // namespace alsub

#define CU(call)                                                                                          \
    do {                                                                                                  \
        cudaError_t _e = (call);                                                                          \
        if (_e != cudaSuccess) return fail(ALSUB_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

static bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

struct LevelHost {
    int64_t V = 0, F = 0, S = 0, E = 0, B = 0;
    int order = 4;
    bool edges_valid = true;
    int32_t *face_off = nullptr, *slot_face = nullptr, *face_vtx = nullptr, *face_edge = nullptr,
            *face_twin = nullptr, *vtx_slot0 = nullptr;
    int2 *edge_hh = nullptr;
    uint32_t *bnd_word = nullptr;
    int32_t *bnd_wpre = nullptr;
    int32_t *loop_stat = nullptr, *loop_base = nullptr;  // Loop: child-edge base scan (status words, bases)
    SpEdge *sp = nullptr;       // special edges of this level [nsp]
    int64_t nsp = 0;            // = 2^l K_0
    int32_t *sv_list = nullptr; // [2 nsp] incident special edges of the special vertices
    uint32_t *spw = nullptr;    // CC fused crease: special-edge bitmask of this level
    int32_t *spwpre = nullptr;
    int64_t nsv = 0;            // special vertices of this level (prefix of the shared table)
    float *pos = nullptr;
};

struct alsub_mesh {
    alsub_allocator alloc{};
    bool custom = false;
    int device = 0;
    std::vector<std::pair<void *, size_t>> mem_create, mem_plan, mem_frames;
    // level-0 inputs
    int32_t V0 = 0, F0 = 0, S0 = 0, Kin = 0, order0 = 0;
    int32_t *in_face_off = nullptr, *in_face_vtx = nullptr, *in_crease = nullptr;
    float *in_sigma = nullptr, *pos0 = nullptr;
    Build0 b0{};
    int32_t E0 = 0, B0 = 0, K0 = 0, NSV0 = 0;
    // a handle made by alsub_mesh_extract: original vertex / face ids of its control mesh
    int32_t *ext_vmap = nullptr, *ext_fmap = nullptr;
    bool extracted = false;
    bool user_creases = false;
    int32_t *sv_vtx = nullptr, *sv_off = nullptr;  // shared special-vertex table (prefix per level)
    int32_t *sv_vtx_create = nullptr, *sv_off_create = nullptr;
    float *hs = nullptr;          // half ring sums (CC, levels >= 2), [3 * max F_l] floats
    int64_t hs_elems = 0;
    float *c0 = nullptr;          // corner-0 contributions (CC, levels >= 1), [3 * max F_l] floats
    int64_t c0_elems = 0;
    float *frame_c0 = nullptr;
    // last level >= 3 (CC): straddling edge-point groups of the grandparent edge kernel (Frames.gside)
    float *gside = nullptr, *frame_gside = nullptr;
    int32_t *gcnt = nullptr, *frame_gcnt = nullptr;
    int32_t gblk = 0;  // grandparent edge blocks
    void *scratch = nullptr;
    size_t scratch_bytes = 0;
    void *scratch_create = nullptr;
    size_t scratch_create_bytes = 0;
    // plan
    int scheme = -1, levels = -1;
    std::vector<LevelHost> lv;
    cudaGraphExec_t gexec = nullptr;
    int64_t graph_launches = 0;
    // kernel probe (alsub_probe): per-replay event pairs retargeted into the graph's two
    // event-record nodes, so one kernel is timed inside every replayed refine
    std::string probe_name;
    int probe_level = -2;
    std::vector<cudaEvent_t> probe_start, probe_stop;
    int32_t probe_next = 0;
    cudaEvent_t probe_cap[2] = {nullptr, nullptr};  // the events used at capture time
    cudaStream_t probe_stream = nullptr;
    cudaEvent_t probe_dep[3] = {nullptr, nullptr, nullptr};
    cudaGraph_t gtemplate = nullptr;                // kept while a probe is armed (node handles)
    cudaGraphNode_t probe_node[2] = {nullptr, nullptr};
    int64_t plan_runs = 0;  // refines run with the current plan (graph recorded from the 2nd on)
    cudaStream_t cap_stream = nullptr;
    cudaStream_t side_stream = nullptr;  // second branch for independent level kernels
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_build = nullptr, ev_aux = nullptr;
    int64_t last_launches = 0;
    // the last refined level's special lists (crease pairs / sigma of level L and the level-L rows
    // of the special-vertex table) are only read by exports and extraction: the refine skips their
    // inheritance step and ensure_last_lists() builds them on first use (lazy_lists = plan property,
    // lists_pending = not built since the last refine)
    bool lazy_lists = false;
    bool lists_pending = false;
    // refinement matrix R (NEXT-1): CSR rows of level rm_levels over the control vertices
    std::vector<std::pair<void *, size_t>> mem_rm;
    int32_t rm_levels = -1, rm_scheme = -1;
    int64_t rm_nnz = 0;
    int32_t *rm_row_off = nullptr;
    int2 *rm_ent = nullptr;
    // blocked form used by alsub_eval_frames_matrix (rmatrix.cu): chunk = owner face (c < F0) or
    // isolated control vertex (F0 + v); rows, support and dense weights per chunk
    int32_t rb_C = 0;
    int32_t *rb_row_off = nullptr, *rb_rows = nullptr, *rb_sup_off = nullptr, *rb_sup = nullptr;
    int64_t *rb_w_off = nullptr;
    float *rb_W = nullptr;
    int64_t rb_wlen = 0;
    float *rb_xt = nullptr;  // one batch of control positions [V0][3][32]
    // frames
    int frames_nb = 0;
    std::vector<float *> frame_buf;
    float *frame_hs = nullptr;
};

// ---------------- memory ----------------
static void *dev_alloc(alsub_mesh *m, size_t bytes, cudaStream_t s, std::vector<std::pair<void *, size_t>> &list) {
    if (bytes == 0) bytes = 16;
    bytes = (bytes + 255) & ~(size_t)255;
    void *p = nullptr;
    if (m->custom) {
        p = m->alloc.alloc(bytes, (void *)s, m->alloc.ctx);
    } else {
        if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
        }
    }
    if (p) list.emplace_back(p, bytes);
    return p;
}

static void free_list(alsub_mesh *m, std::vector<std::pair<void *, size_t>> &list, cudaStream_t s) {
    for (auto &pr : list) {
        if (m->custom) m->alloc.free(pr.first, pr.second, (void *)s, m->alloc.ctx);
        else cudaFreeAsync(pr.first, s);
    }
    list.clear();
}

template <class T>
static T *A(alsub_mesh *m, int64_t n, cudaStream_t s, std::vector<std::pair<void *, size_t>> &list, bool &ok) {
    T *p = (T *)dev_alloc(m, sizeof(T) * (size_t)(n > 0 ? n : 1), s, list);
    if (!p) ok = false;
    return p;
}

// ---------------- device views ----------------
static LevelDev dev_of(const LevelHost &L) {
    LevelDev p{};
    p.V = (int32_t)L.V; p.F = (int32_t)L.F; p.S = (int32_t)L.S; p.E = (int32_t)L.E; p.B = (int32_t)L.B;
    p.order = L.order;
    p.face_off = L.face_off; p.slot_face = L.slot_face;
    p.face_vtx = L.face_vtx; p.face_edge = L.face_edge; p.face_twin = L.face_twin; p.edge_hh = L.edge_hh;
    p.vtx_slot0 = L.vtx_slot0; p.bnd_word = L.bnd_word; p.bnd_wpre = L.bnd_wpre; p.loop_base = L.loop_base;
    p.sp = L.sp; p.nsp = (int32_t)L.nsp; p.sv_list = L.sv_list; p.nsv = (int32_t)L.nsv;
    p.spw = L.spw; p.spwpre = L.spwpre;
    return p;
}

static ChildDev child_of(const LevelHost &L) {
    ChildDev c{};
    c.V = (int32_t)L.V; c.F = (int32_t)L.F; c.S = (int32_t)L.S; c.E = (int32_t)L.E;
    c.face_vtx = L.face_vtx; c.face_edge = L.face_edge; c.face_twin = L.face_twin; c.edge_hh = L.edge_hh;
    c.vtx_slot0 = L.vtx_slot0; c.bnd_word = L.bnd_word; c.bnd_wpre = L.bnd_wpre;
    c.sp = L.sp; c.sv_list = L.sv_list; c.spw = L.spw; c.spwpre = L.spwpre;
    return c;
}

static void set_level0_view(alsub_mesh *m, LevelHost &L) {
    Build0 &b = m->b0;
    L.V = m->V0; L.F = m->F0; L.S = m->S0; L.E = m->E0; L.B = m->B0;
    L.order = m->order0;
    L.face_off = m->in_face_off; L.slot_face = b.slot_face;
    L.face_vtx = m->in_face_vtx; L.face_edge = b.face_edge; L.face_twin = b.face_twin;
    L.edge_hh = b.edge_hh; L.vtx_slot0 = b.vtx_slot0;
    L.bnd_word = b.bnd_word; L.bnd_wpre = b.bnd_wpre;
    L.sp = b.sp; L.nsp = m->K0; L.sv_list = b.sv_list; L.nsv = m->NSV0;
    L.spw = b.spw; L.spwpre = b.spwpre;
    L.pos = m->pos0;
}

// ---------------- create ----------------
static alsub_status map_flags(int32_t flags) {
    if (flags & kFlagMesh) return fail(ALSUB_E_MESH, "face order < 3, repeated vertex in a face, or vertex index out of range");
    if (flags & kFlagNonManifold) return fail(ALSUB_E_NONMANIFOLD, "non-manifold edge, inconsistent orientation or non-manifold vertex");
    if (flags & kFlagCrease) return fail(ALSUB_E_CREASE, "crease pair is not an edge, is duplicated, or has sigma < 0 / NaN");
    return ALSUB_OK;
}

static alsub_status create_impl(const int32_t *face_off, const int32_t *face_vtx, int32_t num_faces, const float *pos,
                                int32_t num_verts, const int32_t *crease_pairs, const float *crease_sigma,
                                int32_t num_creases, const alsub_allocator *alloc, void *stream, alsub_mesh **out,
                                bool lenient);

extern "C" alsub_status alsub_mesh_create(const int32_t *face_off, const int32_t *face_vtx, int32_t num_faces,
                                          const float *pos, int32_t num_verts, const int32_t *crease_pairs,
                                          const float *crease_sigma, int32_t num_creases,
                                          const alsub_allocator *alloc, void *stream, alsub_mesh **out) {
    return create_impl(face_off, face_vtx, num_faces, pos, num_verts, crease_pairs, crease_sigma, num_creases, alloc,
                       stream, out, false);
}

// lenient: crease pairs that are not edges are dropped instead of rejected (extracted meshes, R25)
static alsub_status create_impl(const int32_t *face_off, const int32_t *face_vtx, int32_t num_faces, const float *pos,
                                int32_t num_verts, const int32_t *crease_pairs, const float *crease_sigma,
                                int32_t num_creases, const alsub_allocator *alloc, void *stream, alsub_mesh **out,
                                bool lenient) {
    if (!out) return fail(ALSUB_E_ARG, "out is null");
    *out = nullptr;
    if (num_faces < 0 || num_verts < 0 || num_creases < 0) return fail(ALSUB_E_ARG, "negative count");
    if (!face_off || (num_verts > 0 && !pos)) return fail(ALSUB_E_ARG, "null face_off / pos");
    if (num_creases > 0 && (!crease_pairs || !crease_sigma)) return fail(ALSUB_E_ARG, "null crease arrays");
    cudaStream_t s = (cudaStream_t)stream;
    // face offsets on the host: S0, monotonicity, uniform order
    std::vector<int32_t> off((size_t)num_faces + 1);
    if (is_device_ptr(face_off)) {  // device-resident offsets: one read on the stream before the build
        CU(cudaMemcpyAsync(off.data(), face_off, sizeof(int32_t) * off.size(), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
    } else {
        std::memcpy(off.data(), face_off, sizeof(int32_t) * off.size());
    }
    if (off[0] != 0) return fail(ALSUB_E_MESH, "face_off[0] != 0");
    int order = -1;
    for (int32_t r = 0; r < num_faces; ++r) {
        int64_t c = (int64_t)off[r + 1] - off[r];
        if (c < 3) return fail(ALSUB_E_MESH, "face " + std::to_string(r) + " has order < 3");
        if (order == -1) order = (int)c;
        else if (order != c) order = 0;
    }
    if (order == -1) order = 4;
    if (order != 3 && order != 4) order = 0;
    const int32_t S0 = off[num_faces];
    if (S0 > 0 && !face_vtx) return fail(ALSUB_E_ARG, "null face_vtx");

    alsub_mesh *m = new alsub_mesh();
    if (alloc && alloc->alloc && alloc->free) { m->alloc = *alloc; m->custom = true; }
    cudaGetDevice(&m->device);
    m->V0 = num_verts; m->F0 = num_faces; m->S0 = S0; m->Kin = num_creases; m->order0 = order;
    auto bail = [&](alsub_status st) {
        std::string msg = g_err;
        alsub_mesh_destroy(m);
        g_err = msg;
        return st;
    };
    bool ok = true;
    auto &ML = m->mem_create;
    m->in_face_off = A<int32_t>(m, num_faces + 1, s, ML, ok);
    m->in_face_vtx = A<int32_t>(m, S0, s, ML, ok);
    m->pos0 = A<float>(m, 3 * (int64_t)num_verts, s, ML, ok);
    m->in_crease = A<int32_t>(m, 2 * (int64_t)num_creases, s, ML, ok);
    m->in_sigma = A<float>(m, num_creases, s, ML, ok);
    if (!ok) return bail(fail(ALSUB_E_NOMEM, "device allocation failed"));
    cudaMemcpyAsync(m->in_face_off, off.data(), sizeof(int32_t) * off.size(), cudaMemcpyHostToDevice, s);
    if (S0 > 0) cudaMemcpyAsync(m->in_face_vtx, face_vtx, sizeof(int32_t) * S0, cudaMemcpyDefault, s);
    if (num_verts > 0) cudaMemcpyAsync(m->pos0, pos, sizeof(float) * 3 * (size_t)num_verts, cudaMemcpyDefault, s);
    if (num_creases > 0) {
        cudaMemcpyAsync(m->in_crease, crease_pairs, sizeof(int32_t) * 2 * (size_t)num_creases, cudaMemcpyDefault, s);
        cudaMemcpyAsync(m->in_sigma, crease_sigma, sizeof(float) * (size_t)num_creases, cudaMemcpyDefault, s);
    }
    Build0 &b = m->b0;
    b.V = num_verts; b.F = num_faces; b.S = S0; b.K_in = num_creases; b.order = order;
    b.crease_lenient = lenient ? 1 : 0;
    b.face_off = m->in_face_off; b.face_vtx = m->in_face_vtx; b.crease_in = m->in_crease; b.sigma_in = m->in_sigma;
    b.slot_face = A<int32_t>(m, S0, s, ML, ok);
    b.vtx_slot = A<int32_t>(m, S0, s, ML, ok);
    b.vtx_off = A<int32_t>(m, (int64_t)num_verts + 1, s, ML, ok);
    b.vtx_cnt = A<int32_t>(m, (int64_t)num_verts + 1, s, ML, ok);
    b.edge_cnt = A<int32_t>(m, num_verts, s, ML, ok);
    b.edge_off = A<int32_t>(m, num_verts, s, ML, ok);
    b.face_edge = A<int32_t>(m, S0, s, ML, ok);
    b.face_twin = A<int32_t>(m, S0, s, ML, ok);
    b.vtx_slot0 = A<int32_t>(m, num_verts, s, ML, ok);
    b.vbnd = A<int32_t>(m, num_verts, s, ML, ok);
    b.vtx_cur = A<int32_t>(m, num_verts, s, ML, ok);
    b.flags = A<int32_t>(m, 8, s, ML, ok);
    b.scalars = A<int32_t>(m, 8, s, ML, ok);
    b.long_list = A<int32_t>(m, num_verts, s, ML, ok);
    b.long_keys = A<uint64_t>(m, 4 * (int64_t)S0, s, ML, ok);
    b.nlong = -1;
    m->scratch_bytes = build0_scratch_bytes(num_verts, S0);
    m->scratch = dev_alloc(m, m->scratch_bytes, s, ML);
    b.scratch = m->scratch;
    m->scratch_create = m->scratch;
    m->scratch_create_bytes = m->scratch_bytes;
    if (!ok || !m->scratch) return bail(fail(ALSUB_E_NOMEM, "device allocation failed"));
    cudaMemsetAsync(b.flags, 0, 8 * sizeof(int32_t), s);
    cudaMemsetAsync(b.scalars, 0, 8 * sizeof(int32_t), s);
    init_scheme_tables(s);
    Launches L;
    // The whole level-0 build runs before the one host read: the edge arrays are sized by the
    // upper bound E_0 <= S_0 (every edge has a slot), the kernels that need E_0 read it from the
    // device, and the validation flags, E_0 and the special-list sizes come back together.  The
    // kernels are memory-safe on invalid input (out-of-range ids never become edges); the flags
    // then turn the whole create into an error.
    const int32_t Emax = std::max<int32_t>(S0, 1);
    const int64_t nw = ceil_div(Emax, 32);
    b.edge_hh = A<int2>(m, Emax, s, ML, ok);
    b.bnd_word = A<uint32_t>(m, nw, s, ML, ok);
    b.bnd_wcnt = A<int32_t>(m, nw, s, ML, ok);
    b.bnd_wpre = A<int32_t>(m, nw, s, ML, ok);
    b.edge_sigma = A<float>(m, Emax, s, ML, ok);
    b.edge_cidx = A<int32_t>(m, Emax, s, ML, ok);
    b.sp_flag = A<int32_t>(m, Emax, s, ML, ok);
    b.sp_off = A<int32_t>(m, Emax, s, ML, ok);
    b.sp = A<SpEdge>(m, Emax, s, ML, ok);
    b.sv_vtx = A<int32_t>(m, num_verts, s, ML, ok);
    b.sv_off = A<int32_t>(m, (int64_t)num_verts + 1, s, ML, ok);
    b.sv_cnt = A<int32_t>(m, num_verts, s, ML, ok);
    b.sv_list = A<int32_t>(m, 2 * (int64_t)Emax, s, ML, ok);
    b.spw = A<uint32_t>(m, nw, s, ML, ok);
    b.spwpre = A<int32_t>(m, nw, s, ML, ok);
    m->sv_vtx = m->sv_vtx_create = b.sv_vtx;
    m->sv_off = m->sv_off_create = b.sv_off;
    if (!ok) return bail(fail(ALSUB_E_NOMEM, "device allocation failed"));
    build0_validate(b, s, L);     // a1: validation + M^T row lengths
    build0_count_edges(b, s, L);  // a2 + symbolic a3 -> E_0 on the device
    b.E = Emax;
    build0_fill(b, true, s, L);   // numeric a3, crease matrix, special lists
    int32_t flags = 0, sc[8];
    cudaMemcpyAsync(&flags, b.flags, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(sc, b.scalars, sizeof(sc), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess)  // the create's one host synchronisation
        return bail(fail(ALSUB_E_CUDA, std::string("level-0 build: ") + cudaGetErrorString(cudaGetLastError())));
    if (flags) return bail(map_flags(flags));
    m->E0 = sc[0];
    b.E = sc[0];
    m->B0 = sc[1];
    m->K0 = sc[2];
    m->NSV0 = sc[3];
    b.nlong = sc[5];
    m->user_creases = (m->K0 - m->B0) > 0;
    b.no_special = m->K0 == 0 && m->B0 == 0;
    CU(cudaStreamCreateWithFlags(&m->cap_stream, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&m->side_stream, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&m->ev_fork, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&m->ev_join, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&m->ev_build, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&m->ev_aux, cudaEventDisableTiming));
    m->last_launches = L.n;
    *out = m;
    g_err.clear();
    return ALSUB_OK;
}

extern "C" alsub_status alsub_set_positions(alsub_mesh *m, const float *pos, void *stream) {
    if (!m || (!pos && m->V0 > 0)) return fail(ALSUB_E_ARG, "null argument");
    if (m->V0 > 0)
        CU(cudaMemcpyAsync(m->pos0, pos, sizeof(float) * 3 * (size_t)m->V0, cudaMemcpyDefault, (cudaStream_t)stream));
    return ALSUB_OK;
}

// ---------------- plan ----------------
static void drop_graph(alsub_mesh *m) {
    if (m->gexec) { cudaGraphExecDestroy(m->gexec); m->gexec = nullptr; }
    if (m->gtemplate) { cudaGraphDestroy(m->gtemplate); m->gtemplate = nullptr; }
    m->probe_node[0] = m->probe_node[1] = nullptr;
}

static void free_plan(alsub_mesh *m, cudaStream_t s) {
    drop_graph(m);
    // the refinement matrix indexes the plan's levels: it dies with the plan
    free_list(m, m->mem_rm, s);
    m->rm_levels = -1;
    free_list(m, m->mem_plan, s);
    free_list(m, m->mem_frames, s);
    m->scratch = m->scratch_create;
    m->scratch_bytes = m->scratch_create_bytes;
    m->sv_vtx = m->b0.sv_vtx = m->sv_vtx_create;
    m->sv_off = m->b0.sv_off = m->sv_off_create;
    m->b0.scratch = m->scratch;
    m->frame_buf.clear();
    m->frames_nb = 0;
    m->lv.clear();
    m->scheme = m->levels = -1;
}

static alsub_status check_scheme(alsub_mesh *m, int scheme) {
    if (scheme == ALSUB_LOOP || scheme == ALSUB_SQRT3) {
        if (m->order0 != 3) return fail(ALSUB_E_SCHEME, "Loop and sqrt3 need a triangle mesh");
    }
    if (scheme == ALSUB_SQRT3) {
        if (m->B0 > 0) return fail(ALSUB_E_SCHEME, "sqrt3 boundary rules are omitted by the paper (P:L1002)");
        if (m->user_creases) return fail(ALSUB_E_SCHEME, "sqrt3 has no crease rules");
    }
    return ALSUB_OK;
}

static alsub_status make_plan(alsub_mesh *m, int scheme, int levels, cudaStream_t s) {
    free_plan(m, s);
    std::vector<LevelHost> lv((size_t)levels + 1);
    set_level0_view(m, lv[0]);
    const bool special = scheme != ALSUB_SQRT3 && m->K0 > 0;
    for (int l = 1; l <= levels; ++l) {
        const LevelHost &p = lv[l - 1];
        LevelHost &c = lv[l];
        if (scheme == ALSUB_CATMULL_CLARK) {
            c.V = p.V + p.F + p.E; c.F = p.S; c.S = 4 * p.S; c.E = 2 * p.E + p.S; c.B = 2 * p.B; c.order = 4;
        } else if (scheme == ALSUB_LOOP) {
            c.V = p.V + p.E; c.F = 4 * p.F; c.S = 12 * p.F; c.E = 2 * p.E + 3 * p.F; c.B = 2 * p.B; c.order = 3;
        } else {
            c.V = p.V + p.F; c.F = 3 * p.F; c.S = 9 * p.F; c.E = 3 * p.E; c.B = 0; c.order = 3;
            c.edges_valid = false;
        }
        if (c.V > INT32_MAX || c.S > INT32_MAX || c.E > INT32_MAX || 4 * c.S > INT32_MAX)
            return fail(ALSUB_E_OVERFLOW, "level " + std::to_string(l) + " exceeds int32 ids");
        if (special) {
            c.nsp = 2 * p.nsp;
            c.nsv = p.nsv + p.nsp;
            if (2 * c.nsp > INT32_MAX || c.nsv > INT32_MAX) return fail(ALSUB_E_OVERFLOW, "special lists exceed int32");
        }
    }
    bool ok = true;
    auto &ML = m->mem_plan;
    const int64_t sv_total = std::max<int64_t>(m->V0, special ? lv[levels].nsv : 0) + 1;
    m->sv_vtx = A<int32_t>(m, sv_total, s, ML, ok);
    m->sv_off = A<int32_t>(m, sv_total, s, ML, ok);
    m->hs_elems = 0;
    if (scheme == ALSUB_CATMULL_CLARK)
        for (int l = 2; l + 1 < levels; ++l) m->hs_elems = std::max<int64_t>(m->hs_elems, 3 * lv[l].F);
    m->hs = m->hs_elems ? A<float>(m, m->hs_elems, s, ML, ok) : nullptr;
    m->c0_elems = 0;
    if (scheme == ALSUB_CATMULL_CLARK)
        for (int l = 1; l < levels; ++l) m->c0_elems = std::max<int64_t>(m->c0_elems, 3 * lv[l].F);
    m->c0 = m->c0_elems ? A<float>(m, m->c0_elems, s, ML, ok) : nullptr;
    m->gblk = 0;
    m->gside = nullptr;
    m->gcnt = nullptr;
    if (scheme == ALSUB_CATMULL_CLARK && levels >= 4) {  // compact c0 + straddling groups (cc.cu)
        m->gblk = (int32_t)grid_for(lv[levels - 2].E);
        m->gside = A<float>(m, 12 * (int64_t)m->gblk, s, ML, ok);
        m->gcnt = A<int32_t>(m, m->gblk, s, ML, ok);
        // zero once: the block that finishes a straddling group resets its counter
        if (m->gcnt) cudaMemsetAsync(m->gcnt, 0, sizeof(int32_t) * m->gblk, s);
    }
    m->b0.sv_vtx = m->sv_vtx;
    m->b0.sv_off = m->sv_off;
    int64_t max_scan = std::max<int64_t>(m->V0, m->S0) + 1;
    for (int l = 0; l <= levels; ++l) {
        LevelHost &c = lv[l];
        const bool has_child = l < levels;   // level l is refined
        const bool adj = l + 1 < levels;     // child needs adjacency
        if (l >= 1) {
            c.face_vtx = A<int32_t>(m, c.S, s, ML, ok);
            c.pos = A<float>(m, 3 * c.V, s, ML, ok);
            if (has_child) {
                // CC consumes a level's twins only to emit the adjacency of ITS child (adj)
                if (scheme != ALSUB_CATMULL_CLARK || adj) c.face_twin = A<int32_t>(m, c.S, s, ML, ok);
                // CC, levels >= 3: the last refined level recomputes its edge rows and iterates its
                // parent's edges (cc.cu), so its face_edge / edge pairs are never stored
                const bool last_cc = scheme == ALSUB_CATMULL_CLARK && levels >= 3 && l == levels - 1;
                if (scheme != ALSUB_SQRT3 && !last_cc) {
                    c.face_edge = A<int32_t>(m, c.S, s, ML, ok);
                    c.edge_hh = A<int2>(m, c.E, s, ML, ok);
                }
                if (scheme == ALSUB_CATMULL_CLARK && c.B > 0) {
                    const int64_t nw = ceil_div(c.E, 32);
                    c.bnd_word = A<uint32_t>(m, nw, s, ML, ok);
                    c.bnd_wpre = A<int32_t>(m, nw, s, ML, ok);
                }
            }
            if (special) {
                c.sp = A<SpEdge>(m, c.nsp, s, ML, ok);
                c.sv_list = A<int32_t>(m, 2 * c.nsp, s, ML, ok);
                if (scheme == ALSUB_CATMULL_CLARK && has_child) {
                    c.spw = A<uint32_t>(m, ceil_div(c.E, 32), s, ML, ok);
                    c.spwpre = A<int32_t>(m, ceil_div(c.E, 32), s, ML, ok);
                }
            }
        }
        if (scheme == ALSUB_LOOP && has_child && (adj || special)) {
            c.loop_stat = A<int32_t>(m, (int64_t)(scan_scratch_bytes(c.E) / 4), s, ML, ok);
            c.loop_base = A<int32_t>(m, c.E, s, ML, ok);
        }
    }
    size_t need = std::max(build0_scratch_bytes(m->V0, m->S0), scan_scratch_bytes(max_scan));
    if (need > m->scratch_bytes) {
        void *p = dev_alloc(m, need, s, ML);
        if (!p) ok = false;
        m->scratch = p;
        m->scratch_bytes = need;
        m->b0.scratch = p;
    }
    if (!ok) {
        free_plan(m, s);
        return fail(ALSUB_E_NOMEM, "device allocation failed for the level tables");
    }
    m->lv = std::move(lv);
    m->plan_runs = 0;
    m->scheme = scheme;
    m->levels = levels;
    return ALSUB_OK;
}

// ---------------- the level loop ----------------
constexpr int64_t kFuseCreaseMaxV = 1 << 20;  // levels below this fuse the crease module
// vertex-id segments of sqrt3 level l: [V0 | F0 | F1 | ... | F_{l-1}]
static VSegs make_segs_s3(alsub_mesh *m, int l) {
    VSegs g{};
    g.level = l;
    g.hs_seg = -1;
    int n = 0;
    int32_t mult = 1;
    for (int k = 0; k < l; ++k) mult *= 3;
    g.start[n] = 0; g.len[n] = m->V0; g.type[n] = 0; g.birth[n] = 0; g.mult[n] = mult; ++n;
    for (int k = 1; k <= l; ++k) {
        const LevelHost &q = m->lv[k - 1];
        mult /= 3;
        g.start[n] = (int32_t)q.V; g.len[n] = (int32_t)q.F; g.type[n] = 1; g.birth[n] = (int8_t)k; g.mult[n] = mult;
        g.fvx[k - 1] = q.face_vtx;
        g.ftw[k - 1] = q.face_twin;
        ++n;
    }
    g.nseg = n;
    g.vtx_off0 = m->b0.vtx_off; g.vtx_list0 = m->b0.vtx_slot; g.face_off0 = m->in_face_off;
    g.long_list = m->b0.long_list; g.nlong = std::max(m->b0.nlong, 0);
    g.slot_face0 = m->b0.slot_face; g.vbnd0 = m->b0.vbnd;
    return g;
}

// vertex-id segments of Loop level l: [V0 | E_0 | ... | E_{l-1}] (edge points born at level k + 1
// from the level-k edge pairs)
static VSegs make_segs_loop(alsub_mesh *m, int l) {
    VSegs g{};
    g.level = l;
    g.hs_seg = -1;
    int n = 0;
    g.start[n] = 0; g.len[n] = m->V0; g.type[n] = 0; g.birth[n] = 0; ++n;
    for (int k = 1; k <= l; ++k) {
        const LevelHost &q = m->lv[k - 1];
        g.start[n] = (int32_t)q.V; g.len[n] = (int32_t)q.E; g.type[n] = 2; g.birth[n] = (int8_t)k;
        g.ehh[k - 1] = q.edge_hh;
        ++n;
    }
    g.nseg = n;
    g.vtx_off0 = m->b0.vtx_off; g.vtx_list0 = m->b0.vtx_slot; g.face_off0 = m->in_face_off;
    g.long_list = m->b0.long_list; g.nlong = std::max(m->b0.nlong, 0);
    g.slot_face0 = m->b0.slot_face; g.vbnd0 = m->b0.vbnd;
    return g;
}

// vertex-id segments of CC level l (see VSegs in internal.h)
static VSegs make_segs(alsub_mesh *m, int l) {
    VSegs g{};
    g.level = l;
    int n = 0;
    g.start[n] = 0; g.len[n] = m->V0; g.type[n] = 0; g.birth[n] = 0; ++n;
    for (int k = 1; k <= l; ++k) {
        const LevelHost &q = m->lv[k - 1];
        // face points born at this level (k == l >= 2) are smoothed inside the face kernel
        g.start[n] = (int32_t)q.V; g.len[n] = (k == l && l >= 2) ? 0 : (int32_t)q.F; g.type[n] = 1;
        g.birth[n] = (int8_t)k; ++n;
        g.start[n] = (int32_t)(q.V + q.F); g.len[n] = (int32_t)q.E; g.type[n] = 2; g.birth[n] = (int8_t)k; ++n;
        g.ehh[k - 1] = q.edge_hh;
        g.spw[k - 1] = q.spw;
        g.spwpre[k - 1] = q.spwpre;
        g.nsvb[k - 1] = (int32_t)q.nsv;
        g.bw[k - 1] = q.B > 0 ? q.bnd_word : nullptr;
        g.bwp[k - 1] = q.B > 0 ? q.bnd_wpre : nullptr;
    }
    g.nseg = n;
    g.hs_seg = l >= 2 ? n - 1 : -1;  // the last segment = edge points born at level l
    g.vtx_off0 = m->b0.vtx_off; g.vtx_list0 = m->b0.vtx_slot; g.face_off0 = m->in_face_off;
    g.long_list = m->b0.long_list; g.nlong = std::max(m->b0.nlong, 0);
    g.slot_face0 = m->b0.slot_face; g.vbnd0 = m->b0.vbnd;
    return g;
}

// CC levels whose edge kernel iterates the grandparent edges (k_cc_edge_gp, cc.cu): the last
// refined level (its edge pairs are never stored) and, when it is level 3 or later and its crease
// rules are not fused, the level before it (it then also writes the boundary words of the last
// level; ALSUB_NO_GP_MID=1 keeps k_cc_edge there, for A/B runs)
static bool cc_use_gp(const alsub_mesh *m, int l, bool special) {
    static const bool mid_off = [] {
        const char *e = getenv("ALSUB_NO_GP_MID");
        return e && e[0] == '1';
    }();
    const LevelHost &P = m->lv[l];
    if (l < 2) return false;
    if (P.edge_hh == nullptr) return true;
    return !mid_off && l >= 3 && l == m->levels - 2 && m->gside && !(special && P.V < kFuseCreaseMaxV);
}

// NVTX range (eager launches; `ncu --nvtx --nvtx-include "alsub level 5->6/"` selects a level)
struct Nvtx {
    Nvtx(const char *fmt, int a, int b) {
        char buf[64];
        snprintf(buf, sizeof buf, fmt, a, b);
        nvtxRangePushA(buf);
    }
    ~Nvtx() { nvtxRangePop(); }
};

// build the last refined level's special lists (inheritance half of the crease module only: no
// position writes, nb = 0) if the refine skipped them
static void ensure_last_lists(alsub_mesh *m, cudaStream_t s) {
    if (!m->lists_pending || m->levels < 1) return;
    const int l = m->levels - 1;
    LevelHost &P = m->lv[l];
    LevelDev p = dev_of(P);
    p.sv_vtx = m->sv_vtx;
    p.sv_off = m->sv_off;
    p.inherit = 1;
    ChildDev c = child_of(m->lv[l + 1]);
    c.sv_vtx = m->sv_vtx;
    c.sv_off = m->sv_off;
    Frames fr{nullptr, nullptr, 0, 0, 0, nullptr, 0};
    Launches L;
    const bool cc = m->scheme == ALSUB_CATMULL_CLARK;
    crease_level(p, c, fr, cc ? (int32_t)(P.V + P.F) : (int32_t)P.V, cc ? 0 : 1, true, s, L);
    m->lists_pending = false;
}

static void enqueue_refine(alsub_mesh *m, cudaStream_t s, Launches &L) {
    const int scheme = m->scheme, levels = m->levels;
    m->lazy_lists = false;
    L.side = m->side_stream;
    L.ev_fork = m->ev_fork;
    L.ev_join = m->ev_join;
    L.ev_aux = m->ev_aux;
    // CC with levels: the build's special-list branch stays open into level 0 (cc.cu joins it)
    L.ev_build = (scheme == ALSUB_CATMULL_CLARK && levels > 0) ? m->ev_build : nullptr;
    // a1-a3: level-0 mesh matrix, M^T by counting sort, edge index, creases
    L.level = -1;
    nvtxRangePushA("alsub level-0 build");
    {
        ZeroSegs z;
        build0_zero_segments(m->b0, z);
        for (int l = 1; l < levels; ++l) {  // child boundary / special words (atomicOr targets of the edge kernels)
            if (m->lv[l].bnd_word) z.add(m->lv[l].bnd_word, ceil_div(m->lv[l].E > 0 ? m->lv[l].E : 1, 32));
            if (m->lv[l].spw) z.add(m->lv[l].spw, ceil_div(m->lv[l].E > 0 ? m->lv[l].E : 1, 32));
        }
        for (int l = 0; l < levels; ++l)  // Loop child-edge base scans: status words
            if (m->lv[l].loop_stat) z.add(m->lv[l].loop_stat, (int64_t)(scan_scratch_bytes(m->lv[l].E) / 4));
        zero_segments(z, s, L);
    }
    build0_validate(m->b0, s, L);
    build0_count_edges(m->b0, s, L);
    build0_fill(m->b0, false, s, L);
    nvtxRangePop();
    const bool special = scheme != ALSUB_SQRT3 && m->K0 > 0;
    for (int l = 0; l < levels; ++l) {
        LevelHost &P = m->lv[l];
        LevelHost &C = m->lv[l + 1];
        const bool adj = l + 1 < levels;
        L.level = l;
        Nvtx range_level("alsub level %d->%d", l, l + 1);
        LevelDev p = dev_of(P);
        p.sv_vtx = m->sv_vtx;
        p.sv_off = m->sv_off;
        p.inherit = 1;
        ChildDev c = child_of(C);
        c.sv_vtx = m->sv_vtx;
        c.sv_off = m->sv_off;
        Frames fr{P.pos, C.pos, 3 * P.V, 3 * C.V, 1, m->hs, 0, l >= 1 ? m->c0 : nullptr, 0};
        if (scheme == ALSUB_CATMULL_CLARK) {
            VSegs g = make_segs(m, l);
            LevelDev gp{};
            const bool use_gp = cc_use_gp(m, l, special);
            if (use_gp) {
                gp = dev_of(m->lv[l - 1]);
                g.len[g.hs_seg] = 0;  // the edge kernel smooths the edge points born at level l
                fr.hs = nullptr;      // so the face kernel writes no half sums
            }
            // crease module fused into the level kernels on small levels (the latency of a separate
            // pass dominates there), a separate kernel on large ones (fusion costs occupancy)
            p.crease = (special && !use_gp && P.V < kFuseCreaseMaxV) ? 1 : 0;
            if (use_gp && l >= 3 && m->gside) {  // compact corner sums + straddling groups
                fr.c0shift = 2;
                fr.gside = m->gside;
                fr.gcnt = m->gcnt;
                fr.gsidestride = 12 * (int64_t)m->gblk;
            }
            cc_level(p, c, fr, true, adj, g, use_gp ? &gp : nullptr, s, L);
            if (special && !p.crease) {
                if (!adj) m->lazy_lists = true;  // last level: lists built on demand
                crease_level(p, c, fr, (int32_t)(P.V + P.F), 0, adj, s, L);
            }
        } else if (scheme == ALSUB_LOOP) {
            VSegs g = make_segs_loop(m, l);
            if (special && !adj) m->lazy_lists = true;
            loop_level(p, c, fr, true, adj, P.loop_stat, (adj || special) ? P.loop_base : nullptr, g, s, L,
                       special ? (adj ? 1 : 0) : -1);
        } else {
            VSegs g = make_segs_s3(m, l);
            sqrt3_level(p, c, fr, true, adj, g, s, L);
        }
    }
}

static bool graphs_enabled() {
    const char *e = getenv("ALSUB_NO_GRAPH");
    return !(e && e[0] == '1');
}

extern "C" alsub_status alsub_refine(alsub_mesh *m, alsub_scheme scheme, int32_t levels, void *stream) {
    if (!m) return fail(ALSUB_E_ARG, "null mesh");
    if (scheme < ALSUB_CATMULL_CLARK || scheme > ALSUB_SQRT3) return fail(ALSUB_E_ARG, "unknown scheme");
    if (levels < 0 || levels > 16) return fail(ALSUB_E_ARG, "levels must be in [0, 16]");
    alsub_status st = check_scheme(m, scheme);
    if (st != ALSUB_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if (m->scheme != scheme || m->levels != levels) {
        st = make_plan(m, scheme, levels, s);
        if (st != ALSUB_OK) return st;
    }
    Launches L;
    const bool use_graph = graphs_enabled() && m->plan_runs >= 1;  // one-shot refines run eagerly
    m->plan_runs++;
    if (use_graph) {
        if (!m->gexec) {
            // the plan's allocations are stream-ordered on `s`: make the capture stream wait for them
            cudaEvent_t ev;
            CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            CU(cudaEventRecord(ev, s));
            CU(cudaStreamWaitEvent(m->cap_stream, ev, 0));
            CU(cudaStreamSynchronize(m->cap_stream));
            cudaEventDestroy(ev);
            cudaGraph_t g;
            const bool probe = !m->probe_start.empty();
            if (probe) {
                L.probe_name = m->probe_name.c_str();
                L.probe_level = m->probe_level;
                L.probe_ev[0] = m->probe_cap[0];
                L.probe_ev[1] = m->probe_cap[1];
                L.probe_stream = m->probe_stream;
                for (int k = 0; k < 3; ++k) L.probe_dep[k] = m->probe_dep[k];
            }
            CU(cudaStreamBeginCapture(m->cap_stream, cudaStreamCaptureModeThreadLocal));
            enqueue_refine(m, m->cap_stream, L);
            if (L.probe_hit) {  // join the probe branch
                cudaEventRecord(L.probe_dep[2], L.probe_stream);
                cudaStreamWaitEvent(m->cap_stream, L.probe_dep[2], 0);
            }
            cudaError_t ce = cudaStreamEndCapture(m->cap_stream, &g);
            if (ce != cudaSuccess) return fail(ALSUB_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
            ce = cudaGraphInstantiate(&m->gexec, g, 0);
            if (ce != cudaSuccess) {
                cudaGraphDestroy(g);
                m->gexec = nullptr;
                return fail(ALSUB_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
            }
            if (probe && L.probe_hit) {
                // the two event-record nodes of the probe, to retarget per replay
                size_t nn = 0;
                CU(cudaGraphGetNodes(g, nullptr, &nn));
                std::vector<cudaGraphNode_t> nodes(nn);
                CU(cudaGraphGetNodes(g, nodes.data(), &nn));
                for (cudaGraphNode_t nd : nodes) {
                    cudaGraphNodeType ty;
                    CU(cudaGraphNodeGetType(nd, &ty));
                    if (ty != cudaGraphNodeTypeEventRecord) continue;
                    cudaEvent_t ev;
                    CU(cudaGraphEventRecordNodeGetEvent(nd, &ev));
                    if (ev == m->probe_cap[0]) m->probe_node[0] = nd;
                    if (ev == m->probe_cap[1]) m->probe_node[1] = nd;
                }
                m->gtemplate = g;
            } else {
                cudaGraphDestroy(g);
            }
            m->graph_launches = L.n;
        }
        if (m->probe_node[0] && m->probe_node[1] && m->probe_next < (int32_t)m->probe_start.size()) {
            const int32_t i = m->probe_next++;
            CU(cudaGraphExecEventRecordNodeSetEvent(m->gexec, m->probe_node[0], m->probe_start[i]));
            CU(cudaGraphExecEventRecordNodeSetEvent(m->gexec, m->probe_node[1], m->probe_stop[i]));
        }
        CU(cudaGraphLaunch(m->gexec, s));
        m->last_launches = m->graph_launches;
    } else {
        enqueue_refine(m, s, L);
        m->last_launches = L.n;
    }
    m->lists_pending = m->lazy_lists;
    CU(cudaGetLastError());
    return ALSUB_OK;
}

extern "C" alsub_status alsub_refine_profile(alsub_mesh *m, alsub_scheme scheme, int32_t levels, void *stream,
                                             alsub_kernel_time *out, int32_t cap, int32_t *n_out) {
    if (!m || (cap > 0 && !out)) return fail(ALSUB_E_ARG, "null argument");
    if (scheme < ALSUB_CATMULL_CLARK || scheme > ALSUB_SQRT3) return fail(ALSUB_E_ARG, "unknown scheme");
    if (levels < 0 || levels > 16) return fail(ALSUB_E_ARG, "levels must be in [0, 16]");
    alsub_status st = check_scheme(m, scheme);
    if (st != ALSUB_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if (m->scheme != scheme || m->levels != levels) {
        st = make_plan(m, scheme, levels, s);
        if (st != ALSUB_OK) return st;
    }
    Launches L;
    L.timing = true;
    cudaEvent_t start;
    CU(cudaEventCreate(&start));
    CU(cudaEventRecord(start, s));
    enqueue_refine(m, s, L);
    CU(cudaStreamSynchronize(s));
    CU(cudaGetLastError());
    const int32_t n = (int32_t)L.ev.size();
    cudaEvent_t prev = start;
    for (int32_t i = 0; i < n; ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, prev, L.ev[i]);
        if (i < cap) {
            memset(out[i].name, 0, sizeof(out[i].name));
            strncpy(out[i].name, L.name[i], sizeof(out[i].name) - 1);
            out[i].level = L.lvl[i];
            out[i].ms = ms;
        }
        prev = L.ev[i];
    }
    for (auto e : L.ev) cudaEventDestroy(e);
    cudaEventDestroy(start);
    if (n_out) *n_out = n;
    m->last_launches = L.n;
    m->lists_pending = m->lazy_lists;
    return ALSUB_OK;
}

// ---------------- queries / export ----------------
static const LevelHost *level_of(const alsub_mesh *m, int32_t level) {
    if (level == 0 && m->lv.empty()) return nullptr;
    if (level < 0 || level >= (int32_t)m->lv.size()) return nullptr;
    return &m->lv[level];
}

extern "C" alsub_status alsub_level_counts(const alsub_mesh *m, int32_t level, alsub_counts *out) {
    if (!m || !out) return fail(ALSUB_E_ARG, "null argument");
    memset(out, 0, sizeof(*out));
    if (level == 0) {
        out->verts = m->V0; out->faces = m->F0; out->edges = m->E0; out->boundary_edges = m->B0;
        out->face_slots = m->S0; out->creases_upper_bound = m->K0; out->face_order = m->order0;
        out->edges_valid = 1;
        return ALSUB_OK;
    }
    const LevelHost *L = level_of(m, level);
    if (!L) return fail(ALSUB_E_ARG, "level not built (call alsub_refine first)");
    out->verts = L->V; out->faces = L->F; out->edges = L->E; out->boundary_edges = L->B; out->face_slots = L->S;
    out->creases_upper_bound = L->nsp; out->face_order = L->order;
    out->edges_valid = (L->edges_valid && level < m->levels) ? 1 : 0;
    return ALSUB_OK;
}

__global__ void k_iota_stride(int32_t *o, int64_t n, int32_t c) {
    ALSUB_GRID_WAIT();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) o[i] = (int32_t)(c * i);
}

// copy `bytes` from device src to dst (host or device)
static cudaError_t copy_out(void *dst, const void *src, size_t bytes, cudaStream_t s) {
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s);
}

extern "C" alsub_status alsub_level_topology(const alsub_mesh *mc, int32_t level, int32_t *face_vtx, int32_t *face_off,
                                             int32_t *edge_vtx, int32_t *edge_face, int32_t *crease_pairs,
                                             float *crease_sigma, int32_t *num_creases, void *stream) {
    alsub_mesh *m = const_cast<alsub_mesh *>(mc);
    if (!m) return fail(ALSUB_E_ARG, "null mesh");
    cudaStream_t s = (cudaStream_t)stream;
    LevelHost l0;
    const LevelHost *L;
    if (m->lv.empty()) {
        if (level != 0) return fail(ALSUB_E_ARG, "level not built (call alsub_refine first)");
        set_level0_view(m, l0);
        L = &l0;
    } else {
        L = level_of(m, level);
        if (!L) return fail(ALSUB_E_ARG, "level out of range");
    }
    std::vector<std::pair<void *, size_t>> tmp;
    bool ok = true;
    Launches Ln;
    if (face_vtx) CU(copy_out(face_vtx, L->face_vtx, sizeof(int32_t) * (size_t)L->S, s));
    if (face_off) {
        if (level == 0) {
            CU(copy_out(face_off, m->in_face_off, sizeof(int32_t) * ((size_t)L->F + 1), s));
        } else {
            int32_t *d = is_device_ptr(face_off) ? face_off : A<int32_t>(m, L->F + 1, s, tmp, ok);
            if (!ok) return fail(ALSUB_E_NOMEM, "export buffer");
            launch(Ln, "iota", k_iota_stride, dim3(grid_for(L->F + 1)), dim3(kThreads), 0, s, d, (int64_t)(L->F + 1), (int32_t)L->order);
            if (d != face_off) CU(copy_out(face_off, d, sizeof(int32_t) * ((size_t)L->F + 1), s));
        }
    }
    if (edge_vtx || edge_face) {
        const bool rebuild = L->edge_hh == nullptr && m->scheme == ALSUB_CATMULL_CLARK && level >= 2 &&
                             level < m->levels;
        const bool have = L->edges_valid && (level == 0 || level < m->levels) && (L->edge_hh || rebuild);
        if (!have) { free_list(m, tmp, s); return fail(ALSUB_E_ARG, "edge tables are not kept for this level"); }
        LevelHost Lx = *L;
        if (rebuild) {
            // re-emit the edge pairs of this (last refined) level with the parent's topology kernels,
            // into scratch copies of everything those kernels write (face rows, boundary words and
            // prefixes), so the live tables of the handle are only read (a const export
            // must not race a replay on another stream)
            const int64_t nwx = ceil_div(L->E > 0 ? L->E : 1, 32);
            Lx.edge_hh = A<int2>(m, L->E, s, tmp, ok);
            Lx.face_vtx = A<int32_t>(m, L->S, s, tmp, ok);
            if (L->bnd_word) {
                Lx.bnd_word = A<uint32_t>(m, nwx, s, tmp, ok);
                Lx.bnd_wpre = A<int32_t>(m, nwx, s, tmp, ok);
            }
            if (!ok) { free_list(m, tmp, s); return fail(ALSUB_E_NOMEM, "export buffer"); }
            const LevelHost &Pp = m->lv[level - 1];
            LevelDev pd = dev_of(Pp);
            ChildDev cd = child_of(Lx);
            cd.face_edge = nullptr;
            cd.face_twin = nullptr;
            Frames fr0{nullptr, nullptr, 0, 0, 0, nullptr, 0};
            if (Lx.bnd_word) CU(cudaMemsetAsync(Lx.bnd_word, 0, sizeof(uint32_t) * ceil_div(Lx.E, 32), s));
            VSegs g = make_segs(m, level - 1);
            cc_level(pd, cd, fr0, true, true, g, nullptr, s, Ln);
        }
        L = &Lx;
        int32_t *dv = edge_vtx && !is_device_ptr(edge_vtx) ? A<int32_t>(m, 2 * L->E, s, tmp, ok) : edge_vtx;
        int32_t *df = edge_face && !is_device_ptr(edge_face) ? A<int32_t>(m, 2 * L->E, s, tmp, ok) : edge_face;
        if (!ok) return fail(ALSUB_E_NOMEM, "export buffer");
        export_edges(dev_of(*L), dv, df, s, Ln);
        if (dv != edge_vtx) CU(copy_out(edge_vtx, dv, sizeof(int32_t) * 2 * (size_t)L->E, s));
        if (df != edge_face) CU(copy_out(edge_face, df, sizeof(int32_t) * 2 * (size_t)L->E, s));
    }
    if (crease_pairs || crease_sigma || num_creases) {
        if (level == m->levels) ensure_last_lists(m, s);
        int32_t cnt = (int32_t)L->nsp;
        std::vector<SpEdge> sp;
        if (L->sp && cnt > 0) {
            sp.resize((size_t)cnt);
            CU(cudaMemcpyAsync(sp.data(), L->sp, sizeof(SpEdge) * cnt, cudaMemcpyDeviceToHost, s));
            CU(cudaStreamSynchronize(s));
        }
        std::vector<int32_t> pairs;
        std::vector<float> sig;
        for (const SpEdge &e : sp) {
            if ((e.flags & kSpBoundary) || !(e.sigma > 0.0f)) continue;
            pairs.push_back(e.a);
            pairs.push_back(e.b);
            sig.push_back(e.sigma);
        }
        int32_t k = (int32_t)sig.size();
        if (crease_pairs && k) CU(cudaMemcpyAsync(crease_pairs, pairs.data(), sizeof(int32_t) * 2 * k, cudaMemcpyDefault, s));
        if (crease_sigma && k) CU(cudaMemcpyAsync(crease_sigma, sig.data(), sizeof(float) * k, cudaMemcpyDefault, s));
        if (num_creases) CU(cudaMemcpyAsync(num_creases, &k, sizeof(int32_t), cudaMemcpyDefault, s));
        CU(cudaStreamSynchronize(s));
    }
    if (!tmp.empty()) {
        CU(cudaStreamSynchronize(s));
        free_list(m, tmp, s);
    }
    if ((face_vtx && !is_device_ptr(face_vtx)) || (face_off && !is_device_ptr(face_off))) CU(cudaStreamSynchronize(s));
    CU(cudaGetLastError());
    return ALSUB_OK;
}

extern "C" alsub_status alsub_level_positions(const alsub_mesh *m, int32_t level, float *pos, void *stream) {
    if (!m || !pos) return fail(ALSUB_E_ARG, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    const float *src;
    int64_t V;
    if (level == 0) { src = m->pos0; V = m->V0; }
    else {
        const LevelHost *L = level_of(m, level);
        if (!L) return fail(ALSUB_E_ARG, "level out of range");
        src = L->pos; V = L->V;
    }
    CU(cudaMemcpyAsync(pos, src, sizeof(float) * 3 * (size_t)V, cudaMemcpyDefault, s));
    if (!is_device_ptr(pos)) CU(cudaStreamSynchronize(s));
    return ALSUB_OK;
}

// ---------------- selective subdivision: extraction ----------------
extern "C" alsub_status alsub_mesh_extract(const alsub_mesh *m, int32_t level, const uint8_t *vsel, int32_t rings,
                                           void *stream, alsub_mesh **out) {
    if (!m || !out) return fail(ALSUB_E_ARG, "null argument");
    *out = nullptr;
    if (rings < 1) return fail(ALSUB_E_ARG, "rings must be >= 1");
    if (level < 0 || (level > 0 && level > m->levels)) return fail(ALSUB_E_ARG, "level outside 0 .. levels of the last alsub_refine");
    cudaStream_t s = (cudaStream_t)stream;
    ExSrcHost h{};
    if (level == 0) {
        h = ExSrcHost{m->V0, m->F0, m->S0, m->order0 == 0 ? 0 : m->order0, m->in_face_off, m->in_face_vtx, m->pos0,
                      m->b0.sp, m->K0};
        if (m->order0 != 0) h.face_off = nullptr;
    } else {
        const LevelHost &L = m->lv[level];
        const bool special = m->scheme != ALSUB_SQRT3 && m->K0 > 0;
        if (special && level == m->levels) ensure_last_lists(const_cast<alsub_mesh *>(m), (cudaStream_t)stream);
        h = ExSrcHost{(int32_t)L.V, (int32_t)L.F, (int32_t)L.S, L.order, nullptr, L.face_vtx, L.pos,
                      special ? L.sp : nullptr, special ? (int32_t)L.nsp : 0};
    }
    alsub_mesh *mm = const_cast<alsub_mesh *>(m);
    std::vector<std::pair<void *, size_t>> tmp;
    bool ok = true;
    const int64_t V = h.V, F = h.F, S = h.S, K = h.nsp;
    const uint8_t *vsel_dev = vsel;
    if (vsel && !is_device_ptr(vsel)) {
        uint8_t *d = A<uint8_t>(mm, V, s, tmp, ok);
        if (ok && V > 0) CU(cudaMemcpyAsync(d, vsel, (size_t)V, cudaMemcpyHostToDevice, s));
        vsel_dev = d;
    }
    ExWork w{};
    w.n = A<int32_t>(mm, V, s, tmp, ok); w.x = A<int32_t>(mm, V, s, tmp, ok); w.vid = A<int32_t>(mm, V, s, tmp, ok);
    w.q = A<int32_t>(mm, F, s, tmp, ok); w.fid = A<int32_t>(mm, F, s, tmp, ok); w.fo = A<int32_t>(mm, F, s, tmp, ok);
    w.foff = A<int32_t>(mm, F, s, tmp, ok); w.cflag = A<int32_t>(mm, K, s, tmp, ok); w.cid = A<int32_t>(mm, K, s, tmp, ok);
    w.tot = A<int32_t>(mm, 4, s, tmp, ok);
    w.scratch = dev_alloc(mm, scan_scratch_bytes(std::max(std::max(V, F), std::max(K, (int64_t)1))), s, tmp);
    ExOutHost o{};
    o.face_off = A<int32_t>(mm, F + 1, s, tmp, ok); o.face_vtx = A<int32_t>(mm, S, s, tmp, ok);
    o.vmap = A<int32_t>(mm, V, s, tmp, ok); o.fmap = A<int32_t>(mm, F, s, tmp, ok);
    o.crease = A<int32_t>(mm, 2 * K, s, tmp, ok); o.pos = A<float>(mm, 3 * V, s, tmp, ok);
    o.sigma = A<float>(mm, K, s, tmp, ok);
    if (!ok || !w.scratch) { free_list(mm, tmp, s); return fail(ALSUB_E_NOMEM, "extraction buffers"); }
    Launches L;
    extract_level(h, vsel_dev, rings, w, o, s, L);
    int32_t tot[4] = {0, 0, 0, 0};
    CU(cudaMemcpyAsync(tot, w.tot, sizeof(tot), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    alsub_mesh *n = nullptr;
    const alsub_allocator *al = m->custom ? &m->alloc : nullptr;
    alsub_status st = create_impl(o.face_off, o.face_vtx, tot[1], o.pos, tot[0], o.crease, o.sigma, tot[3], al, stream,
                                  &n, true);
    if (st != ALSUB_OK) { free_list(mm, tmp, s); return st; }
    n->ext_vmap = A<int32_t>(n, tot[0], s, n->mem_create, ok);
    n->ext_fmap = A<int32_t>(n, tot[1], s, n->mem_create, ok);
    if (!ok) { free_list(mm, tmp, s); alsub_mesh_destroy(n); return fail(ALSUB_E_NOMEM, "extraction maps"); }
    if (tot[0] > 0) CU(cudaMemcpyAsync(n->ext_vmap, o.vmap, sizeof(int32_t) * tot[0], cudaMemcpyDeviceToDevice, s));
    if (tot[1] > 0) CU(cudaMemcpyAsync(n->ext_fmap, o.fmap, sizeof(int32_t) * tot[1], cudaMemcpyDeviceToDevice, s));
    n->extracted = true;
    free_list(mm, tmp, s);
    CU(cudaGetLastError());
    *out = n;
    return ALSUB_OK;
}

extern "C" alsub_status alsub_extract_maps(const alsub_mesh *m, int32_t *vtx_map, int32_t *face_map, void *stream) {
    if (!m) return fail(ALSUB_E_ARG, "null mesh");
    if (!m->extracted) return fail(ALSUB_E_ARG, "not a handle made by alsub_mesh_extract");
    cudaStream_t s = (cudaStream_t)stream;
    if (vtx_map && m->V0 > 0) CU(cudaMemcpyAsync(vtx_map, m->ext_vmap, sizeof(int32_t) * m->V0, cudaMemcpyDefault, s));
    if (face_map && m->F0 > 0) CU(cudaMemcpyAsync(face_map, m->ext_fmap, sizeof(int32_t) * m->F0, cudaMemcpyDefault, s));
    if ((vtx_map && !is_device_ptr(vtx_map)) || (face_map && !is_device_ptr(face_map))) CU(cudaStreamSynchronize(s));
    return ALSUB_OK;
}

// ---------------- static mode ----------------
// One level of static evaluation over the stored topology of level l (only the eval
// half of every module runs): positions fr.P (level l) -> fr.Pn (level l + 1) for fr.nb frames.
static void static_level(alsub_mesh *m, int l, const Frames &fr, cudaStream_t s, Launches &L) {
    const int scheme = m->scheme;
    const bool special = scheme != ALSUB_SQRT3 && m->K0 > 0;
    const LevelHost &Pl = m->lv[l];
    LevelDev p = dev_of(Pl);
    p.sv_vtx = m->sv_vtx;
    p.sv_off = m->sv_off;
    p.inherit = 0;
    ChildDev c{};
    if (scheme == ALSUB_CATMULL_CLARK) {
        VSegs g = make_segs(m, l);
        LevelDev gp{};
        const bool use_gp = cc_use_gp(m, l, special);
        Frames fx = fr;
        if (use_gp) {
            gp = dev_of(m->lv[l - 1]);
            g.len[g.hs_seg] = 0;  // the edge kernel smooths the edge points born at level l
            fx.hs = nullptr;
        }
        p.crease = (special && !use_gp && Pl.V < kFuseCreaseMaxV) ? 1 : 0;
        if (use_gp && l >= 3 && m->gside) {  // compact corner sums + straddling groups
            fx.c0shift = 2;
            fx.gside = fr.nb == 1 ? m->gside : m->frame_gside;
            fx.gcnt = fr.nb == 1 ? m->gcnt : m->frame_gcnt;
            fx.gsidestride = 12 * (int64_t)m->gblk;
        }
        cc_level(p, c, fx, false, false, g, use_gp ? &gp : nullptr, s, L);
        if (special && !p.crease) crease_level(p, c, fx, (int32_t)(Pl.V + Pl.F), 0, false, s, L);
    } else if (scheme == ALSUB_LOOP) {
        VSegs g = make_segs_loop(m, l);
        loop_level(p, c, fr, false, false, nullptr, nullptr, g, s, L, special ? 0 : -1);
    } else {
        VSegs g = make_segs_s3(m, l);
        sqrt3_level(p, c, fr, false, false, g, s, L);
    }
}

extern "C" alsub_status alsub_level_positions_ptr(alsub_mesh *m, int32_t level, float **pos_dev) {
    if (!m || !pos_dev) return fail(ALSUB_E_ARG, "null argument");
    if (level == 0) { *pos_dev = m->pos0; return ALSUB_OK; }
    LevelHost *L = const_cast<LevelHost *>(level_of(m, level));
    if (!L) return fail(ALSUB_E_ARG, "level out of range");
    *pos_dev = L->pos;
    return ALSUB_OK;
}

extern "C" alsub_status alsub_reevaluate(alsub_mesh *m, int32_t from_level, void *stream) {
    if (!m) return fail(ALSUB_E_ARG, "null argument");
    if (m->levels < 0 || from_level < 0 || from_level > m->levels)
        return fail(ALSUB_E_ARG, "from_level outside 0 .. levels of the last alsub_refine");
    cudaStream_t s = (cudaStream_t)stream;
    Launches L;
    L.side = m->side_stream;
    L.ev_fork = m->ev_fork;
    L.ev_join = m->ev_join;
    L.ev_aux = m->ev_aux;
    for (int l = from_level; l < m->levels; ++l) {
        const float *P = l == 0 ? m->pos0 : m->lv[l].pos;
        Frames fr{P, m->lv[l + 1].pos, 3 * m->lv[l].V, 3 * m->lv[l + 1].V, 1, m->hs, 0,
                  (l >= 1 && m->scheme == ALSUB_CATMULL_CLARK) ? m->c0 : nullptr, 0};
        static_level(m, l, fr, s, L);
    }
    m->last_launches = L.n;
    CU(cudaGetLastError());
    return ALSUB_OK;
}

extern "C" alsub_status alsub_eval_attributes(alsub_mesh *m, int32_t levels, const float *attr_in, int32_t channels,
                                              float *attr_out, void *stream) {
    if (!m || channels < 0 || (channels > 0 && (!attr_in || !attr_out))) return fail(ALSUB_E_ARG, "bad argument");
    if (m->levels < 0 || levels < 0 || levels > m->levels) return fail(ALSUB_E_ARG, "levels exceed the last alsub_refine");
    if (channels == 0) return ALSUB_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t V0 = m->V0, VL = m->lv[levels].V;
    const int32_t ng = (channels + 2) / 3;
    std::vector<std::pair<void *, size_t>> tmp;
    bool ok = true;
    float *in_dev = const_cast<float *>(attr_in), *out_dev = attr_out;
    if (!is_device_ptr(attr_in)) in_dev = A<float>(m, V0 * channels, s, tmp, ok);
    if (!is_device_ptr(attr_out)) out_dev = A<float>(m, VL * channels, s, tmp, ok);
    float *fin = A<float>(m, 3 * V0 * ng, s, tmp, ok), *fout = A<float>(m, 3 * VL * ng, s, tmp, ok);
    if (!ok) { free_list(m, tmp, s); return fail(ALSUB_E_NOMEM, "attribute staging buffers"); }
    if (in_dev != attr_in) CU(cudaMemcpyAsync(in_dev, attr_in, sizeof(float) * V0 * channels, cudaMemcpyHostToDevice, s));
    Launches L;
    pack_channels(in_dev, V0, channels, fin, s, L);
    const alsub_status st = alsub_eval_frames(m, levels, fin, ng, fout, stream);
    if (st != ALSUB_OK) { free_list(m, tmp, s); return st; }
    unpack_channels(fout, VL, channels, out_dev, s, L);
    if (out_dev != attr_out) {
        CU(cudaMemcpyAsync(attr_out, out_dev, sizeof(float) * VL * channels, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
    }
    m->last_launches += L.n;
    free_list(m, tmp, s);
    CU(cudaGetLastError());
    return ALSUB_OK;
}

// ---------------- refinement matrix R (NEXT-1) ----------------
extern "C" alsub_status alsub_build_refinement_matrix(alsub_mesh *m, int32_t levels, void *stream) {
    if (!m) return fail(ALSUB_E_ARG, "null mesh");
    if (m->levels < 1 || levels < 1 || levels > m->levels) return fail(ALSUB_E_ARG, "levels outside 1 .. levels of the last alsub_refine");
    if (m->scheme == ALSUB_SQRT3) return fail(ALSUB_E_SCHEME, "sqrt3 faces do not nest in their parents: no per-face support");
    cudaStream_t s = (cudaStream_t)stream;
    free_list(m, m->mem_rm, s);
    m->rm_levels = -1;
    const int32_t V0 = m->V0, F0 = m->F0;
    const int64_t VL = m->lv[levels].V, FL = m->lv[levels].F;
    // host: the control faces, their 1-ring vertex sets S_f and a colouring of the control vertices
    // with no two vertices of one colour in any S_f
    std::vector<int32_t> off((size_t)F0 + 1), fv((size_t)m->S0);
    CU(cudaMemcpyAsync(off.data(), m->in_face_off, sizeof(int32_t) * off.size(), cudaMemcpyDeviceToHost, s));
    if (m->S0 > 0) CU(cudaMemcpyAsync(fv.data(), m->in_face_vtx, sizeof(int32_t) * fv.size(), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    std::vector<int32_t> vf_off((size_t)V0 + 1, 0), vf;
    for (int32_t h = 0; h < m->S0; ++h) ++vf_off[fv[h] + 1];
    for (int32_t v = 0; v < V0; ++v) vf_off[v + 1] += vf_off[v];
    vf.resize((size_t)m->S0);
    {
        std::vector<int32_t> cur(vf_off.begin(), vf_off.end() - 1);
        for (int32_t r = 0; r < F0; ++r)
            for (int32_t h = off[r]; h < off[r + 1]; ++h) vf[cur[fv[h]]++] = r;
    }
    std::vector<int32_t> sup_off((size_t)F0 + 1, 0), sup, mark((size_t)V0, -1);
    for (int32_t r = 0; r < F0; ++r) {
        const size_t b = sup.size();
        for (int32_t h = off[r]; h < off[r + 1]; ++h)
            for (int32_t q = vf_off[fv[h]]; q < vf_off[fv[h] + 1]; ++q) {
                const int32_t g = vf[q];
                for (int32_t k = off[g]; k < off[g + 1]; ++k)
                    if (mark[fv[k]] != r) { mark[fv[k]] = r; sup.push_back(fv[k]); }
            }
        std::sort(sup.begin() + b, sup.end());
        sup_off[r + 1] = (int32_t)sup.size();
    }
    // faces whose support holds v (the inverse lists), then greedy colouring in vertex order
    std::vector<int32_t> fs_off((size_t)V0 + 1, 0), fs;
    for (int32_t v : sup) ++fs_off[v + 1];
    for (int32_t v = 0; v < V0; ++v) fs_off[v + 1] += fs_off[v];
    fs.resize(sup.size());
    {
        std::vector<int32_t> cur(fs_off.begin(), fs_off.end() - 1);
        for (int32_t r = 0; r < F0; ++r)
            for (int32_t k = sup_off[r]; k < sup_off[r + 1]; ++k) fs[cur[sup[k]]++] = r;
    }
    std::vector<int32_t> colour((size_t)V0, -1), used;
    int32_t ncol = 0;
    for (int32_t v = 0; v < V0; ++v) {
        used.assign((size_t)ncol + 1, 0);
        for (int32_t q = fs_off[v]; q < fs_off[v + 1]; ++q)
            for (int32_t k = sup_off[fs[q]]; k < sup_off[fs[q] + 1]; ++k)
                if (colour[sup[k]] >= 0) used[colour[sup[k]]] = 1;
        int32_t c = 0;
        while (used[c]) ++c;
        colour[v] = c;
        ncol = std::max(ncol, c + 1);
    }
    const int32_t nprobe = (ncol + 2) / 3;
    // chunks of the blocked form: the F0 owner faces, then one per isolated control vertex (its row
    // is the identity: support {v})
    std::vector<int32_t> iso_chunk((size_t)V0, -1);
    int32_t C = F0;
    for (int32_t v = 0; v < V0; ++v)
        if (vf_off[v + 1] == vf_off[v]) {
            iso_chunk[v] = C++;
            sup.push_back(v);
            sup_off.push_back((int32_t)sup.size());
        }
    // device: probes through the static path, owners, two-pass CSR assembly
    std::vector<std::pair<void *, size_t>> tmp;
    bool ok = true;
    m->rb_sup_off = A<int32_t>(m, (int64_t)C + 1, s, m->mem_rm, ok);
    m->rb_sup = A<int32_t>(m, (int64_t)sup.size(), s, m->mem_rm, ok);
    int32_t *d_sup_off = m->rb_sup_off, *d_sup = m->rb_sup;
    int32_t *d_col = A<int32_t>(m, V0, s, tmp, ok), *d_owner = A<int32_t>(m, VL, s, tmp, ok);
    int32_t *d_len = A<int32_t>(m, VL + 1, s, tmp, ok), *d_tot = A<int32_t>(m, 1, s, tmp, ok);
    int64_t *d_nnz = A<int64_t>(m, 1, s, tmp, ok);
    int32_t *d_chunk = A<int32_t>(m, VL, s, tmp, ok), *d_cnt = A<int32_t>(m, (int64_t)C + 1, s, tmp, ok);
    int32_t *d_cur = A<int32_t>(m, C, s, tmp, ok), *d_pos = A<int32_t>(m, VL, s, tmp, ok);
    int64_t *d_wlen = A<int64_t>(m, C, s, tmp, ok);
    int32_t *d_iso = A<int32_t>(m, V0, s, tmp, ok);
    float *d_pin = A<float>(m, 3 * (int64_t)V0 * std::max(nprobe, 1), s, tmp, ok);
    float *d_pout = A<float>(m, 3 * VL * std::max(nprobe, 1), s, tmp, ok);
    void *scr = dev_alloc(m, scan_scratch_bytes(std::max<int64_t>(VL, C) + 1), s, tmp);
    m->rm_row_off = A<int32_t>(m, VL + 1, s, m->mem_rm, ok);
    m->rb_xt = A<float>(m, 3 * (int64_t)V0 * kRmLanes + 4, s, m->mem_rm, ok);  // + the chunk counter
    m->rb_row_off = A<int32_t>(m, (int64_t)C + 1, s, m->mem_rm, ok);
    m->rb_rows = A<int32_t>(m, VL, s, m->mem_rm, ok);
    m->rb_w_off = A<int64_t>(m, (int64_t)C + 1, s, m->mem_rm, ok);
    if (!ok || !scr) { free_list(m, tmp, s); free_list(m, m->mem_rm, s); return fail(ALSUB_E_NOMEM, "refinement matrix buffers"); }
    CU(cudaMemcpyAsync(d_sup_off, sup_off.data(), sizeof(int32_t) * sup_off.size(), cudaMemcpyHostToDevice, s));
    if (!sup.empty()) CU(cudaMemcpyAsync(d_sup, sup.data(), sizeof(int32_t) * sup.size(), cudaMemcpyHostToDevice, s));
    if (V0 > 0) CU(cudaMemcpyAsync(d_col, colour.data(), sizeof(int32_t) * V0, cudaMemcpyHostToDevice, s));
    if (V0 > 0) CU(cudaMemcpyAsync(d_iso, iso_chunk.data(), sizeof(int32_t) * V0, cudaMemcpyHostToDevice, s));
    Launches L;
    rm_probes(V0, d_col, nprobe, d_pin, s, L);
    alsub_status st = nprobe > 0 ? alsub_eval_frames(m, levels, d_pin, nprobe, d_pout, stream) : ALSUB_OK;
    if (st != ALSUB_OK) { free_list(m, tmp, s); free_list(m, m->mem_rm, s); return st; }
    {
        ZeroSegs z;
        z.add(d_owner, VL, INT32_MAX);
        z.add(d_len + VL, 1, 0);
        z.add(d_nnz, 2, 0);
        z.add(d_cnt, (int64_t)C + 1, 0);
        z.add(d_cur, C, 0);
        zero_segments(z, s, L);
    }
    const int shift = m->scheme == ALSUB_CATMULL_CLARK ? 2 * (levels - 1) : 2 * levels;
    rm_owner(m->lv[levels].face_vtx, (int32_t)FL, m->lv[levels].order, shift,
             m->scheme == ALSUB_CATMULL_CLARK ? m->b0.slot_face : nullptr, d_owner, s, L);
    rm_assemble((int32_t)VL, d_owner, d_sup_off, d_sup, d_col, d_pout, 3 * VL, false, d_len, nullptr, nullptr, d_nnz, s, L);
    scan_exclusive(d_len, m->rm_row_off, VL + 1, d_tot, scr, s, L);
    // blocked form: rows grouped by chunk (counting sort + per-chunk sort), W lengths scanned in 64 bits
    rb_hist((int32_t)VL, d_owner, d_iso, d_chunk, d_cnt, s, L);
    scan_exclusive(d_cnt, m->rb_row_off, (int64_t)C + 1, nullptr, scr, s, L);
    rb_scatter((int32_t)VL, d_chunk, m->rb_row_off, d_cur, m->rb_rows, s, L);
    rb_sort(C, m->rb_row_off, d_sup_off, m->rb_rows, d_pos, d_wlen, m->rb_w_off, s, L);
    int64_t nnz = 0, wlen = 0;
    CU(cudaMemcpyAsync(&nnz, d_nnz, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(&wlen, m->rb_w_off + C, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (nnz > INT32_MAX) {  // the CSR export's int32 row offsets would wrap
        free_list(m, tmp, s);
        free_list(m, m->mem_rm, s);
        return fail(ALSUB_E_OVERFLOW, "refinement matrix has more than 2^31 - 1 non-zeros");
    }
    m->rm_ent = A<int2>(m, std::max<int64_t>(nnz, 1), s, m->mem_rm, ok);
    m->rb_W = A<float>(m, std::max<int64_t>(wlen, 1), s, m->mem_rm, ok);
    if (!ok) { free_list(m, tmp, s); free_list(m, m->mem_rm, s); return fail(ALSUB_E_NOMEM, "refinement matrix entries"); }
    rm_assemble((int32_t)VL, d_owner, d_sup_off, d_sup, d_col, d_pout, 3 * VL, true, nullptr, m->rm_row_off, m->rm_ent, nullptr,
                s, L);
    if (wlen > 0) CU(cudaMemsetAsync(m->rb_W, 0, sizeof(float) * (size_t)wlen, s));
    rb_fill((int32_t)VL, d_chunk, d_pos, m->rb_row_off, d_sup_off, d_sup, m->rb_w_off, d_col, d_pout, 3 * VL, m->rb_W, s, L);
    free_list(m, tmp, s);
    m->rm_levels = levels;
    m->rm_scheme = m->scheme;
    m->rm_nnz = nnz;
    m->rb_C = C;
    m->rb_wlen = wlen;
    m->last_launches = L.n;
    CU(cudaGetLastError());
    return ALSUB_OK;
}

extern "C" alsub_status alsub_refinement_matrix_info(const alsub_mesh *m, int32_t *levels, int64_t *rows, int64_t *nnz) {
    if (!m) return fail(ALSUB_E_ARG, "null mesh");
    if (m->rm_levels < 0) return fail(ALSUB_E_ARG, "no refinement matrix: call alsub_build_refinement_matrix");
    if (levels) *levels = m->rm_levels;
    if (rows) *rows = m->lv[m->rm_levels].V;
    if (nnz) *nnz = m->rm_nnz;
    return ALSUB_OK;
}

extern "C" alsub_status alsub_refinement_matrix_blocks(const alsub_mesh *m, int64_t *chunks, int64_t *weights) {
    if (!m) return fail(ALSUB_E_ARG, "null mesh");
    if (m->rm_levels < 0) return fail(ALSUB_E_ARG, "no refinement matrix: call alsub_build_refinement_matrix");
    if (chunks) *chunks = m->rb_C;
    if (weights) *weights = m->rb_wlen;
    return ALSUB_OK;
}

extern "C" alsub_status alsub_refinement_matrix_csr(const alsub_mesh *m, int32_t *row_off, int32_t *cols, float *vals,
                                                    void *stream) {
    if (!m) return fail(ALSUB_E_ARG, "null mesh");
    if (m->rm_levels < 0) return fail(ALSUB_E_ARG, "no refinement matrix: call alsub_build_refinement_matrix");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t VL = m->lv[m->rm_levels].V;
    if (row_off) CU(cudaMemcpyAsync(row_off, m->rm_row_off, sizeof(int32_t) * (VL + 1), cudaMemcpyDefault, s));
    if ((cols || vals) && m->rm_nnz > 0) {
        std::vector<int2> e((size_t)m->rm_nnz);
        CU(cudaMemcpyAsync(e.data(), m->rm_ent, sizeof(int2) * e.size(), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        std::vector<int32_t> c(e.size());
        std::vector<float> v(e.size());
        for (size_t i = 0; i < e.size(); ++i) {
            c[i] = e[i].x;
            memcpy(&v[i], &e[i].y, sizeof(float));
        }
        if (cols) CU(cudaMemcpyAsync(cols, c.data(), sizeof(int32_t) * c.size(), cudaMemcpyDefault, s));
        if (vals) CU(cudaMemcpyAsync(vals, v.data(), sizeof(float) * v.size(), cudaMemcpyDefault, s));
    }
    CU(cudaStreamSynchronize(s));
    return ALSUB_OK;
}

static alsub_status eval_frames_matrix(alsub_mesh *m, const float *frames_in, int32_t num_frames, float *frames_out,
                                       int32_t *summary, void *stream) {
    if (!m || num_frames < 0 || (num_frames > 0 && (!frames_in || !frames_out))) return fail(ALSUB_E_ARG, "bad argument");
    if (m->rm_levels < 0) return fail(ALSUB_E_ARG, "no refinement matrix: call alsub_build_refinement_matrix");
    if (num_frames > 0 && (!is_device_ptr(frames_in) || !is_device_ptr(frames_out) || (summary && !is_device_ptr(summary))))
        return fail(ALSUB_E_ARG, "alsub_eval_frames_matrix takes device pointers");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t V0 = m->V0, VL = m->lv[m->rm_levels].V;
    Launches L;
    for (int32_t f0 = 0; f0 < num_frames; f0 += kRmLanes) {
        const int32_t n = std::min(kRmLanes, num_frames - f0);
        SummaryRec *rec = summary ? reinterpret_cast<SummaryRec *>(summary) + f0 : nullptr;
        if (rec) summary_init(rec, n, s, L);
        rb_eval(m->rb_C, m->rb_row_off, m->rb_sup_off, m->rb_w_off, m->rb_rows, m->rb_sup, m->rb_W,
                frames_in + 3 * V0 * (int64_t)f0, (int32_t)V0, n, m->rb_xt, VL, frames_out + 3 * VL * (int64_t)f0, rec,
                s, L);
        if (rec) summary_decode(rec, n, s, L);
    }
    m->last_launches = L.n;
    CU(cudaGetLastError());
    return ALSUB_OK;
}

extern "C" alsub_status alsub_eval_frames_matrix(alsub_mesh *m, const float *frames_in, int32_t num_frames,
                                                 float *frames_out, void *stream) {
    return eval_frames_matrix(m, frames_in, num_frames, frames_out, nullptr, stream);
}

extern "C" alsub_status alsub_eval_frames_matrix_summary(alsub_mesh *m, const float *frames_in, int32_t num_frames,
                                                         float *frames_out, int32_t *summary, void *stream) {
    if (!summary && num_frames > 0) return fail(ALSUB_E_ARG, "null summary");
    return eval_frames_matrix(m, frames_in, num_frames, frames_out, summary, stream);
}

// ---------------- static mode: frames ----------------
extern "C" alsub_status alsub_eval_frames(alsub_mesh *m, int32_t levels, const float *frames_in, int32_t num_frames,
                                          float *frames_out, void *stream) {
    if (!m || num_frames < 0 || (num_frames > 0 && (!frames_in || !frames_out))) return fail(ALSUB_E_ARG, "bad argument");
    if (m->levels < 0 || levels < 0 || levels > m->levels) return fail(ALSUB_E_ARG, "levels exceed the last alsub_refine");
    cudaStream_t s = (cudaStream_t)stream;
    const int scheme = m->scheme;
    const int64_t V0 = m->V0, VL = m->lv[levels].V;
    if (num_frames == 0) return ALSUB_OK;
    if (levels == 0) {
        CU(cudaMemcpyAsync(frames_out, frames_in, sizeof(float) * 3 * (size_t)V0 * num_frames, cudaMemcpyDefault, s));
        return ALSUB_OK;
    }
    const bool in_dev = is_device_ptr(frames_in), out_dev = is_device_ptr(frames_out);
    const int nb_max = getenv("ALSUB_FRAME_BATCH") ? std::max(1, std::min(64, atoi(getenv("ALSUB_FRAME_BATCH")))) : 8;
    const int nb = std::min(num_frames, nb_max);
    // per-level batch buffers of 3 V_l nb floats for l = 0 (if host input) .. levels (if host output)
    if (m->frames_nb < nb || (int)m->frame_buf.size() != m->levels + 1) {
        free_list(m, m->mem_frames, s);
        m->frame_buf.assign((size_t)m->levels + 1, nullptr);
        bool ok = true;
        for (int l = 0; l <= m->levels; ++l)
            m->frame_buf[l] = A<float>(m, 3 * m->lv[l].V * nb, s, m->mem_frames, ok);
        m->frame_hs = m->hs_elems ? A<float>(m, m->hs_elems * nb, s, m->mem_frames, ok) : nullptr;
        m->frame_c0 = m->c0_elems ? A<float>(m, m->c0_elems * nb, s, m->mem_frames, ok) : nullptr;
        m->frame_gside = m->gblk ? A<float>(m, 12 * (int64_t)m->gblk * nb, s, m->mem_frames, ok) : nullptr;
        m->frame_gcnt = m->gblk ? A<int32_t>(m, m->gblk, s, m->mem_frames, ok) : nullptr;
        if (m->frame_gcnt) cudaMemsetAsync(m->frame_gcnt, 0, sizeof(int32_t) * m->gblk, s);
        if (!ok) return fail(ALSUB_E_NOMEM, "frame batch buffers");
        m->frames_nb = nb;
    }
    const bool special = scheme != ALSUB_SQRT3 && m->K0 > 0;
    Launches L;
    L.side = m->side_stream;
    L.ev_fork = m->ev_fork;
    L.ev_join = m->ev_join;
    L.ev_aux = m->ev_aux;
    for (int32_t f0 = 0; f0 < num_frames; f0 += nb) {
        const int n = std::min(nb, num_frames - f0);
        const float *Pin = frames_in + 3 * V0 * (int64_t)f0;
        if (!in_dev) {
            CU(cudaMemcpyAsync(m->frame_buf[0], Pin, sizeof(float) * 3 * V0 * n, cudaMemcpyHostToDevice, s));
            Pin = m->frame_buf[0];
        }
        float *Pout_final = out_dev ? frames_out + 3 * VL * (int64_t)f0 : m->frame_buf[levels];
        const float *P = Pin;
        for (int l = 0; l < levels; ++l) {
            float *Pn = (l + 1 == levels) ? Pout_final : m->frame_buf[l + 1];
            // frame-major [n][V][3] at every level (a frame-interleaved [V][n][3] layout was measured
            // slower: its per-frame stores are strided, profiles/r01_frames_experiments.md)
            Frames fr{P, Pn, 3 * m->lv[l].V, 3 * m->lv[l + 1].V, n, m->frame_hs, m->hs_elems,
                      (l >= 1 && scheme == ALSUB_CATMULL_CLARK) ? m->frame_c0 : nullptr, m->c0_elems};
            static_level(m, l, fr, s, L);
            P = Pn;
        }
        if (!out_dev)
            CU(cudaMemcpyAsync(frames_out + 3 * VL * (int64_t)f0, Pout_final, sizeof(float) * 3 * VL * n,
                               cudaMemcpyDeviceToHost, s));
    }
    if (!out_dev) CU(cudaStreamSynchronize(s));
    m->last_launches = L.n;
    CU(cudaGetLastError());
    return ALSUB_OK;
}

static void free_probe_events(alsub_mesh *m) {
    for (cudaEvent_t e : m->probe_start) cudaEventDestroy(e);
    for (cudaEvent_t e : m->probe_stop) cudaEventDestroy(e);
    m->probe_start.clear();
    m->probe_stop.clear();
    for (cudaEvent_t &e : m->probe_cap)
        if (e) { cudaEventDestroy(e); e = nullptr; }
    for (cudaEvent_t &e : m->probe_dep)
        if (e) { cudaEventDestroy(e); e = nullptr; }
    if (m->probe_stream) { cudaStreamDestroy(m->probe_stream); m->probe_stream = nullptr; }
}

extern "C" alsub_status alsub_probe(alsub_mesh *m, int32_t level, const char *kernel, int32_t steps) {
    if (!m) return fail(ALSUB_E_ARG, "null mesh");
    if (steps < 0 || steps > 1 << 20) return fail(ALSUB_E_ARG, "steps must be in [0, 2^20]");
    if (steps > 0 && !kernel) return fail(ALSUB_E_ARG, "null kernel name");
    CU(cudaDeviceSynchronize());  // events of an earlier probe may still be pending
    const bool same = steps > 0 && !m->probe_start.empty() && m->probe_level == level && m->probe_name == kernel;
    if (!same) {
        drop_graph(m);  // the next alsub_refine re-captures (with or without the probe nodes)
        free_probe_events(m);
        if (steps == 0) return ALSUB_OK;
        m->probe_name = kernel;
        m->probe_level = level;
        for (cudaEvent_t &e : m->probe_cap) CU(cudaEventCreate(&e));
        for (cudaEvent_t &e : m->probe_dep) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CU(cudaStreamCreateWithFlags(&m->probe_stream, cudaStreamNonBlocking));
    }
    const size_t have = m->probe_start.size();
    for (size_t i = have; i < (size_t)steps; ++i) {
        cudaEvent_t a, b;
        CU(cudaEventCreate(&a));
        CU(cudaEventCreate(&b));
        m->probe_start.push_back(a);
        m->probe_stop.push_back(b);
    }
    m->probe_next = 0;
    return ALSUB_OK;
}

extern "C" alsub_status alsub_probe_read(alsub_mesh *m, float *ms, int32_t cap, int32_t *count) {
    if (!m || !count) return fail(ALSUB_E_ARG, "null argument");
    const int32_t n = m->probe_next;
    *count = n;
    if (!m->probe_start.empty() && m->gexec && !m->probe_node[0])
        return fail(ALSUB_E_ARG, "the probe matched no kernel of the captured refine");
    if (n == 0) return ALSUB_OK;
    CU(cudaEventSynchronize(m->probe_stop[n - 1]));
    for (int32_t i = 0; i < n && i < cap; ++i) CU(cudaEventElapsedTime(ms + i, m->probe_start[i], m->probe_stop[i]));
    return ALSUB_OK;
}

extern "C" alsub_status alsub_probe_read_offsets(alsub_mesh *m, void *const *ref_events, float *start_ms, float *stop_ms,
                                                 int32_t cap, int32_t *count) {
    if (!m || !ref_events || !start_ms || !stop_ms || !count) return fail(ALSUB_E_ARG, "null argument");
    const int32_t n = m->probe_next;
    *count = n;
    if (!m->probe_start.empty() && m->gexec && !m->probe_node[0])
        return fail(ALSUB_E_ARG, "the probe matched no kernel of the captured refine");
    if (n == 0) return ALSUB_OK;
    CU(cudaEventSynchronize(m->probe_stop[n - 1]));
    for (int32_t i = 0; i < n && i < cap; ++i) {
        cudaEvent_t r = (cudaEvent_t)ref_events[i];
        CU(cudaEventElapsedTime(start_ms + i, r, m->probe_start[i]));
        CU(cudaEventElapsedTime(stop_ms + i, r, m->probe_stop[i]));
    }
    return ALSUB_OK;
}

extern "C" int64_t alsub_last_launch_count(const alsub_mesh *m) { return m ? m->last_launches : 0; }

extern "C" void alsub_mesh_destroy(alsub_mesh *m) {
    if (!m) return;
    cudaStream_t s = m->cap_stream ? m->cap_stream : (cudaStream_t)0;
    cudaDeviceSynchronize();
    drop_graph(m);
    free_probe_events(m);
    free_list(m, m->mem_frames, s);
    free_list(m, m->mem_rm, s);
    free_list(m, m->mem_plan, s);
    free_list(m, m->mem_create, s);
    cudaStreamSynchronize(s);
    if (m->cap_stream) cudaStreamDestroy(m->cap_stream);
    if (m->side_stream) cudaStreamDestroy(m->side_stream);
    if (m->ev_fork) cudaEventDestroy(m->ev_fork);
    if (m->ev_join) cudaEventDestroy(m->ev_join);
    if (m->ev_build) cudaEventDestroy(m->ev_build);
    if (m->ev_aux) cudaEventDestroy(m->ev_aux);
    delete m;
}

extern "C" const char *alsub_last_error(void) { return g_err.c_str(); }
extern "C" const char *alsub_version(void) { return "alsub-b200 0.1 (sm_100a)"; }

namespace alsub {
bool Launches::probing(const char *kname) const {
    return probe_name && !probe_hit && level == probe_level && strcmp(kname, probe_name) == 0;
}
bool pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("ALSUB_NO_PDL");
        v = (e && e[0] == '1') ? 0 : 1;
    }
    return v == 1;
}
}  // namespace alsub
