// extract.cu -- selective / feature-adaptive subdivision, the extraction module (SURVEY.md 8(f)
// NEXT-3; PAPER.md §"Selective and Feature Adaptive Subdivision", Fig.
// module_selective).
//
//   x_0          selected vertices: a caller mask, or the extraordinary vertices n = M 1 != 4
//                (Eq. vo)
//   q_i = M^T x_i   faces with a selected vertex
//   x_{i+1} = M q_i vertices of those faces, `rings` times
//   X, X̊         identity with the unselected rows / columns deleted: selected vertices and
//                faces keep their relative order
//   P' = X P,  M' = X M X̊   the extracted positions and mesh
// plus the creases of the level restricted to pairs of selected vertices (pairs that are not an
// edge of an extracted face are dropped by the new handle's level-0 build, reading R25).
//
// Boolean products are flag gathers (no atomics on floats): one thread per face reads its
// vertices' flags (q = M^T x), one thread per selected face sets its vertices' flags (x = M q;
// every writer stores the same 1).  Ids are exclusive scans of the flags.
#include "internal.h"

namespace alsub {

struct ExSrc {
    int32_t V, F, S, order;  // order 3 / 4: face r = slots [order r, order r + order); 0: face_off
    const int32_t *face_off, *face_vtx;
    const float *pos;
    const SpEdge *sp;
    int32_t nsp;
};

ALSUB_D int32_t ex_first(const ExSrc &m, int32_t r) { return m.order ? m.order * r : __ldg(m.face_off + r); }
ALSUB_D int32_t ex_count(const ExSrc &m, int32_t r) {
    return m.order ? m.order : __ldg(m.face_off + r + 1) - __ldg(m.face_off + r);
}

// n = M 1 (faces per vertex, Eq. vo)
__global__ void k_ex_valence(ExSrc m, int32_t *__restrict__ n) {
    ALSUB_GRID_WAIT();
    const int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (h < m.S) atomicAdd(n + __ldg(m.face_vtx + h), 1);
}

// x_0: the caller's mask, or n != 4
__global__ void k_ex_seed(int32_t V, const uint8_t *__restrict__ vsel, const int32_t *__restrict__ n,
                          int32_t *__restrict__ x) {
    ALSUB_GRID_WAIT();
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < V) x[v] = vsel ? (vsel[v] != 0) : (n[v] != 4);
}

// q = M^T x (boolean): face r is selected iff one of its vertices is
__global__ void k_ex_faces(ExSrc m, const int32_t *__restrict__ x, int32_t *__restrict__ q) {
    ALSUB_GRID_WAIT();
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m.F) return;
    const int32_t o = ex_first(m, r), c = ex_count(m, r);
    int32_t sel = 0;
    for (int32_t t = 0; t < c; ++t) sel |= x[__ldg(m.face_vtx + o + t)];
    q[r] = sel;
}

// x = M q (boolean): the vertices of the selected faces (x cleared before)
__global__ void k_ex_verts(ExSrc m, const int32_t *__restrict__ q, int32_t *__restrict__ x) {
    ALSUB_GRID_WAIT();
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m.F || !q[r]) return;
    const int32_t o = ex_first(m, r), c = ex_count(m, r);
    for (int32_t t = 0; t < c; ++t) x[__ldg(m.face_vtx + o + t)] = 1;
}

// per-face slot count of the selected faces (scanned into the extracted face_off) and the crease
// flags (live, non-boundary special edges with both endpoints selected)
__global__ void k_ex_counts(ExSrc m, const int32_t *__restrict__ q, const int32_t *__restrict__ x,
                            int32_t *__restrict__ fo, int32_t *__restrict__ cflag) {
    ALSUB_GRID_WAIT();
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m.F) fo[i] = q[i] ? ex_count(m, i) : 0;
    if (i < m.nsp) {
        const SpEdge e = m.sp[i];
        cflag[i] = (e.sigma > 0.0f && !(e.flags & kSpBoundary) && x[e.a] && x[e.b]) ? 1 : 0;
    }
}

struct ExOut {
    int32_t *face_off, *face_vtx, *vmap, *fmap, *crease;
    float *pos, *sigma;
    const int32_t *vid, *fid, *foff, *cid;  // exclusive scans of x, q, fo, cflag
    const int32_t *tot;                     // [4] totals: V', F', S', K'
};

__global__ void k_ex_emit_faces(ExSrc m, const int32_t *__restrict__ q, ExOut o) {
    ALSUB_GRID_WAIT();
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m.F || !q[r]) return;
    const int32_t rr = o.fid[r], base = o.foff[r];
    const int32_t f0 = ex_first(m, r), c = ex_count(m, r);
    o.face_off[rr] = base;
    if (rr == o.tot[1] - 1) o.face_off[rr + 1] = base + c;
    for (int32_t t = 0; t < c; ++t) o.face_vtx[base + t] = o.vid[__ldg(m.face_vtx + f0 + t)];
    o.fmap[rr] = r;
}

__global__ void k_ex_emit_verts(ExSrc m, const int32_t *__restrict__ x, ExOut o) {
    ALSUB_GRID_WAIT();
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= m.V || !x[v]) return;
    const int32_t vv = o.vid[v];
    o.pos[3 * (int64_t)vv + 0] = m.pos[3 * (int64_t)v + 0];
    o.pos[3 * (int64_t)vv + 1] = m.pos[3 * (int64_t)v + 1];
    o.pos[3 * (int64_t)vv + 2] = m.pos[3 * (int64_t)v + 2];
    o.vmap[vv] = v;
}

__global__ void k_ex_emit_creases(ExSrc m, const int32_t *__restrict__ cflag, ExOut o) {
    ALSUB_GRID_WAIT();
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m.nsp || !cflag[j]) return;
    const SpEdge e = m.sp[j];
    const int32_t k = o.cid[j];
    o.crease[2 * k] = o.vid[e.a];
    o.crease[2 * k + 1] = o.vid[e.b];
    o.sigma[k] = e.sigma;
}

void extract_level(const ExSrcHost &h, const uint8_t *vsel, int32_t rings, ExWork &w, ExOutHost &out, cudaStream_t s,
                   Launches &L) {
    ExSrc m{h.V, h.F, h.S, h.order, h.face_off, h.face_vtx, h.pos, h.sp, h.nsp};
    cudaMemsetAsync(w.n, 0, sizeof(int32_t) * (size_t)std::max(m.V, 1), s);
    cudaMemsetAsync(w.tot, 0, sizeof(int32_t) * 4, s);
    cudaMemsetAsync(out.face_off, 0, sizeof(int32_t), s);
    if (!vsel && m.S > 0) launch(L, "ex_valence", k_ex_valence, dim3(grid_for(m.S)), dim3(kThreads), 0, s, m, w.n);
    if (m.V > 0) launch(L, "ex_seed", k_ex_seed, dim3(grid_for(m.V)), dim3(kThreads), 0, s, m.V, vsel, w.n, w.x);
    for (int i = 0; i < rings; ++i) {
        if (m.F > 0) launch(L, "ex_faces", k_ex_faces, dim3(grid_for(m.F)), dim3(kThreads), 0, s, m, w.x, w.q);
        if (m.V > 0) cudaMemsetAsync(w.x, 0, sizeof(int32_t) * (size_t)m.V, s);
        if (m.F > 0) launch(L, "ex_verts", k_ex_verts, dim3(grid_for(m.F)), dim3(kThreads), 0, s, m, w.q, w.x);
    }
    const int64_t nc = std::max<int64_t>(m.F, m.nsp);
    if (nc > 0) launch(L, "ex_counts", k_ex_counts, dim3(grid_for(nc)), dim3(kThreads), 0, s, m, w.q, w.x, w.fo, w.cflag);
    scan_exclusive(w.x, w.vid, m.V, w.tot + 0, w.scratch, s, L);
    scan_exclusive(w.q, w.fid, m.F, w.tot + 1, w.scratch, s, L);
    scan_exclusive(w.fo, w.foff, m.F, w.tot + 2, w.scratch, s, L);
    scan_exclusive(w.cflag, w.cid, m.nsp, w.tot + 3, w.scratch, s, L);
    ExOut o{out.face_off, out.face_vtx, out.vmap, out.fmap, out.crease, out.pos, out.sigma,
            w.vid, w.fid, w.foff, w.cid, w.tot};
    if (m.F > 0) launch(L, "ex_emit_faces", k_ex_emit_faces, dim3(grid_for(m.F)), dim3(kThreads), 0, s, m, w.q, o);
    const int64_t nv = std::max<int64_t>(m.V, 1);
    launch(L, "ex_emit_verts", k_ex_emit_verts, dim3(grid_for(nv)), dim3(kThreads), 0, s, m, w.x, o);
    if (m.nsp > 0) launch(L, "ex_emit_creases", k_ex_emit_creases, dim3(grid_for(m.nsp)), dim3(kThreads), 0, s, m, w.cflag, o);
}

}  // namespace alsub
