// build0.cu -- level-0 topology from arbitrary face lists.
//
// a1  mesh matrix M (CSC: face_off / face_vtx) + validation
// a2  M^T by a stable device radix sort of (vertex, slot) pairs + run-length offsets;
//     vertex valence n = M 1 (Eq. vo) = row length
// a3  the implicit mapped SpGEMMs E = M M^T {Q_c + Q_c^{c-1}}[lambda] and F = M M^T {Q_c}[gamma]
//      evaluated as in the paper's implicit SpGEMM: every collision of
//     vertex j with its face neighbours next(h) = Q_c and prev(h) = Q_c^{c-1} is visited from j's
//     incident slots; a symbolic pass counts the distinct neighbours i < j (the upper-triangular
//     non-zeros of column j of E), a scan turns the counts into ids -- edge id = rank of (j, i) in
//     column-major order (reading R1) -- and a numeric pass fills face_edge / face_twin
//     (F(i,j) and F(j,i)) and the multiplicity checks (E(i,j) in {1, 2}).
// Then the crease matrix C is attached to edge ids and the special-edge list
// (boundary edges = infinitely sharp creases, reading R6) and special-vertex table are built.
#include "internal.h"

namespace alsub {

using T0 = Topo<0>;

__global__ void k_validate_faces(const int32_t *__restrict__ face_off, const int32_t *__restrict__ face_vtx,
                                 int32_t F, int32_t V, int32_t *__restrict__ slot_face, int32_t *__restrict__ sk,
                                 int32_t *__restrict__ sv, int32_t *flags) {
    int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= F) return;
    int32_t o = face_off[r], c = face_off[r + 1] - o;
    if (c < 3) { atomicOr(flags, kFlagMesh); return; }
    for (int32_t t = 0; t < c; ++t) {
        int32_t v = face_vtx[o + t];
        slot_face[o + t] = r;
        sk[o + t] = v;
        sv[o + t] = o + t;
        if (v < 0 || v >= V) { atomicOr(flags, kFlagMesh); sk[o + t] = 0; continue; }
        for (int32_t u = 0; u < t; ++u)
            if (face_vtx[o + u] == v) atomicOr(flags, kFlagMesh);
    }
}

// Candidate q of vertex j's collision list: slot vtx_slot[o0 + q/2], neighbour next (q even) or prev.
struct Cand {
    const int32_t *face_vtx, *vtx_slot;
    T0 tp;
    int32_t o0;
    ALSUB_D int32_t slot(int32_t q) const { return __ldg(vtx_slot + o0 + (q >> 1)); }
    ALSUB_D int32_t vert(int32_t q) const {
        int32_t h = slot(q);
        return __ldg(face_vtx + ((q & 1) ? tp.prev(h) : tp.next(h)));
    }
    // first occurrence of value x among candidates [0, q)
    ALSUB_D bool first(int32_t q, int32_t x) const {
        for (int32_t p = 0; p < q; ++p)
            if (vert(p) == x) return false;
        return true;
    }
};

// Warp-per-vertex collision processing: lane q < 2n holds candidate q of vertex j (slot q/2,
// neighbour next (q even) or prev (q odd)); duplicates are found with __match_any_sync and the
// rank of a distinct neighbour among the distinct neighbours < j with a ballot per lane.
// Vertices with more than 16 incident faces fall back to a serial loop on lane 0.
struct WarpCand {
    int32_t x;     // neighbour vertex (INT32_MAX = none)
    int32_t slot;  // the slot of the directed edge (j -> x for next, x -> j for prev)
    bool first;    // first occurrence of x among the candidates
    unsigned peers;
};

ALSUB_D WarpCand warp_cand(const int32_t *face_vtx, const int32_t *vtx_slot, T0 tp, int32_t o0, int32_t n, int lane) {
    WarpCand c{INT32_MAX, -1, false, 0u};
    if (lane < 2 * n) {
        const int32_t h = __ldg(vtx_slot + o0 + (lane >> 1));
        if (lane & 1) {
            const int32_t hp = tp.prev(h);
            c.x = __ldg(face_vtx + hp);
            c.slot = hp;
        } else {
            c.x = __ldg(face_vtx + tp.next(h));
            c.slot = h;
        }
    }
    c.peers = __match_any_sync(0xffffffffu, c.x);
    c.first = c.x != INT32_MAX && (__ffs(c.peers) - 1) == lane;
    return c;
}

// symbolic pass: number of distinct neighbours i < j of vertex j (non-zeros of E's column j above
// the diagonal)
__global__ void k_edge_count(const int32_t *__restrict__ face_vtx, const int32_t *__restrict__ vtx_off,
                             const int32_t *__restrict__ vtx_slot, T0 tp, int32_t V, int32_t *__restrict__ cnt) {
    const int32_t j = (int32_t)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (j >= V) return;
    const int32_t o0 = vtx_off[j], n = vtx_off[j + 1] - o0;
    if (n <= 16) {
        const WarpCand c = warp_cand(face_vtx, vtx_slot, tp, o0, n, lane);
        const unsigned b = __ballot_sync(0xffffffffu, c.first && c.x < j);
        if (lane == 0) cnt[j] = __popc(b);
        return;
    }
    if (lane != 0) return;
    Cand cd{face_vtx, vtx_slot, tp, o0};
    int32_t k = 0;
    for (int32_t q = 0; q < 2 * n; ++q) {
        int32_t x = cd.vert(q);
        if (x < j && cd.first(q, x)) ++k;
    }
    cnt[j] = k;
}

ALSUB_D void emit_edge(int32_t e, int32_t s_ij, int32_t s_ji, int32_t i, int32_t j, int32_t *face_edge, int32_t *face_twin,
                       int2 *edge_hh, uint32_t *bnd_word, int32_t *vbnd, int32_t *scalars) {
    if (s_ij >= 0) { face_edge[s_ij] = e; face_twin[s_ij] = s_ji; }
    if (s_ji >= 0) { face_edge[s_ji] = e; face_twin[s_ji] = s_ij; }
    const int32_t own = s_ij < 0 ? s_ji : (s_ji < 0 ? s_ij : min(s_ij, s_ji));
    const int32_t oth = s_ij < 0 || s_ji < 0 ? -1 : max(s_ij, s_ji);
    edge_hh[e] = make_int2(own, oth);
    if (oth < 0) {
        atomicOr(bnd_word + (e >> 5), 1u << (e & 31));
        atomicAdd(scalars + 1, 1);
        vbnd[i] = 1;
        vbnd[j] = 1;
    }
}

// numeric pass: ids, F(i,j) / F(j,i) as twin slots, multiplicity checks, boundary bits
__global__ void k_edge_fill(const int32_t *__restrict__ face_vtx, const int32_t *__restrict__ vtx_off,
                            const int32_t *__restrict__ vtx_slot, T0 tp, int32_t V,
                            const int32_t *__restrict__ edge_off, int32_t *__restrict__ face_edge,
                            int32_t *__restrict__ face_twin, int2 *__restrict__ edge_hh,
                            uint32_t *__restrict__ bnd_word, int32_t *__restrict__ vbnd,
                            int32_t *__restrict__ scalars, int32_t *flags) {
    const int32_t j = (int32_t)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (j >= V) return;
    const int32_t o0 = vtx_off[j], n = vtx_off[j + 1] - o0;
    if (n <= 16) {
        const WarpCand c = warp_cand(face_vtx, vtx_slot, tp, o0, n, lane);
        const bool mine = c.first && c.x < j;
        int32_t rank = 0;
        for (int k = 0; k < 32; ++k) {
            const int32_t xk = __shfl_sync(0xffffffffu, c.x, k);
            const unsigned b = __ballot_sync(0xffffffffu, c.first && c.x < xk);
            if (lane == k) rank = __popc(b);
        }
        // the directed slots of the edge among the candidate lanes: even lanes carry j -> x,
        // odd lanes x -> j; two of a kind = orientation error / non-manifold edge (E(i,j) > 2)
        const unsigned ev = c.peers & 0x55555555u, od = c.peers & 0xAAAAAAAAu;
        const int32_t s_ji = __shfl_sync(0xffffffffu, c.slot, ev ? __ffs(ev) - 1 : 0);
        const int32_t s_ij = __shfl_sync(0xffffffffu, c.slot, od ? __ffs(od) - 1 : 0);
        if (mine) {
            if (__popc(ev) > 1 || __popc(od) > 1) atomicOr(flags, kFlagNonManifold);
            emit_edge(edge_off[j] + rank, od ? s_ij : -1, ev ? s_ji : -1, c.x, j, face_edge, face_twin, edge_hh,
                      bnd_word, vbnd, scalars);
        }
        return;
    }
    if (lane != 0) return;
    Cand cd{face_vtx, vtx_slot, tp, o0};
    const int32_t nq = 2 * n;
    for (int32_t q = 0; q < nq; ++q) {
        int32_t i = cd.vert(q);
        if (i >= j || !cd.first(q, i)) continue;
        int32_t rank = 0;
        for (int32_t p = 0; p < nq; ++p) {
            int32_t x = cd.vert(p);
            if (x < i && cd.first(p, x)) ++rank;
        }
        int32_t s_ji = -1, s_ij = -1, m_ji = 0, m_ij = 0;
        for (int32_t a = 0; a < n; ++a) {
            int32_t h = cd.slot(2 * a);
            if (__ldg(face_vtx + tp.next(h)) == i) { s_ji = h; ++m_ji; }
            int32_t hp = tp.prev(h);
            if (__ldg(face_vtx + hp) == i) { s_ij = hp; ++m_ij; }
        }
        if (m_ji > 1 || m_ij > 1) atomicOr(flags, kFlagNonManifold);
        emit_edge(edge_off[j] + rank, s_ij, s_ji, i, j, face_edge, face_twin, edge_hh, bnd_word, vbnd, scalars);
    }
}

__global__ void k_slot0(const int32_t *__restrict__ vtx_off, const int32_t *__restrict__ vtx_slot, int32_t V,
                        int32_t *__restrict__ slot0) {
    int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    int32_t o = vtx_off[v];
    slot0[v] = vtx_off[v + 1] > o ? vtx_slot[o] : -1;
}

// a vertex whose interior faces form a closed fan that misses some incident face is non-manifold
// (reading R18); open fans (bowties) are allowed and end up as corners.
__global__ void k_check_fans(const int32_t *__restrict__ face_twin, const int32_t *__restrict__ vtx_off,
                             const int32_t *__restrict__ slot0, T0 tp, int32_t V, int32_t *flags) {
    int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    int32_t h0 = slot0[v];
    if (h0 < 0) return;
    int32_t deg = vtx_off[v + 1] - vtx_off[v];
    int32_t h = h0, n = 0;
    do {
        ++n;
        h = face_twin[tp.prev(h)];
    } while (h >= 0 && h != h0 && n <= deg);
    if (h == h0 && n != deg) atomicOr(flags, kFlagNonManifold);
}

__global__ void k_word_popc(const uint32_t *__restrict__ w, int32_t n, int32_t *__restrict__ c) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) c[i] = __popc(w[i]);
}

__global__ void k_crease_lookup(const int32_t *__restrict__ crease, const float *__restrict__ sigma, int32_t K,
                                const int32_t *__restrict__ face_vtx, const int32_t *__restrict__ vtx_off,
                                const int32_t *__restrict__ vtx_slot, const int32_t *__restrict__ face_edge,
                                const int2 *__restrict__ edge_hh, T0 tp,
                                int32_t V, float *__restrict__ edge_sigma, int32_t *__restrict__ edge_cidx,
                                int32_t *flags) {
    int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    int32_t a = crease[2 * k], b = crease[2 * k + 1];
    float sg = sigma[k];
    if (a < 0 || a >= V || b < 0 || b >= V || a == b || !(sg >= 0.0f)) { atomicOr(flags, kFlagCrease); return; }
    int32_t j = max(a, b), i = min(a, b), e = -1;
    for (int32_t p = vtx_off[j]; p < vtx_off[j + 1]; ++p) {
        int32_t h = vtx_slot[p];
        if (face_vtx[tp.next(h)] == i) { e = face_edge[h]; break; }
        int32_t hp = tp.prev(h);
        if (face_vtx[hp] == i) { e = face_edge[hp]; break; }
    }
    if (e < 0) { atomicOr(flags, kFlagCrease); return; }
    if (atomicCAS(edge_cidx + e, -1, k) != -1) { atomicOr(flags, kFlagCrease); return; }
    bool bnd = edge_hh[e].y < 0;
    if (sg > 0.0f && !bnd) edge_sigma[e] = sg;  // boundary edges are infinitely sharp anyway
}

__global__ void k_special_flag(const int2 *__restrict__ edge_hh, const float *__restrict__ edge_sigma, int32_t E,
                               int32_t *__restrict__ flag) {
    int32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    flag[e] = (edge_hh[e].y < 0 || edge_sigma[e] > 0.0f) ? 1 : 0;
}

__global__ void k_special_fill(const int2 *__restrict__ edge_hh, const int32_t *__restrict__ face_vtx,
                               const float *__restrict__ edge_sigma, const int32_t *__restrict__ flag,
                               const int32_t *__restrict__ off, T0 tp, int32_t E, SpEdge *__restrict__ sp,
                               int32_t *__restrict__ v_mark) {
    int32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E || !flag[e]) return;
    int32_t h = edge_hh[e].x;
    int32_t va = face_vtx[h], vb = face_vtx[tp.next(h)];
    bool bnd = edge_hh[e].y < 0;
    SpEdge s;
    s.e = e;
    s.a = min(va, vb);
    s.b = max(va, vb);
    s.ia = s.ib = -1;
    s.sigma = bnd ? __int_as_float(0x7f800000) : edge_sigma[e];
    s.flags = bnd ? kSpBoundary : 0;
    s.pad = 0;
    sp[off[e]] = s;
    v_mark[s.a] = 1;
    v_mark[s.b] = 1;
}

__global__ void k_sv_fill(const int32_t *__restrict__ v_mark, const int32_t *__restrict__ v_idx, int32_t V,
                          int32_t *__restrict__ sv_vtx) {
    int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < V && v_mark[v]) sv_vtx[v_idx[v]] = v;
}

__global__ void k_sp_index(SpEdge *__restrict__ sp, const int32_t *__restrict__ count,
                           const int32_t *__restrict__ v_idx, int32_t cap, int32_t *__restrict__ sv_cnt) {
    int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cap || j >= *count) return;
    const int32_t ia = v_idx[sp[j].a], ib = v_idx[sp[j].b];
    sp[j].ia = ia;
    sp[j].ib = ib;
    atomicAdd(sv_cnt + ia, 1);
    atomicAdd(sv_cnt + ib, 1);
}

// special-vertex CSR: incident special edges of every special vertex, ascending
__global__ void k_sv_list(const SpEdge *__restrict__ sp, const int32_t *__restrict__ count, int32_t cap,
                          const int32_t *__restrict__ sv_off, int32_t *__restrict__ sv_cur, int32_t *__restrict__ sv_list) {
    int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cap || j >= *count) return;
    const int32_t ia = sp[j].ia, ib = sp[j].ib;
    sv_list[sv_off[ia] + atomicAdd(sv_cur + ia, 1)] = j;
    sv_list[sv_off[ib] + atomicAdd(sv_cur + ib, 1)] = j;
}

__global__ void k_sv_sort(const int32_t *__restrict__ nsv, int32_t cap, const int32_t *__restrict__ sv_off,
                          int32_t *__restrict__ sv_list) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cap || i >= *nsv) return;
    const int32_t o = sv_off[i], n = sv_off[i + 1] - o;
    for (int32_t a = 1; a < n; ++a) {
        const int32_t x = sv_list[o + a];
        int32_t b = a - 1;
        while (b >= 0 && sv_list[o + b] > x) { sv_list[o + b + 1] = sv_list[o + b]; --b; }
        sv_list[o + b + 1] = x;
    }
}

// ------------------------------------------------------------------------------------------
void build0_validate(Build0 &b, cudaStream_t s, Launches &L) {
    if (b.F > 0) {
        k_validate_faces<<<grid_for(b.F), kThreads, 0, s>>>(b.face_off, b.face_vtx, b.F, b.V, b.slot_face, b.sort_k,
                                                            b.sort_v, b.flags);
        L.done("b0_validate", s);
    }
}

static int bits_for(int32_t V) {
    int bits = 1;
    while (bits < 31 && (1ll << bits) < (long long)V) ++bits;
    return bits;
}

void build0_count_edges(Build0 &b, cudaStream_t s, Launches &L) {
    T0 tp{b.face_off, b.slot_face};
    build0_validate(b, s, L);  // also (re)writes the sort input
    radix_sort_pairs(b.sort_k, b.sort_v, b.sort_k2, b.sort_v2, b.S, bits_for(b.V), b.scratch, s, L);
    offsets_from_sorted(b.sort_k, b.S, b.vtx_off, b.V, s, L);
    cudaMemcpyAsync(b.vtx_slot, b.sort_v, sizeof(int32_t) * (size_t)b.S, cudaMemcpyDeviceToDevice, s);
    if (b.V > 0) {
        k_edge_count<<<grid_for(32 * (int64_t)b.V), kThreads, 0, s>>>(b.face_vtx, b.vtx_off, b.vtx_slot, tp, b.V,
                                                                        b.edge_cnt);
        L.done("b0_edge_count", s);
    }
    scan_exclusive(b.edge_cnt, b.edge_off, b.V, b.scalars + 0, b.scratch, s, L);
}

void build0_fill(Build0 &b, bool check_fans, cudaStream_t s, Launches &L) {
    T0 tp{b.face_off, b.slot_face};
    const int32_t E = b.E;
    const int32_t nw = (int32_t)ceil_div(E > 0 ? E : 1, 32);
    cudaMemsetAsync(b.scalars + 1, 0, 3 * sizeof(int32_t), s);
    cudaMemsetAsync(b.bnd_word, 0, sizeof(uint32_t) * nw, s);
    if (b.V > 0) cudaMemsetAsync(b.vbnd, 0, sizeof(int32_t) * b.V, s);
    if (b.V > 0) {
        k_edge_fill<<<grid_for(32 * (int64_t)b.V), kThreads, 0, s>>>(b.face_vtx, b.vtx_off, b.vtx_slot, tp, b.V, b.edge_off,
                                                       b.face_edge, b.face_twin, b.edge_hh, b.bnd_word, b.vbnd,
                                                       b.scalars, b.flags);
        L.done("b0_edge_fill", s);
        k_slot0<<<grid_for(b.V), kThreads, 0, s>>>(b.vtx_off, b.vtx_slot, b.V, b.vtx_slot0);
        L.done("b0_slot0", s);
        if (check_fans) {
            k_check_fans<<<grid_for(b.V), kThreads, 0, s>>>(b.face_twin, b.vtx_off, b.vtx_slot0, tp, b.V, b.flags);
            L.done("b0_check_fans", s);
        }
    }
    k_word_popc<<<grid_for(nw), kThreads, 0, s>>>(b.bnd_word, nw, b.bnd_wcnt);
    L.done("b0_popc", s);
    scan_exclusive(b.bnd_wcnt, b.bnd_wpre, nw, nullptr, b.scratch, s, L);
    if (E > 0) {
        cudaMemsetAsync(b.edge_sigma, 0, sizeof(float) * E, s);
        cudaMemsetAsync(b.edge_cidx, 0xff, sizeof(int32_t) * E, s);
    }
    if (b.K_in > 0) {
        k_crease_lookup<<<grid_for(b.K_in), kThreads, 0, s>>>(b.crease_in, b.sigma_in, b.K_in, b.face_vtx, b.vtx_off,
                                                              b.vtx_slot, b.face_edge, b.edge_hh, tp,
                                                              b.V, b.edge_sigma, b.edge_cidx, b.flags);
        L.done("b0_crease_lookup", s);
    }
    if (E > 0) {
        k_special_flag<<<grid_for(E), kThreads, 0, s>>>(b.edge_hh, b.edge_sigma, E, b.sp_flag);
        L.done("b0_special_flag", s);
    }
    scan_exclusive(b.sp_flag, b.sp_off, E, b.scalars + 2, b.scratch, s, L);
    if (b.V > 0) cudaMemsetAsync(b.v_mark, 0, sizeof(int32_t) * b.V, s);
    if (E > 0 && b.sp) {
        k_special_fill<<<grid_for(E), kThreads, 0, s>>>(b.edge_hh, b.face_vtx, b.edge_sigma, b.sp_flag, b.sp_off, tp,
                                                        E, b.sp, b.v_mark);
        L.done("b0_special_fill", s);
    }
    scan_exclusive(b.v_mark, b.v_idx, b.V, b.scalars + 3, b.scratch, s, L);
    if (b.V > 0 && b.sv_vtx) {
        k_sv_fill<<<grid_for(b.V), kThreads, 0, s>>>(b.v_mark, b.v_idx, b.V, b.sv_vtx);
        L.done("b0_sv_fill", s);
    }
    if (b.V > 0) {
        cudaMemsetAsync(b.sv_cnt, 0, sizeof(int32_t) * b.V, s);
        cudaMemsetAsync(b.sv_cur, 0, sizeof(int32_t) * b.V, s);
    }
    if (E > 0) {
        k_sp_index<<<grid_for(E), kThreads, 0, s>>>(b.sp, b.scalars + 2, b.v_idx, E, b.sv_cnt);
        L.done("b0_sp_index", s);
    }
    scan_exclusive(b.sv_cnt, b.sv_off, b.V, b.sv_off + b.V, b.scratch, s, L);
    if (E > 0) {
        k_sv_list<<<grid_for(E), kThreads, 0, s>>>(b.sp, b.scalars + 2, E, b.sv_off, b.sv_cur, b.sv_list);
        L.done("b0_sv_list", s);
    }
    if (b.V > 0) {
        k_sv_sort<<<grid_for(b.V), kThreads, 0, s>>>(b.scalars + 3, b.V, b.sv_off, b.sv_list);
        L.done("b0_sv_sort", s);
    }
}

}  // namespace alsub
