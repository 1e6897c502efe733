// loop_sqrt3.cu -- the Loop (App. B) and sqrt3 (App. A) variants
// (SURVEY.md 8(a) rows a10, a11).  Same structure as cc.cu: per-face, per-edge and per-vertex
// gathers with closed-form child adjacency.
//
// Loop:   G(a,b) = vertex opposite the directed edge = face_vtx[prev(slot a->b)] (Eq. G);
//         e = 3/8 (p_a + p_b) + 1/8 (p_G(a,b) + p_G(b,a)) (reading R11);
//         S = (1 - n beta) p + beta sum p_j (Eq. loop_smooth);
//         children (k, e_kl, e_mk), (l, e_lm, e_kl), (m, e_mk, e_lm), (e_kl, e_lm, e_mk).
//         Child edge ids: the children of parent edge e are [(a,ep), (b,ep), (ep_x,ep) for the
//         distinct edges x < e sharing a triangle with e, ascending]; base_e = scan of counts.
// sqrt3:  f = barycenters; S = (1 - alpha) p + alpha/n sum p_j (Eqs. sqrt2, alpha);
//         child 3i+t = (p_k, fp_F(l,k), fp_i) (CCW reading R13); closed only.
#include <algorithm>

#include "internal.h"
#include "scan.cuh"

namespace alsub {

__constant__ float c_beta[65];   // Loop beta_n, n <= 64 (host: double -> fp32, reading R16)
__constant__ float c_alpha[65];  // sqrt3 alpha_n

ALSUB_D float loop_beta(int n) {
    if (n <= 64) return c_beta[n];
    const float c = 0.375f + 0.25f * cospif(2.0f / (float)n);
    return (0.625f - c * c) / (float)n;
}
ALSUB_D float sqrt3_alpha(int n) {
    if (n <= 64) return c_alpha[n];
    return (4.0f - 2.0f * cospif(2.0f / (float)n)) / 9.0f;
}

void init_scheme_tables(cudaStream_t s) {
    float beta[65], alpha[65];
    beta[0] = alpha[0] = 0.f;
    for (int n = 1; n <= 64; ++n) {
        double c = 0.375 + 0.25 * cos(2.0 * M_PI / n);
        beta[n] = (float)((0.625 - c * c) / n);
        alpha[n] = (float)((4.0 - 2.0 * cos(2.0 * M_PI / n)) / 9.0);
    }
    cudaMemcpyToSymbolAsync(c_beta, beta, sizeof(beta), 0, cudaMemcpyHostToDevice, s);
    cudaMemcpyToSymbolAsync(c_alpha, alpha, sizeof(alpha), 0, cudaMemcpyHostToDevice, s);
}

using T3 = Topo<3>;

// ------------------------------------------------------------------------------------------
// Loop
// ------------------------------------------------------------------------------------------
ALSUB_D int32_t tri_next(int32_t h) { int32_t t = h % 3; return t == 2 ? h - 2 : h + 1; }
ALSUB_D int32_t tri_prev(int32_t h) { int32_t t = h % 3; return t == 0 ? h + 2 : h - 1; }

// the (up to two) other edges of the face owning slot h
ALSUB_D void other_edges(const int32_t *face_edge, int32_t h, int32_t &x, int32_t &y) {
    x = __ldg(face_edge + tri_next(h));
    y = __ldg(face_edge + tri_prev(h));
}

// child-edge count of parent edge e: its two halves + one inner edge per distinct neighbour edge
// x < e of its faces; the exclusive scan of these counts is the block base of e's children
struct LoopCountSrc {
    LevelDev p;
    ALSUB_D int32_t operator()(int64_t ei) const {
        const int32_t e = (int32_t)ei;
        const int2 hh = __ldg(p.edge_hh + e);
        const int32_t h = hh.x, tw = hh.y;
        int32_t n[4];
        other_edges(p.face_edge, h, n[0], n[1]);
        n[2] = n[3] = INT32_MAX;
        if (tw >= 0) other_edges(p.face_edge, tw, n[2], n[3]);
        int32_t c = 2;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            bool dup = false;
#pragma unroll
            for (int k = 0; k < i; ++k) dup |= (n[k] == n[i]);
            c += (n[i] < e && !dup);
        }
        return c;
    }
};

// counts fused into the scan's load phase (one launch); `stat` = scan status words, zeroed by the
// refine's k_zero
void loop_edge_base(const LevelDev &p, int32_t *stat, int32_t *base, cudaStream_t s, Launches &L) {
    if (p.E <= 0) return;
    const int64_t tiles = ceil_div(p.E, kScanTile);
    launch(L, "loop_base", k_scan<LoopCountSrc>, dim3((unsigned)tiles), dim3(kScanThreads), 0, s, LoopCountSrc{p}, base,
           (int64_t)p.E, reinterpret_cast<unsigned long long *>(stat), (int32_t *)nullptr);
}

// id of the child edge between ep_x and ep_m inside a face (x < m): base_m + 2 + rank of x among
// the distinct neighbours of m (the other edges of m's two faces) -- all of which are compared with x.
ALSUB_D int32_t loop_inner(const LevelDev &p, int32_t m, int32_t x, int32_t z, int32_t m_twin) {
    int32_t n[3] = {z, INT32_MAX, INT32_MAX};
    if (m_twin >= 0) other_edges(p.face_edge, m_twin, n[1], n[2]);
    int32_t rank = 0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        bool dup = n[i] == x;
#pragma unroll
        for (int k = 0; k < i; ++k) dup |= (n[k] == n[i]);
        rank += (n[i] < x && !dup);
    }
    return __ldg(p.loop_base + m) + 2 + rank;
}

// a warp's 32 x 12 child-row ints (4 child triangles per face) staged in shared memory and written
// as 12 coalesced 128-B stores
// word q of the warp's 384 sits at q + q / 96: the stores of one k from lanes l, l + 8, l + 16,
// l + 24 (96 words apart) would otherwise share a bank (4-way conflicts)
ALSUB_D void warp_store_12(int32_t *stage, const int32_t (&v)[12], int32_t *dst, int64_t w0, int64_t n, int lane) {
#pragma unroll
    for (int k = 0; k < 12; ++k) {
        const int q = lane * 12 + k;
        stage[q + q / 96] = v[k];
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 12; ++k) {
        const int64_t o = w0 + k * 32 + lane;
        const int q = k * 32 + lane;
        if (o < n) dst[o] = stage[q + q / 96];
    }
    __syncwarp();
}

template <bool ADJ>
__global__ void __launch_bounds__(kThreads) k_loop_face(LevelDev p, ChildDev c) {
    ALSUB_GRID_WAIT();
    __shared__ int32_t s_stage[kThreads / 32][12 * 32 + 4];
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = r < p.F;
    const int lane = threadIdx.x & 31;
    int32_t *stage = s_stage[threadIdx.x >> 5];
    const int64_t w0 = 12 * (int64_t)(r - lane), n = 12 * (int64_t)p.F;
    const int32_t V = p.V;
    int32_t v[3], e[3];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        v[t] = valid ? __ldg(p.face_vtx + 3 * r + t) : 0;
        e[t] = valid ? __ldg(p.face_edge + 3 * r + t) : 0;
    }
    int32_t rows[12];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        rows[3 * t + 0] = v[t];
        rows[3 * t + 1] = V + e[t];
        rows[3 * t + 2] = V + e[(t + 2) % 3];
    }
    rows[9] = V + e[0];
    rows[10] = V + e[1];
    rows[11] = V + e[2];
    warp_store_12(stage, rows, c.face_vtx, w0, n, lane);
    if constexpr (ADJ) {
        int32_t tw[3];
#pragma unroll
        for (int t = 0; t < 3; ++t) tw[t] = valid ? __ldg(p.face_twin + 3 * r + t) : -1;
        // inner edge between edges i and j of this face
        auto inner = [&](int i, int j) {
            const int k = 3 - i - j;  // the third edge
            const int mi = e[i] > e[j] ? i : j, xi = e[i] > e[j] ? j : i;
            return loop_inner(p, e[mi], e[xi], e[k], tw[mi]);
        };
        int32_t in01 = 0, in12 = 0, in20 = 0;
        if (valid) {
            in01 = inner(0, 1);
            in12 = inner(1, 2);
            in20 = inner(2, 0);
        }
        const int32_t inner_t_tm1[3] = {in20, in01, in12};  // between e_t and e_{t-1}
        int32_t fe[12], ft[12];
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            const int tn = (t + 1) % 3, tp = (t + 2) % 3;
            fe[3 * t + 0] = valid ? __ldg(p.loop_base + e[t]) + (v[t] > v[tn]) : 0;
            fe[3 * t + 1] = inner_t_tm1[t];
            fe[3 * t + 2] = valid ? __ldg(p.loop_base + e[tp]) + (v[t] > v[tp]) : 0;
            const int32_t a = tw[t], b = tw[tp];
            ft[3 * t + 0] = a >= 0 ? 3 * (4 * (a / 3) + (a % 3 + 1) % 3) + 2 : -1;
            ft[3 * t + 1] = 3 * (4 * r + 3) + tp;
            ft[3 * t + 2] = b >= 0 ? 3 * (4 * (b / 3) + b % 3) + 0 : -1;
            if (valid) c.edge_hh[inner_t_tm1[t]] = make_int2(12 * r + 3 * t + 1, 3 * (4 * r + 3) + tp);
        }
        fe[9] = in01;
        fe[10] = in12;
        fe[11] = in20;
        ft[9] = 3 * (4 * r + 1) + 1;
        ft[10] = 3 * (4 * r + 2) + 1;
        ft[11] = 3 * (4 * r + 0) + 1;
        warp_store_12(stage, fe, c.face_edge, w0, n, lane);
        warp_store_12(stage, ft, c.face_twin, w0, n, lane);
    }
}

ALSUB_D int32_t loop_c0(int32_t x) { return 12 * (x / 3) + 3 * (x % 3); }
ALSUB_D int32_t loop_c2next(int32_t x) { return 3 * (4 * (x / 3) + (x % 3 + 1) % 3) + 2; }

// IT edges per thread, every load stage issued for all of them before any is consumed (the
// kernel is a chain edge pair -> face row -> positions)
template <bool ADJ, int IT = 2>
__global__ void __launch_bounds__(kThreads) k_loop_edge(LevelDev p, ChildDev c, Frames fr) {
    ALSUB_GRID_WAIT();
    const int32_t e0 = blockIdx.x * (kThreads * IT) + threadIdx.x;
    const int32_t V = p.V;
    int2 hh[IT];
#pragma unroll
    for (int k = 0; k < IT; ++k) {
        const int32_t e = e0 + k * kThreads;
        hh[k] = e < p.E ? __ldg(p.edge_hh + e) : make_int2(0, -1);
    }
    int32_t va[IT], vb[IT], g1[IT], g2[IT];
#pragma unroll
    for (int k = 0; k < IT; ++k) {
        const int32_t h = hh[k].x, tw = hh[k].y;
        va[k] = __ldg(p.face_vtx + h);
        vb[k] = __ldg(p.face_vtx + tri_next(h));
        g1[k] = __ldg(p.face_vtx + tri_prev(h));
        g2[k] = tw >= 0 ? __ldg(p.face_vtx + tri_prev(tw)) : -1;
    }
    for (int f = 0; f < fr.nb; ++f) {
        const PR P = fr.rd(f);
        P3 ab[IT], gg[IT];
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            ab[k] = ld3(P, va[k]) + ld3(P, vb[k]);
            gg[k] = hh[k].y >= 0 ? ld3(P, g1[k]) + ld3(P, g2[k]) : p3zero();
        }
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            const int32_t e = e0 + k * kThreads;
            if (e >= p.E) continue;
            const P3 out = hh[k].y < 0 ? 0.5f * ab[k] : 0.375f * ab[k] + 0.125f * gg[k];
            st3(fr.wr(f), (int64_t)V + e, out);
        }
    }
    if constexpr (ADJ) {
        auto pair = [](int32_t x, int32_t y) {
            if (x < 0) return make_int2(y, -1);
            if (y < 0) return make_int2(x, -1);
            return make_int2(min(x, y), max(x, y));
        };
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            const int32_t e = e0 + k * kThreads;
            if (e >= p.E) continue;
            const int32_t h = hh[k].x, tw = hh[k].y;
            const int32_t base = __ldg(p.loop_base + e);
            const int32_t h_ab = va[k] < vb[k] ? h : tw, h_ba = va[k] < vb[k] ? tw : h;
            // (lo,ep): lo->ep in the child of h_ab, ep->lo in the child after h_ba; (hi,ep) symmetric
            c.edge_hh[base + 0] = pair(h_ab >= 0 ? loop_c0(h_ab) : -1, h_ba >= 0 ? loop_c2next(h_ba) : -1);
            c.edge_hh[base + 1] = pair(h_ba >= 0 ? loop_c0(h_ba) : -1, h_ab >= 0 ? loop_c2next(h_ab) : -1);
        }
    }
}

// Vertex kernel, class-structured like the CC one (no twin walk): level-l vertex ids are
// [V0 | E_0 | E_1 | ... | E_{l-1}] (level-0 vertices, then the edge points born at each level).
// A vertex's incident slots are closed-form at its birth level -- level-0 vertices: their M^T row;
// the edge point of level-(m-1) slot h = 3R + t: {12R + 3t + 1, 12R + 3((t+1)%3) + 2, 12R + 9 + t}
// and the same for its twin slot -- and every later level maps a slot x to corner 0 of the child
// at that corner, c0(x) = 12(x/3) + 3(x%3).  The neighbours are face_vtx[next(slot)], all loads
// independent.  S = (1 - n beta_n) p + beta_n sum p_j (Eq. loop vertex); boundary vertices keep p
// (the crease module sets them, boundary = inf crease).

template <bool ADJ>
__global__ void __launch_bounds__(kThreads) k_loop_vertex(LevelDev p, ChildDev c, Frames fr, VSegs g) {
    ALSUB_GRID_WAIT();
    const int32_t v0 = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = v0 < p.V;
    const int32_t v = valid ? v0 : p.V - 1;
    int s = g.nseg - 1;
    while (s > 0 && v < g.start[s]) --s;
    const int32_t j = v - g.start[s];
    const int hops = g.level - g.birth[s];
    const bool lv0 = g.type[s] == 0;
    int32_t n = 0, o = 0;
    int32_t R[2] = {0, 0}, T[2] = {0, 0};
    bool bnd = false;
    if (lv0) {
        o = __ldg(g.vtx_off0 + j);
        n = __ldg(g.vtx_off0 + j + 1) - o;
        bnd = __ldg(g.vbnd0 + j) != 0;
    } else {
        const int2 hh = __ldg(g.ehh[g.birth[s] - 1] + j);
        bnd = hh.y < 0;
        n = 6;
        R[0] = hh.x / 3; T[0] = hh.x % 3;
        R[1] = hh.y / 3; T[1] = hh.y % 3;
    }
    // birth slot k, mapped `hops` levels down to this level
    auto slot = [&](int32_t k) {
        int32_t x;
        if (lv0) {
            x = __ldg(g.vtx_list0 + o + k);
        } else {
            const int q = k >= 3, u = k - 3 * q;
            const int32_t r = q ? R[1] : R[0], t = q ? T[1] : T[0];
            x = u == 0 ? 12 * r + 3 * t + 1 : (u == 1 ? 12 * r + 3 * ((t + 1) % 3) + 2 : 12 * r + 9 + t);
        }
        for (int h = 0; h < hops; ++h) x = loop_c0(x);
        return x;
    };
    // long level-0 rings: summed by the whole warp after the per-lane pass
    const bool lng = valid && lv0 && !bnd && n > kLongRing;
    for (int f = 0; f < fr.nb && valid && !lng; ++f) {
        const PR P = fr.rd(f);
        const PW Pn = fr.wr(f);
        const P3 pv = ld3(P, v);
        if (bnd || n == 0) { st3(Pn, v, pv); continue; }
        P3 acc = p3zero();
        for (int32_t k0 = 0; k0 < n; k0 += 4) {  // four independent neighbour lookups in flight
            int32_t nb[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) nb[u] = k0 + u < n ? __ldg(p.face_vtx + tri_next(slot(k0 + u))) : -1;
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (nb[u] >= 0) acc = acc + ld3(P, nb[u]);
        }
        const float beta = loop_beta(n);
        st3(Pn, v, (1.0f - (float)n * beta) * pv + beta * acc);
    }
    const int lane = threadIdx.x & 31;
    unsigned m = __ballot_sync(0xffffffffu, lng);
    while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const int32_t jj = __shfl_sync(0xffffffffu, j, src), vv = __shfl_sync(0xffffffffu, v, src);
        const int32_t oo = __ldg(g.vtx_off0 + jj), nn = __ldg(g.vtx_off0 + jj + 1) - oo;
        const float beta = loop_beta(nn);
        for (int f = 0; f < fr.nb; ++f) {
            const PR P = fr.rd(f);
            P3 acc = p3zero();
            for (int32_t k0 = lane; k0 < nn; k0 += 32 * 8) {  // 8 independent chains per lane
                int32_t x[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) x[u] = k0 + 32 * u < nn ? __ldg(g.vtx_list0 + oo + k0 + 32 * u) : -1;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (x[u] < 0) continue;
                    for (int h = 0; h < g.level; ++h) x[u] = loop_c0(x[u]);  // born at level 0 (the lane's
                    x[u] = __ldg(p.face_vtx + tri_next(x[u]));             // own segment may differ)
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (x[u] >= 0) acc = acc + ld3(P, x[u]);
            }
            acc = warp_sum(acc);
            if (lane == 0) st3(fr.wr(f), vv, (1.0f - (float)nn * beta) * ld3(P, vv) + beta * acc);
        }
    }
}

// stat / base: the child-edge base scan of this level (nullptr: not needed -- last level without
// creases).  Dependencies: face and edge kernels need the bases, the vertex kernel does not.  The
// vertex kernel launches first on the main stream (programmatic launch after the previous level),
// the scan and the edge kernel run on the side branch, and the face kernel follows the vertex
// kernel once the scan is done (torus100k Loop L4 0.551 -> 0.547 ms, ico L6 0.070 -> 0.068 ms
// against the vertex kernel on the side branch).
void loop_level(const LevelDev &p, const ChildDev &c, const Frames &fr, bool topo, bool adj, int32_t *stat,
                int32_t *base, const VSegs &g, cudaStream_t s, Launches &L, int crease) {
    const bool A = adj && topo;
    const bool fork = L.can_fork();
    // (config 2b, creased tet Loop L6: 0.096 -> 0.093 ms against the crease pass after the join)
    const bool side_crease = crease >= 0 && fork && L.ev_aux;
    cudaStream_t se = s;
    if (fork) {
        cudaEventRecord(L.ev_fork, s);
        cudaStreamWaitEvent(L.side, L.ev_fork, 0);
        se = L.side;
    }
    if (p.V > 0) {
        if (A) launch(L, "loop_vertex", k_loop_vertex<true>, dim3(grid_for(p.V)), dim3(kThreads), 0, s, p, c, fr, g);
        else launch(L, "loop_vertex", k_loop_vertex<false>, dim3(grid_for(p.V)), dim3(kThreads), 0, s, p, c, fr, g);
    }
    if (side_crease) cudaEventRecord(L.ev_aux, s);
    if (base) {
        loop_edge_base(p, stat, base, se, L);
        if (fork) {  // the face kernel (main) waits for the bases
            cudaEventRecord(L.ev_fork, se);
            cudaStreamWaitEvent(s, L.ev_fork, 0);
        }
    }
    if (p.E > 0) {
        if (A) launch(L, "loop_edge", k_loop_edge<true>, dim3(grid_for(p.E, 2 * kThreads)), dim3(kThreads), 0, se, p, c, fr);
        else launch(L, "loop_edge", k_loop_edge<false>, dim3(grid_for(p.E, 2 * kThreads)), dim3(kThreads), 0, se, p, c, fr);
    }
    if (side_crease) {  // overrides need the edge points (this branch) and the vertex points (ev_aux)
        cudaStreamWaitEvent(se, L.ev_aux, 0);
        crease_level(p, c, fr, p.V, 1, crease == 1, se, L);
    }
    if (topo && p.F > 0) {
        if (A) launch(L, "loop_face", k_loop_face<true>, dim3(grid_for(p.F)), dim3(kThreads), 0, s, p, c);
        else launch(L, "loop_face", k_loop_face<false>, dim3(grid_for(p.F)), dim3(kThreads), 0, s, p, c);
    }
    if (fork) {
        cudaEventRecord(L.ev_join, L.side);
        cudaStreamWaitEvent(s, L.ev_join, 0);
    }
    if (crease >= 0 && !side_crease) crease_level(p, c, fr, p.V, 1, crease == 1, s, L);
}

// ------------------------------------------------------------------------------------------
// sqrt3
// ------------------------------------------------------------------------------------------
// face kernel: barycenter (P:L1010 with (1,2,3) -> 1/3) and the three children (p_k, fp_F(l,k), fp_i)
// (CCW reading R13) + child twins; a warp's 32 x 36 B of child rows are staged in
// shared memory and written as 9 coalesced 128 B stores.
ALSUB_D void warp_store_9(int32_t *stage, const int32_t (&v)[9], int32_t *dst, int64_t w0, int64_t n, int lane) {
#pragma unroll
    for (int k = 0; k < 9; ++k) stage[lane * 9 + k] = v[k];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        const int64_t o = w0 + k * 32 + lane;
        if (o < n) dst[o] = stage[k * 32 + lane];
    }
    __syncwarp();
}

template <bool ADJ, int NBC>
__global__ void __launch_bounds__(kThreads) k_s3_face(LevelDev p, ChildDev c, Frames fr, bool topo) {
    ALSUB_GRID_WAIT();
    __shared__ int32_t s_stage[kThreads / 32][9 * 32];
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = i < p.F;
    const int lane = threadIdx.x & 31;
    const int32_t V = p.V;
    int32_t v[3], tw[3];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        v[t] = valid ? __ldg(p.face_vtx + 3 * i + t) : 0;
        tw[t] = valid ? __ldg(p.face_twin + 3 * i + t) : 0;
    }
    const int nb = NBC ? NBC : fr.nb;
    for (int f = 0; f < nb; ++f) {
        const PR P = fr.rd(f);
        const P3 s = ld3w(P, v[0]) + ld3w(P, v[1]) + ld3w(P, v[2]);
        if (valid) st3(fr.wr(f), (int64_t)V + i, (1.0f / 3.0f) * s);
    }
    if (!topo) return;
    int32_t *stage = s_stage[threadIdx.x >> 5];
    const int64_t w0 = 9 * (int64_t)(i - lane), n = 9 * (int64_t)p.F;
    int32_t rows[9];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        rows[3 * t + 0] = v[t];
        rows[3 * t + 1] = V + tw[t] / 3;
        rows[3 * t + 2] = V + i;
    }
    warp_store_9(stage, rows, c.face_vtx, w0, n, lane);
    if constexpr (ADJ) {
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            const int32_t a = tw[t], b = tw[(t + 2) % 3];
            const int32_t na = a / 3, ua = a % 3, nb2 = b / 3, wb = b % 3;
            rows[3 * t + 0] = 3 * (3 * na + (ua + 1) % 3) + 2;
            rows[3 * t + 1] = 3 * (3 * na + ua) + 1;
            rows[3 * t + 2] = 3 * (3 * nb2 + wb) + 0;
        }
        warp_store_9(stage, rows, c.face_twin, w0, n, lane);
    }
}

// vertex kernel: S = (1 - alpha) p + alpha/n sum p_j (Eqs. sqrt2, alpha) over the closed-form row
// of M of every vertex class: a vertex born at level m has level-l slots
// 3^(l-m) x its level-m slots; a face point of face i (level m-1) has level-m slots
// {9i + 3t + 2} u {3 tw_t + 1}; face points born at this level read their six neighbours straight
// from the parent rows (the triangle's corners and the three neighbouring face points).
template <int NBC>
__global__ void __launch_bounds__(kThreads) k_s3_vertex(LevelDev p, Frames fr, VSegs g) {
    ALSUB_GRID_WAIT();
    __shared__ int32_t s_lo[kMaxSeg], s_pre[kMaxSeg + 1];
    const int64_t nblk = gridDim.x, b = blockIdx.x;
    // warp 0: this block's task range of every segment (nseg = 1 + l <= 16) and their exclusive
    // prefix by a shuffle scan (one barrier)
    if (threadIdx.x < 32) {
        int32_t lo = 0, cnt = 0;
        if ((int)threadIdx.x < g.nseg) {
            const int64_t tasks = (g.len[threadIdx.x] + 31) >> 5;
            lo = (int32_t)(b * tasks / nblk);
            cnt = (int32_t)((b + 1) * tasks / nblk) - lo;
        }
        int32_t inc = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int32_t o = __shfl_up_sync(0xffffffffu, inc, d);
            if ((int)threadIdx.x >= d) inc += o;
        }
        if ((int)threadIdx.x < g.nseg) {
            s_lo[threadIdx.x] = lo;
            s_pre[threadIdx.x] = inc - cnt;
        }
        if ((int)threadIdx.x == g.nseg - 1) s_pre[g.nseg] = inc;
    }
    __syncthreads();
    const int32_t ntask = s_pre[g.nseg];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    const int nb = NBC ? NBC : fr.nb;
    int s = 0;
    for (int32_t task = warp; task < ntask; task += nwarp) {
        while (s_pre[s + 1] <= task) ++s;
        const int32_t j = ((s_lo[s] + (task - s_pre[s])) << 5) + lane;
        const int32_t mult = g.mult[s];
        const bool closed = g.level >= 1;
        const int32_t vfp = g.start[g.nseg - 1];  // first face point born at this level (= V_{l-1})
        if (g.type[s] == 0) {  // warp-uniform: long level-0 rings summed by the whole warp
            const bool lng = j < g.len[s] && __ldg(g.vtx_off0 + j + 1) - __ldg(g.vtx_off0 + j) > kLongRing;
            unsigned m = __ballot_sync(0xffffffffu, lng);
            while (m) {
                const int src = __ffs(m) - 1;
                m &= m - 1;
                const int32_t jj = j - lane + src, vv = g.start[s] + jj;
                const int32_t oo = __ldg(g.vtx_off0 + jj), nn = __ldg(g.vtx_off0 + jj + 1) - oo;
                const float alpha = sqrt3_alpha(nn);
                for (int f = 0; f < nb; ++f) {
                    const PR P = fr.rd(f);
                    P3 acc = p3zero();
                    for (int32_t k0 = lane; k0 < nn; k0 += 32 * 8) {  // 8 independent chains per lane
                        int32_t q[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) q[u] = k0 + 32 * u < nn ? __ldg(g.vtx_list0 + oo + k0 + 32 * u) * mult : -1;
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (q[u] >= 0) q[u] = closed ? vfp + q[u] / 9 : __ldg(p.face_vtx + tri_next(q[u]));
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (q[u] >= 0) acc = acc + ld3w(P, q[u]);
                    }
                    acc = warp_sum(acc);
                    if (lane == 0) st3(fr.wr(f), vv, (1.0f - alpha) * ld3w(P, vv) + (alpha / (float)nn) * acc);
                }
            }
            if (lng) continue;
        }
        if (j >= g.len[s]) continue;
        const int32_t v = g.start[s] + j;
        if (g.type[s] == 1 && g.birth[s] == g.level) {
            // face point of parent face j: neighbours = its corners + the 3 adjacent face points
            const int m1 = g.birth[s] - 1;
            int32_t nbv[6];
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                nbv[t] = __ldg(g.fvx[m1] + 3 * j + t);
                nbv[3 + t] = g.start[s] + __ldg(g.ftw[m1] + 3 * j + t) / 3;
            }
            constexpr float alpha = 1.0f / 3.0f;  // alpha_6 = (4 - 2 cos(pi/3)) / 9
            for (int f = 0; f < nb; ++f) {
                const PR P = fr.rd(f);
                P3 acc = ld3w(P, nbv[0]);
#pragma unroll
                for (int k = 1; k < 6; ++k) acc = acc + ld3w(P, nbv[k]);
                st3(fr.wr(f), v, (1.0f - alpha) * ld3w(P, v) + (alpha / 6.0f) * acc);
            }
            continue;
        }
        int32_t sl[6];
        int32_t n = 0;
        const int32_t *list = nullptr;
        if (g.type[s] == 1) {
            const int m1 = g.birth[s] - 1;
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                sl[t] = (9 * j + 3 * t + 2) * mult;
                sl[3 + t] = (3 * __ldg(g.ftw[m1] + 3 * j + t) + 1) * mult;
            }
            n = 6;
        } else {
            const int32_t o = __ldg(g.vtx_off0 + j);
            n = __ldg(g.vtx_off0 + j + 1) - o;
            list = g.vtx_list0 + o;
        }
        const float alpha = n > 0 ? sqrt3_alpha(n) : 0.0f;
        // level >= 1: every neighbour of an old vertex is a face point born at this level, the one
        // of the level-(l-1) face (slot / 9) holding the vertex's level-l slot -- no face lookup
        for (int f = 0; f < nb; ++f) {
            const PR P = fr.rd(f);
            const PW Pn = fr.wr(f);
            const P3 pv = ld3w(P, v);
            if (n == 0) { st3(Pn, v, pv); continue; }
            P3 acc = p3zero();
            if (list) {
                for (int32_t k = 0; k < n; ++k) {
                    const int32_t sk = __ldg(list + k) * mult;
                    acc = acc + ld3w(P, closed ? vfp + sk / 9 : __ldg(p.face_vtx + tri_next(sk)));
                }
            } else {
                int32_t nbv[6];
#pragma unroll
                for (int k = 0; k < 6; ++k) nbv[k] = closed ? vfp + sl[k] / 9 : __ldg(p.face_vtx + tri_next(sl[k]));
#pragma unroll
                for (int k = 0; k < 6; ++k) acc = acc + ld3w(P, nbv[k]);
            }
            st3(Pn, v, (1.0f - alpha) * pv + (alpha / (float)n) * acc);
        }
    }
}

void sqrt3_level(const LevelDev &p, const ChildDev &c, const Frames &fr, bool topo, bool adj, const VSegs &g,
                 cudaStream_t s, Launches &L) {
    const bool A = adj && topo;
    const bool one = fr.nb == 1;
    // the vertex kernel reads only level-l positions and writes the old vertices, the face kernel
    // the new face points (and the child topology): independent parallel branches. The gather-bound
    // vertex kernel is the
    // longer one once it shares the GPU with the bandwidth-bound face kernel, so it is launched
    // FIRST, on the main stream (programmatic launch after the previous level, first pick of SM
    // slots), and the face kernel takes the side branch (config 4 0.3625 -> 0.348 ms; face first
    // with the vertex kernel on the side: its CTAs wait for slots, 68 -> 182 us live)
    const bool fork = L.can_fork();
    cudaStream_t sv = s, sf = s;
    if (fork) {
        cudaEventRecord(L.ev_fork, s);
        cudaStreamWaitEvent(L.side, L.ev_fork, 0);
        sf = L.side;
    }
    auto face = [&]() {
        if (p.F <= 0) return;
        if (A) {
            if (one) launch(L, "s3_face", k_s3_face<true, 1>, dim3(grid_for(p.F)), dim3(kThreads), 0, sf, p, c, fr, topo);
            else launch(L, "s3_face", k_s3_face<true, 0>, dim3(grid_for(p.F)), dim3(kThreads), 0, sf, p, c, fr, topo);
        } else {
            if (one) launch(L, "s3_face", k_s3_face<false, 1>, dim3(grid_for(p.F)), dim3(kThreads), 0, sf, p, c, fr, topo);
            else launch(L, "s3_face", k_s3_face<false, 0>, dim3(grid_for(p.F)), dim3(kThreads), 0, sf, p, c, fr, topo);
        }
    };
    auto vertex = [&]() {
        if (p.V <= 0) return;
        const unsigned nblk = (unsigned)std::max<int64_t>(grid_for(p.V, 4 * kThreads),
                                                          std::min<int64_t>(grid_for(p.V, kThreads), 2 * 148));
        if (one) launch(L, "s3_vertex", k_s3_vertex<1>, dim3(nblk), dim3(kThreads), 0, sv, p, fr, g);
        else launch(L, "s3_vertex", k_s3_vertex<0>, dim3(nblk), dim3(kThreads), 0, sv, p, fr, g);
    };
    vertex();
    face();
    if (fork) {
        cudaEventRecord(L.ev_join, L.side);
        cudaStreamWaitEvent(s, L.ev_join, 0);
    }
}

}  // namespace alsub
