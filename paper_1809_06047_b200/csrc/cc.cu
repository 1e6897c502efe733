// cc.cu -- one Catmull-Clark level (SURVEY.md 8(a) rows a3', a4-a6, a8).
//
// Three gather kernels per level, each parallel over the items it WRITES so that every store is
// coalesced and no float atomics are needed (replacing the paper's direct SpMV with atomics,
// P:L622-627, by deterministic gathers):
//   k_cc_face*   per parent face r: f_r = M^T P with val -> 1/c_r and the child
//                faces (v_t, ep(v_t,v_t+1), fp_r, ep(v_t-1,v_t)) = M_{i+1}'s columns;
//                when another level follows, also the child face_edge / face_twin / vertex slot
//                in closed form (the structured edge ids of DESIGN.md, no sort, no SpGEMM).
//   k_cc_edge    per parent edge e: e = 1/4 (p_k + p_l + f_r + f_s), boundary
//                midpoint; child edge owners for the next level.
//   k_cc_vertex  per parent vertex: S(p) = (1 - 2/n) p + 1/n^2 sum_{incident slots}(p_next + f)
//                = s1 + s2 + s3 of P:L332-357 (s2 = F P, s3 = M f) via a 1-ring walk.
// Boundary vertices and creases are overwritten afterwards by crease.cu (boundary = inf crease).
#include <algorithm>

#include "crease_fused.cuh"
#include "internal.h"

namespace alsub {

// base id of the child-edge block of parent edge e: sum_{e' < e} (4 - bnd_e')
template <bool BND>
ALSUB_D int32_t cc_base(const uint32_t *w, const int32_t *wp, int32_t e) {
    if constexpr (BND) return 4 * e - bprefix(w, wp, e);
    else return 4 * e;
}

// ---------------- face kernel: reduced quad matrix (levels >= 1, or all-quad input) --------
// Each thread owns one parent quad and produces 4 child rows (64 B) per output array; a warp's
// 32 x 64 B = 2 KB are staged in shared memory and written back as 4 fully coalesced 512 B
// stores (child rows 4 r0 .. 4 r0 + 127 are contiguous).  Row t of lane l sits at slot
// 4 l + ((t + l/2) mod 4): with the plain slot 4 l + t the 32 lanes' 16-B stores of one t fall on
// 8 of the 32 banks (16 wavefronts instead of 4 -- ncu showed the kernel L1-data-pipe bound on
// these conflicts); the rotation spreads them over all banks, and the read-back (four lanes per
// source lane, a permutation of its 4 slots) stays conflict-free.
ALSUB_D void warp_store_rows(int4 *stage, const int4 (&rows)[4], int4 *dst, int64_t row0, int64_t nrows, int lane) {
#pragma unroll
    for (int t = 0; t < 4; ++t) stage[lane * 4 + ((t + (lane >> 1)) & 3)] = rows[t];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t rr = row0 + k * 32 + lane;
        const int src = k * 8 + (lane >> 2), t = lane & 3;
        if (rr < nrows) dst[rr] = stage[src * 4 + ((t + (src >> 1)) & 3)];
    }
    __syncwarp();
}

// the edge-id row of level-l face r = child (R, t) of level-(l-1) quad R, in closed form from R's
// rows (what the level-(l-1) face kernel would have stored as face_edge; used at the last level)
ALSUB_D int4 child_edge_row(const LevelDev &gp, int32_t r) {
    const int32_t R = r >> 2, t = r & 3, tn = (t + 1) & 3, tp = (t + 3) & 3;
    const int4 a = __ldg(reinterpret_cast<const int4 *>(gp.face_vtx) + R);
    const int4 b = __ldg(reinterpret_cast<const int4 *>(gp.face_edge) + R);
    const int4 c = __ldg(reinterpret_cast<const int4 *>(gp.face_twin) + R);
    const int32_t v[4] = {a.x, a.y, a.z, a.w}, e[4] = {b.x, b.y, b.z, b.w}, tw[4] = {c.x, c.y, c.z, c.w};
    const int32_t bt = 4 * e[t] - (gp.B > 0 ? bprefix(gp.bnd_word, gp.bnd_wpre, e[t]) : 0);
    const int32_t bq = 4 * e[tp] - (gp.B > 0 ? bprefix(gp.bnd_word, gp.bnd_wpre, e[tp]) : 0);
    const int32_t h = 4 * R + t, hp = 4 * R + tp;
    return make_int4(bt + (v[t] > v[tn]), bt + 2 + (tw[t] >= 0 && tw[t] < h), bq + 2 + (tw[tp] >= 0 && tw[tp] < hp),
                     bq + (v[t] > v[tp]));
}

// fpo >= 0 (levels l >= 3): first id of the face points born at level l-1.  The face point of
// level-(l-2) quad j is corner 0 of exactly the four level-l faces 16 j + 4 t + 2 (t = 0..3, the
// corner-2 children of its four level-(l-1) faces), i.e. lanes 2, 6, 10, 14 of a 16-lane group:
// its vertex point 1/2 p + 1/16 sum_t c0[16 j + 4 t + 2] is a shuffle reduction here instead of
// four c0 gathers in the vertex kernel.
template <bool ADJ, bool BND, int NBC, bool GPE>
__global__ void __launch_bounds__(kThreads, NBC ? (ADJ ? 6 : 8) : 0) k_cc_face_quad(LevelDev p, ChildDev c, Frames fr, bool topo, bool fpv,
                                                         LevelDev gp, int32_t fpo) {
    ALSUB_GRID_WAIT();
    __shared__ int4 s_stage[kThreads / 32][128];
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = r < p.F;
    const int lane = threadIdx.x & 31;
    int4 *stage = s_stage[threadIdx.x >> 5];
    const int4 fv = valid ? __ldg(reinterpret_cast<const int4 *>(p.face_vtx) + r) : make_int4(0, 0, 0, 0);
    const int32_t v[4] = {fv.x, fv.y, fv.z, fv.w};
    const int32_t V = p.V, F = p.F;
    const int nb = NBC ? NBC : fr.nb;
    // edge-id row: loaded (or recomputed from the grandparent rows) up front so that its loads are
    // in flight together with the position gathers
    int4 fe = make_int4(0, 0, 0, 0);
    if (topo && valid) {
        if constexpr (GPE) fe = child_edge_row(gp, r);
        else fe = __ldg(reinterpret_cast<const int4 *>(p.face_edge) + r);
    }
    for (int f = 0; f < nb; ++f) {
        const PR P = fr.rd(f);
        const PW Pn = fr.wr(f);
        const P3 p0 = ld3(P, v[0]), p1 = ld3(P, v[1]), p2 = ld3(P, v[2]), p3 = ld3(P, v[3]);
        const P3 fc = 0.25f * (p0 + p1 + p2 + p3);
        if (valid) st3(Pn, V + r, fc);
        if (valid && fr.c0 && (r & ((1 << fr.c0shift) - 1)) == 0) st3(fr.c0w(f), r >> fr.c0shift, p1 + fc);
        if (fpo >= 0) {
            P3 acc = p1 + fc;
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 4);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 4);
            acc.z += __shfl_xor_sync(0xffffffffu, acc.z, 4);
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 8);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 8);
            acc.z += __shfl_xor_sync(0xffffffffu, acc.z, 8);
            if (valid && (lane & 15) == 2) st3(Pn, (int64_t)fpo + (r >> 4), 0.5f * p0 + 0.0625f * acc);
        }
        if (fpv) {
            // (1) the edge point of parent slot r (born at this level) sits at corner 1 of child
            // r and corner 3 of child r+1 (mod 4): its half ring sum from this parent face is
            // (p2 + f_r) + (p0 + f_{r+1}); the vertex kernel adds the two halves of the edge
            // (at the last level the edge kernel finishes these vertices itself, see k_cc_edge_gp)
            // (not needed when the edge kernel iterates the grandparent edges: fr.hs = nullptr)
            if (!GPE && fr.hs != nullptr) {
                const P3 q = p0 + fc;
                const int src = (lane & ~3) | ((lane + 1) & 3);
                P3 qn;
                qn.x = __shfl_sync(0xffffffffu, q.x, src);
                qn.y = __shfl_sync(0xffffffffu, q.y, src);
                qn.z = __shfl_sync(0xffffffffu, q.z, src);
                if (valid) st3(fr.hsw(f), r, p2 + fc + qn);
            }
            // (2) corner 2 of the four children of a quad is the parent's face point (born at this
            // level, valence 4): its vertex point needs exactly these four faces' f and their
            // corner-3 vertices -- reduce over the 4 sibling lanes (no gather, no vertex pass)
            P3 acc = p3 + fc;
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
            acc.z += __shfl_xor_sync(0xffffffffu, acc.z, 1);
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 2);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 2);
            acc.z += __shfl_xor_sync(0xffffffffu, acc.z, 2);
            if (valid && (r & 3) == 0) st3(Pn, v[2], 0.5f * p2 + 0.0625f * acc);
        }
    }
    if (!topo) return;
    const int32_t e[4] = {fe.x, fe.y, fe.z, fe.w};
    const int64_t row0 = 4 * (int64_t)(r - lane), nrows = 4 * (int64_t)F;
    {
        int4 rows[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) rows[t] = make_int4(v[t], V + F + e[t], V + r, V + F + e[(t + 3) & 3]);
        warp_store_rows(stage, rows, reinterpret_cast<int4 *>(c.face_vtx), row0, nrows, lane);
    }
    if constexpr (ADJ) {
        if (c.face_edge == nullptr) return;  // the child is the last level: its rows are recomputed there
        const int4 ft = valid ? __ldg(reinterpret_cast<const int4 *>(p.face_twin) + r) : make_int4(-1, -1, -1, -1);
        const int32_t tw[4] = {ft.x, ft.y, ft.z, ft.w};
        int32_t base[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) base[t] = valid ? cc_base<BND>(p.bnd_word, p.bnd_wpre, e[t]) : 0;
        const int32_t h0 = 4 * r;
        int4 rows[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int tn = (t + 1) & 3, tp = (t + 3) & 3;
            const int32_t h = h0 + t, hp = h0 + tp;
            rows[t] = make_int4(base[t] + (v[t] > v[tn]), base[t] + 2 + (tw[t] >= 0 && tw[t] < h),
                                base[tp] + 2 + (tw[tp] >= 0 && tw[tp] < hp), base[tp] + (v[t] > v[tp]));
        }
        warp_store_rows(stage, rows, reinterpret_cast<int4 *>(c.face_edge), row0, nrows, lane);
        if (c.face_twin == nullptr) return;  // the child is the last refined level: no twins needed
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int tn = (t + 1) & 3, tp = (t + 3) & 3;
            const int32_t hp = h0 + tp;
            const int32_t twn = tw[t] >= 0 ? ((tw[t] & ~3) | ((tw[t] + 1) & 3)) : -1;
            rows[t] = make_int4(tw[t] >= 0 ? 4 * twn + 3 : -1, 4 * (h0 + tn) + 2, 4 * hp + 1,
                                tw[tp] >= 0 ? 4 * tw[tp] : -1);
        }
        warp_store_rows(stage, rows, reinterpret_cast<int4 *>(c.face_twin), row0, nrows, lane);
    }
}

// ---------------- face kernel: general matrix (level 0: mixed orders or triangles) ---------
template <int ORDER, bool ADJ, bool BND, int NBC>
__global__ void __launch_bounds__(kThreads) k_cc_face_gen(LevelDev p, ChildDev c, Frames fr, bool topo) {
    ALSUB_GRID_WAIT();
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= p.F) return;
    const Topo<ORDER> tp{p.face_off, p.slot_face};
    const int32_t o = tp.first(r), n = tp.order(r);
    const int32_t V = p.V, F = p.F;
    const float inv = 1.0f / (float)n;
    const int nb = NBC ? NBC : fr.nb;
    if (n == 3 || n == 4) {
        // triangles and quads (almost every face): the face's rows loaded together, then the
        // position gathers together (the general loop below is a serial chain per corner)
        int32_t v[4], e[4], tw[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            v[t] = t < n ? __ldg(p.face_vtx + o + t) : 0;
            e[t] = (topo && t < n) ? __ldg(p.face_edge + o + t) : 0;
            tw[t] = (ADJ && topo && t < n) ? __ldg(p.face_twin + o + t) : -1;
        }
        for (int f = 0; f < nb; ++f) {
            const PR P = fr.rd(f);
            P3 q[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) q[t] = t < n ? ld3(P, v[t]) : p3zero();
            P3 s = p3zero();
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (t < n) s = s + q[t];
            st3(fr.wr(f), V + r, inv * s);
        }
        if (!topo) return;
        int32_t base[4];
        if constexpr (ADJ) {
#pragma unroll
            for (int t = 0; t < 4; ++t) base[t] = t < n ? cc_base<BND>(p.bnd_word, p.bnd_wpre, e[t]) : 0;
        }
        // (neighbours by selects on n, so every register index is a compile-time constant)
        const bool quad = n == 4;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            if (t >= n) break;
            const bool wrap = t + 1 == n;
            const int tn = wrap ? 0 : t + 1, tq = t == 0 ? n - 1 : t - 1;
            const int32_t h = o + t, hn = o + tn, hp = o + tq;
            const int32_t vt = v[t], vn = wrap ? v[0] : v[t < 3 ? t + 1 : 0];
            const int32_t vp = t == 0 ? (quad ? v[3] : v[2]) : v[t > 0 ? t - 1 : 0];
            const int32_t et = e[t], ep = t == 0 ? (quad ? e[3] : e[2]) : e[t > 0 ? t - 1 : 0];
            reinterpret_cast<int4 *>(c.face_vtx)[h] = make_int4(vt, V + F + et, V + r, V + F + ep);
            if constexpr (ADJ) {
                const int32_t twt = tw[t], twp = t == 0 ? (quad ? tw[3] : tw[2]) : tw[t > 0 ? t - 1 : 0];
                const int32_t bt = base[t], bp = t == 0 ? (quad ? base[3] : base[2]) : base[t > 0 ? t - 1 : 0];
                reinterpret_cast<int4 *>(c.face_edge)[h] =
                    make_int4(bt + (vt > vn), bt + 2 + (twt >= 0 && twt < h), bp + 2 + (twp >= 0 && twp < hp),
                              bp + (vt > vp));
                if (c.face_twin)
                    reinterpret_cast<int4 *>(c.face_twin)[h] =
                        make_int4(twt >= 0 ? 4 * tp.next(twt) + 3 : -1, 4 * hn + 2, 4 * hp + 1, twp >= 0 ? 4 * twp : -1);
            }
        }
        return;
    }
    for (int f = 0; f < nb; ++f) {
        const PR P = fr.rd(f);
        P3 s = p3zero();
        for (int32_t t = 0; t < n; ++t) s = s + ld3(P, __ldg(p.face_vtx + o + t));
        st3(fr.wr(f), V + r, inv * s);
    }
    if (!topo) return;
    for (int32_t t = 0; t < n; ++t) {
        const int32_t tn = t + 1 == n ? 0 : t + 1, tq = t == 0 ? n - 1 : t - 1;
        const int32_t h = o + t, hn = o + tn, hp = o + tq;
        const int32_t vt = __ldg(p.face_vtx + h), vn = __ldg(p.face_vtx + hn), vp = __ldg(p.face_vtx + hp);
        const int32_t et = __ldg(p.face_edge + h), ep = __ldg(p.face_edge + hp);
        reinterpret_cast<int4 *>(c.face_vtx)[h] = make_int4(vt, V + F + et, V + r, V + F + ep);
        if constexpr (ADJ) {
            const int32_t twt = __ldg(p.face_twin + h), twp = __ldg(p.face_twin + hp);
            const int32_t bt = cc_base<BND>(p.bnd_word, p.bnd_wpre, et);
            const int32_t bp = cc_base<BND>(p.bnd_word, p.bnd_wpre, ep);
            reinterpret_cast<int4 *>(c.face_edge)[h] =
                make_int4(bt + (vt > vn), bt + 2 + (twt >= 0 && twt < h), bp + 2 + (twp >= 0 && twp < hp),
                          bp + (vt > vp));
            if (c.face_twin)
                reinterpret_cast<int4 *>(c.face_twin)[h] =
                    make_int4(twt >= 0 ? 4 * tp.next(twt) + 3 : -1, 4 * hn + 2, 4 * hp + 1, twp >= 0 ? 4 * twp : -1);
        }
    }
}

// ---------------- edge kernel ----------------
// per parent edge e with pair (h = smallest slot, tw = the other or -1).  IT edges per thread
// with all loads of a stage issued before any is consumed (memory-level parallelism: the kernel
// is a chain edge pair -> face row -> positions).  NBC = compile-time frame count (0 = runtime).
template <int ORDER>
ALSUB_D void edge_ends(const LevelDev &p, const Topo<ORDER> &tp, int32_t h, int32_t &va, int32_t &vb, int32_t &hn) {
    if constexpr (ORDER == 4) {
        const int4 row = __ldg(reinterpret_cast<const int4 *>(p.face_vtx) + (h >> 2));
        const int t = h & 3;
        const int32_t r[4] = {row.x, row.y, row.z, row.w};
        va = r[t];
        vb = r[(t + 1) & 3];
        hn = (h & ~3) | ((h + 1) & 3);
    } else {
        hn = tp.next(h);
        va = __ldg(p.face_vtx + h);
        vb = __ldg(p.face_vtx + hn);
    }
}

template <int ORDER, bool ADJ, bool BND, int NBC, int IT, bool CR>
__global__ void __launch_bounds__(kThreads) k_cc_edge(LevelDev p, ChildDev c, Frames fr, bool topo) {
    ALSUB_GRID_WAIT();
    const Topo<ORDER> tp{p.face_off, p.slot_face};
    const int32_t e0 = blockIdx.x * (kThreads * IT) + threadIdx.x;
    const int32_t V = p.V, F = p.F;
    const int nb = NBC ? NBC : fr.nb;
    int32_t hv[IT], tv[IT], va[IT], vb[IT], hn[IT], jl[IT], bpk[IT], spk[IT];
    float sg[IT];
    const bool bnd = ADJ ? BND : p.B > 0;
#pragma unroll
    for (int k = 0; k < IT; ++k) {
        const int32_t e = e0 + k * kThreads;
        const int2 hh = e < p.E ? __ldg(p.edge_hh + e) : make_int2(0, -1);
        hv[k] = hh.x;
        tv[k] = hh.y;
        // fused crease module: list index of the edge (boundary / creased edges are ~1% of a level)
        jl[k] = (CR && e < p.E) ? sp_index(p.spw, p.spwpre, e) : -1;
        // the topology half's per-word prefixes depend on e alone: loaded here, with the pair, rather
        // than after the position stores (one round trip fewer per edge on the latency-bound levels)
        bpk[k] = (topo && bnd && e < p.E) ? bprefix(p.bnd_word, p.bnd_wpre, e) : 0;
        spk[k] = (CR && ADJ && topo && c.spw && e < p.E) ? sp_prefix(p.spw, p.spwpre, e) : 0;
    }
#pragma unroll
    for (int k = 0; k < IT; ++k) {
        edge_ends<ORDER>(p, tp, hv[k], va[k], vb[k], hn[k]);
        sg[k] = jl[k] >= 0 ? p.sp[jl[k]].sigma : 0.0f;
    }
    for (int f = 0; f < nb; ++f) {
        const PR P = fr.rd(f);
        const PW Pn = fr.wr(f);
        P3 ab[IT], fs[IT];
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            ab[k] = ld3(P, va[k]) + ld3(P, vb[k]);
            fs[k] = tv[k] >= 0 ? ld3c(Pn, V + tp.face(hv[k])) + ld3c(Pn, V + tp.face(tv[k])) : p3zero();
        }
#pragma unroll
        for (int k = 0; k < IT; ++k) {
            const int32_t e = e0 + k * kThreads;
            if (e >= p.E) continue;
            P3 out = tv[k] < 0 ? 0.5f * ab[k] : 0.25f * (ab[k] + fs[k]);
            if (jl[k] >= 0) out = crease_edge_point(sg[k], out, 0.5f * ab[k]);
            st3(Pn, (int64_t)V + F + e, out);
        }
    }
    if (!topo) return;
#pragma unroll
    for (int k = 0; k < IT; ++k) {
        const int32_t e = e0 + k * kThreads;
        if (e >= p.E) continue;
        const int32_t h = hv[k], tw = tv[k];
        // structured child edge ids: block [base, base + 4 - bnd) = (lo,ep), (hi,ep), (fp_min,ep), (fp_max,ep)
        const int32_t bp = bpk[k];
        const int32_t base = 4 * e - bp;
        if (CR && p.inherit && jl[k] >= 0) fused_inherit(p, c, jl[k], p.sp[jl[k]], base, V + F + e);
        if constexpr (ADJ) {
            const bool fwd = va[k] < vb[k];
            const int32_t h_ab = fwd ? h : tw, h_ba = fwd ? tw : h;
            // child half-edges: (lo,ep): lo->ep = 4 h_ab, ep->lo = 4 next(h_ba) + 3; (hi,ep) symmetric
            const int32_t a0 = h_ab >= 0 ? 4 * h_ab : -1, a1 = h_ba >= 0 ? 4 * tp.next(h_ba) + 3 : -1;
            const int32_t b0 = h_ba >= 0 ? 4 * h_ba : -1, b1 = h_ab >= 0 ? 4 * tp.next(h_ab) + 3 : -1;
            auto pair = [](int32_t x, int32_t y) {
                if (x < 0) return make_int2(y, -1);
                if (y < 0) return make_int2(x, -1);
                return make_int2(min(x, y), max(x, y));
            };
            if (c.edge_hh) {
                const int2 q0 = pair(a0, a1), q1 = pair(b0, b1);
                const int2 q2 = pair(4 * h + 1, 4 * hn[k] + 2);  // (fp of face(h), ep); h < tw
                // 16-B stores where the block's start parity allows (the pairs are 8 B each): an
                // even base takes (0,1) and (2,3) as int4, an odd one (1,2) -- half the store
                // instructions, each sector written in two halves instead of four quarters
                int4 *d4 = reinterpret_cast<int4 *>(c.edge_hh);
                if (tw >= 0) {
                    const int2 q3 = pair(4 * tw + 1, 4 * tp.next(tw) + 2);
                    if ((base & 1) == 0) {
                        d4[base >> 1] = make_int4(q0.x, q0.y, q1.x, q1.y);
                        d4[(base >> 1) + 1] = make_int4(q2.x, q2.y, q3.x, q3.y);
                    } else {
                        c.edge_hh[base] = q0;
                        d4[(base + 1) >> 1] = make_int4(q1.x, q1.y, q2.x, q2.y);
                        c.edge_hh[base + 3] = q3;
                    }
                } else if ((base & 1) == 0) {
                    d4[base >> 1] = make_int4(q0.x, q0.y, q1.x, q1.y);
                    c.edge_hh[base + 2] = q2;
                } else {
                    c.edge_hh[base] = q0;
                    d4[(base + 1) >> 1] = make_int4(q1.x, q1.y, q2.x, q2.y);
                }
            }
            const int32_t nch = tw < 0 ? 3 : 4;
            if constexpr (BND) {
                // child boundary bits and, in closed form, the child per-word prefix:
                // bprefix'(base + k) = 2 bprefix(e) + bnd_e min(k, 2)
                if (tw < 0) {
                    atomicOr(c.bnd_word + (base >> 5), 1u << (base & 31));
                    atomicOr(c.bnd_word + ((base + 1) >> 5), 1u << ((base + 1) & 31));
                }
                const int32_t w = (base + 31) >> 5;
                if (32 * w < base + nch) {
                    const int32_t kk = 32 * w - base;
                    c.bnd_wpre[w] = 2 * bp + (tw < 0 ? min(kk, 2) : 0);
                }
            }
            if (CR && c.spw) fused_child_words(c, base, nch, spk[k], jl[k] >= 0);
        }
    }
}

// ---------------- last-level edge kernel over the grandparent edges ----------------
// At the last refined level l (>= 2) the level-l edges are iterated as the 3-4 children of each
// level-(l-1) edge e' = (h', tw'): (lo,ep), (hi,ep), (fp_R,ep), (fp_S,ep) with ids base(e')+k and
// faces {h_ab, next(h_ba)}, {h_ba, next(h_ab)}, {h', next(h')}, {tw', next(tw')} (level-l face
// index = level-(l-1) slot).  Five position gathers and four face points serve all four edge
// points, and the level-l edge pairs never need to be stored.  The same values are exactly the
// 1-ring of the level-l vertex ep (an edge point born at level l, valence 4: neighbours lo, hi,
// fp_R, fp_S; faces h, next(h), tw, next(tw)), so its vertex point
//   S(ep) = 1/2 p_ep + 1/16 (p_lo + p_hi + p_R + p_S + f_h + f_next(h) + f_tw + f_next(tw))
// (Eq. pos_update with n = 4) is stored here too, at id ep (coalesced: consecutive e).
// Boundary edge points keep p; the crease pass overwrites every special vertex afterwards.
// epo >= 0: first id of the edge points born at level l-1 (ids [epo, V_{l-1})).  Such a vertex x =
// ep(e'') of a level-(l-2) edge e'' is the max endpoint of exactly the level-(l-1) edges
// base(e'') .. base(e'') + 3 (interior e''), consecutive threads here, and each of those threads
// holds one ring term: x's next vertex in one incident level-l face is the thread's edge point,
// and the thread's two faces at x are two of x's four (each counted by two threads).  So
//   S(x) = 1/2 p_x + 1/16 sum_k (p_ep_k + 1/2 (f_a_k + f_b_k))
// is a block-shared sum over the group when all four threads are in one block (the vertex kernel
// does the few groups that straddle a block boundary, and boundary e'').
template <int NBC>
__global__ void __launch_bounds__(kThreads, NBC ? 5 : 0) k_cc_edge_gp(LevelDev p, LevelDev gp, ChildDev c, Frames fr,
                                                       int32_t epo, const int2 *ehh2) {
    ALSUB_GRID_WAIT();
    // the block's children are the contiguous id range [base(e_first), base(e_last) + nch): staged
    // in shared memory and written back as one coalesced float run.  Staging is one array per
    // coordinate, child a at a + a/32 (thread t's children start near 4 t, so without the skew a
    // warp's stores of one child k land on 8 banks); rows kSo floats apart (kSo = 11 mod 32) so the
    // read-back's x/y/z of neighbouring children fall on different banks
    constexpr int kSo = 4 * kThreads + 4 * kThreads / 32 + 11;
    __shared__ float s_out[3 * kSo];
    __shared__ int32_t s_base0, s_end;
    const int32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = e < gp.E;
    int2 hh = make_int2(0, -1);
    if (valid) hh = __ldg(gp.edge_hh + e);
    const int32_t h = hh.x, tw = hh.y;
    const int32_t R = h >> 2, t = h & 3;
    const int4 row = valid ? __ldg(reinterpret_cast<const int4 *>(gp.face_vtx) + R) : make_int4(0, 0, 0, 0);
    // (selects, not a dynamically indexed array: that would live in local memory)
    const int32_t va = t == 0 ? row.x : t == 1 ? row.y : t == 2 ? row.z : row.w;
    const int32_t vb = t == 0 ? row.y : t == 1 ? row.z : t == 2 ? row.w : row.x;
    const int32_t Vg = gp.V, Fg = gp.F;
    const int32_t ep = Vg + Fg + e, fpR = Vg + R, fpS = tw >= 0 ? Vg + (tw >> 2) : 0;
    const int32_t nh = (h & ~3) | ((h + 1) & 3), nt = tw >= 0 ? ((tw & ~3) | ((tw + 1) & 3)) : 0;
    const int32_t bp = (valid && gp.B > 0) ? bprefix(gp.bnd_word, gp.bnd_wpre, e) : 0;
    const int32_t base = valid ? 4 * e - bp : 0;
    const int32_t nch = tw < 0 ? 3 : 4;
    const int32_t last = min((int32_t)(blockIdx.x * blockDim.x + blockDim.x), gp.E) - 1;
    if (threadIdx.x == 0) s_base0 = base;
    if (valid && e == last) s_end = base + nch;
    const bool fwd = va < vb;  // h runs lo -> hi
    const int32_t lo = fwd ? va : vb, hi = fwd ? vb : va;
    const int32_t f0a = fwd ? h : tw, f0b = fwd ? nt : nh;  // faces of (lo, ep)
    const int32_t f1a = fwd ? tw : h, f1b = fwd ? nh : nt;  // faces of (hi, ep)
    const int32_t V = p.V, F = p.F;
    const int nb = NBC ? NBC : fr.nb;
    // ring-sum group of hi (an edge point born at level l-1): position k in its group
    // (bprefix(e) = 2 bprefix''(e'') inside an interior group, so k = e - base(e''))
    __shared__ float s_ring[3][kThreads + 1];
    __shared__ int32_t s_hi[kThreads];
    const bool inx = valid && epo >= 0 && hi >= epo && hi < Vg && tw >= 0;
    s_hi[threadIdx.x] = inx ? hi : -1;
    // a group across two blocks (fr.gside, last level): its members leave their terms in gside slot
    // e0 / kThreads; the second of the two blocks to finish sums them (last-arriver counter gcnt)
    __shared__ int32_t s_sx[2];  // the straddling group's vertex: [0] from the previous block, [1] into the next
    if (threadIdx.x < 2) s_sx[threadIdx.x] = -1;
    __syncthreads();
    int32_t gslot = -1, gk = 0;
    if (inx && fr.gside) {
        const int32_t k = e - 4 * (hi - epo) + (bp >> 1), e0 = e - k;
        // (boundary edges of level l-2 have no such group: their edge point's ring is the vertex kernel's)
        if ((e0 & (kThreads - 1)) > kThreads - 4 && __ldg(ehh2 + (hi - epo)).y >= 0) {
            gslot = e0 / kThreads;
            gk = k;
            s_sx[gslot - (int32_t)blockIdx.x + 1] = hi;
        }
    }
    bool lead = false;
    if (inx && e - 4 * (hi - epo) + (bp >> 1) == 0 && threadIdx.x + 3 < blockDim.x)
        lead = s_hi[threadIdx.x + 1] == hi && s_hi[threadIdx.x + 2] == hi && s_hi[threadIdx.x + 3] == hi;
    const int32_t base0 = s_base0, n = s_end - base0;
    const int32_t o = base - base0;
    for (int f = 0; f < nb; ++f) {
        const PR P = fr.rd(f);
        const PW Pn = fr.wr(f);
        P3 phx = p3zero();
        if (valid) {
            const P3 plo = ld3(P, lo), phi = ld3(P, hi), pep = ld3(P, ep), pR = ld3(P, fpR);
            phx = phi;
            const P3 fh = ld3c(Pn, V + h), fnh = ld3c(Pn, V + nh);
            P3 q[4];
            q[2] = 0.25f * (pR + pep + fh + fnh);
            if (tw < 0) {
                q[0] = 0.5f * (plo + pep);
                q[1] = 0.5f * (phi + pep);
                st3(Pn, ep, pep);
            } else {
                const P3 pS = ld3(P, fpS), ft = ld3c(Pn, V + tw), fnt = ld3c(Pn, V + nt);
                const P3 fa = (f0a == h ? fh : ft) + (f0b == nh ? fnh : fnt);
                const P3 fb = (f1a == h ? fh : ft) + (f1b == nh ? fnh : fnt);
                q[0] = 0.25f * (plo + pep + fa);
                q[1] = 0.25f * (phi + pep + fb);
                q[3] = 0.25f * (pS + pep + ft + fnt);
                st3(Pn, ep, 0.5f * pep + 0.0625f * ((plo + phi) + (pR + pS) + (fh + fnh) + (ft + fnt)));
                if (inx) {
                    const P3 fx = fwd ? (fnh + ft) : (fh + fnt);  // this edge's two faces at hi
                    const P3 rt = pep + 0.5f * fx;
                    s_ring[0][threadIdx.x] = rt.x;
                    s_ring[1][threadIdx.x] = rt.y;
                    s_ring[2][threadIdx.x] = rt.z;
                    if (gslot >= 0) {  // a group across two blocks: its term, published before the block's barrier
                        float *gs = fr.gside + f * fr.gsidestride + 12 * (int64_t)gslot + 3 * gk;
                        gs[0] = rt.x;
                        gs[1] = rt.y;
                        gs[2] = rt.z;
                        __threadfence();
                    }
                }
            }

#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (k >= nch) break;
                const int a = o + k, sa = a + (a >> 5);
                s_out[sa] = q[k].x;
                s_out[kSo + sa] = q[k].y;
                s_out[2 * kSo + sa] = q[k].z;
            }
        }
        __syncthreads();
        if (lead) {
            const int t0 = threadIdx.x;
            const P3 acc{(s_ring[0][t0] + s_ring[0][t0 + 1]) + (s_ring[0][t0 + 2] + s_ring[0][t0 + 3]),
                         (s_ring[1][t0] + s_ring[1][t0 + 1]) + (s_ring[1][t0 + 2] + s_ring[1][t0 + 3]),
                         (s_ring[2][t0] + s_ring[2][t0 + 1]) + (s_ring[2][t0 + 2] + s_ring[2][t0 + 3])};
            st3(Pn, hi, 0.5f * phx + 0.0625f * acc);
        }
        if (Pn.vs == 3) {
            float *dst = Pn.p + 3 * ((int64_t)V + F + base0);
            for (int32_t i = threadIdx.x; i < 3 * n; i += blockDim.x) {
                const int32_t a = i / 3, cc = i - 3 * a;
                dst[i] = s_out[cc * kSo + a + (a >> 5)];
            }
        } else {
            for (int32_t a = threadIdx.x; a < n; a += blockDim.x) {
                const int32_t sa = a + (a >> 5);
                st3(Pn, (int64_t)V + F + base0 + a, P3{s_out[sa], s_out[kSo + sa], s_out[2 * kSo + sa]});
            }
        }
        __syncthreads();
    }
    // a level before the last (c.bnd_word set): the boundary words of level l+1.  Child k of e is
    // the level-l edge x = base + k, boundary iff e is and k < 2, with the level-l prefix
    // bprefix(x) = 2 bprefix(e) + bnd_e min(k, 2); x's own children start at 4x - bprefix(x)
    // (the same closed forms k_cc_edge writes one level at a time)
    if (c.bnd_word != nullptr && valid) {
        const int32_t bpe = 4 * e - base;
        for (int k = 0; k < nch; ++k) {
            const int32_t x = base + k;
            const bool bx = tw < 0 && k < 2;
            const int32_t bpx = 2 * bpe + (tw < 0 ? min(k, 2) : 0);
            const int32_t b2 = 4 * x - bpx;
            if (bx) {
                atomicOr(c.bnd_word + (b2 >> 5), 1u << (b2 & 31));
                atomicOr(c.bnd_word + ((b2 + 1) >> 5), 1u << ((b2 + 1) & 31));
            }
            const int32_t w = (b2 + 31) >> 5;
            if (32 * w < b2 + (bx ? 3 : 4)) c.bnd_wpre[w] = 2 * bpx + (bx ? min(32 * w - b2, 2) : 0);
        }
    }
    // straddling groups: S(x) = 1/2 p_x + 1/16 sum_k (p_ep_k + 1/2 (f_a,k + f_b,k)), by the block
    // that arrives second (both blocks' terms are in gside by then; the counter is reset for the
    // next launch)
    if (fr.gside && threadIdx.x < 2) {
        const int32_t x = s_sx[threadIdx.x];
        if (x >= 0) {
            const int32_t slot = (int32_t)blockIdx.x - 1 + threadIdx.x;
            __threadfence();
            if (atomicAdd(fr.gcnt + slot, 1) == 1) {
                __threadfence();
                fr.gcnt[slot] = 0;
                for (int f = 0; f < nb; ++f) {
                    const float *gs = fr.gside + f * fr.gsidestride + 12 * (int64_t)slot;
                    float t[12];
#pragma unroll
                    for (int i = 0; i < 12; ++i) t[i] = __ldcg(gs + i);
                    const P3 acc{(t[0] + t[3]) + (t[6] + t[9]), (t[1] + t[4]) + (t[7] + t[10]),
                                 (t[2] + t[5]) + (t[8] + t[11])};
                    st3(fr.wr(f), x, 0.5f * ld3(fr.rd(f), x) + 0.0625f * acc);
                }
            }
        }
    }
}

// ---------------- vertex kernel: class-structured incident slots ----------------
// S(p) = (1 - 2/n) p + 1/n^2 sum_{incident slots x} (p_{v(next(x))} + f_{face(x)})
// (Eq. pos_update split: s2 = F P and s3 = M f as gathers over M's row of p).
// The row of M of a level-l vertex is closed-form from the level it was born at (VSegs):
//   level-0 vertex v : 4^l x its level-0 slots (M^T from the counting sort)
//   face point of face r of level m-1 : 4^(l-m) x {4 (off_r + t) + 2}
//   edge point of edge (h, tw) of level m-1 : 4^(l-m) x {4h+1, 4 next(h)+3, 4tw+1, 4 next(tw)+3}
// so no twin walk (no dependent chain) is needed; all loads of a vertex are issued together.
template <int ORDER>
struct VtxCtx {
    const int32_t *face_vtx;
    Topo<ORDER> tl;
    int32_t V;
};

// store the vertex point of v: the smooth value, overridden by the boundary/crease rule when v is
// a special vertex (fused crease module)
ALSUB_D void emit_vertex(const Frames &fr, int f, int32_t v, const VCr &cr, P3 smooth) {
    st3(fr.wr(f), v, cr.k >= 2 ? crease_vertex_point(cr, fr.rd(f), v, smooth) : smooth);
}

// accumulate the smooth point of v over N slots for every frame
template <int ORDER, int N>
ALSUB_D void smooth_fixed(const VtxCtx<ORDER> &x, const Frames &fr, int32_t v, const int32_t (&sl)[N], const VCr &cr) {
    int32_t nb[N], fc[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        nb[k] = __ldg(x.face_vtx + x.tl.next(sl[k]));
        fc[k] = x.V + x.tl.face(sl[k]);
    }
    constexpr float inv = 1.0f / (float)N;
    for (int f = 0; f < fr.nb; ++f) {
        const PR P = fr.rd(f);
        const PW Pn = fr.wr(f);
        P3 acc = ld3(P, nb[0]) + ld3c(Pn, fc[0]);
#pragma unroll
        for (int k = 1; k < N; ++k) acc = acc + ld3(P, nb[k]) + ld3c(Pn, fc[k]);
        emit_vertex(fr, f, v, cr, (1.0f - 2.0f * inv) * ld3(P, v) + (inv * inv) * acc);
    }
}

template <int ORDER>
ALSUB_D void smooth_list(const VtxCtx<ORDER> &x, const Frames &fr, int32_t v, const int32_t *list, int32_t n,
                         int shift, bool quad_fp, int32_t off, const VCr &cr) {
    for (int f = 0; f < fr.nb; ++f) {
        const PR P = fr.rd(f);
        const PW Pn = fr.wr(f);
        P3 acc = p3zero();
        for (int32_t k = 0; k < n; ++k) {
            const int32_t s = quad_fp ? ((4 * (off + k) + 2) << shift) : (__ldg(list + k) << shift);
            acc = acc + ld3(P, __ldg(x.face_vtx + x.tl.next(s))) + ld3c(Pn, x.V + x.tl.face(s));
        }
        const P3 pv = ld3(P, v);
        if (n == 0) { st3(Pn, v, pv); continue; }
        const float inv = 1.0f / (float)n;
        emit_vertex(fr, f, v, cr, (1.0f - 2.0f * inv) * pv + (inv * inv) * acc);
    }
}

ALSUB_D void copy_point(const Frames &fr, int32_t v, const VCr &cr) {
    for (int f = 0; f < fr.nb; ++f) emit_vertex(fr, f, v, cr, ld3(fr.rd(f), v));
}

// vertex born before this level: every incident level-l face q has it at corner 0, and the face
// kernel left c0[q] = p(corner 1) + f_q, so S = (1 - 2/n) p + 1/n^2 sum_q c0[q]
template <int N>
ALSUB_D void smooth_c0(const Frames &fr, int32_t v, const int32_t (&q)[N], const VCr &cr) {
    constexpr float inv = 1.0f / (float)N;
    const int cs = fr.c0shift;
    for (int f = 0; f < fr.nb; ++f) {
        const PR c0 = fr.c0r(f);
        P3 acc = ld3c(c0, q[0] >> cs);
#pragma unroll
        for (int k = 1; k < N; ++k) acc = acc + ld3c(c0, q[k] >> cs);
        emit_vertex(fr, f, v, cr, (1.0f - 2.0f * inv) * ld3(fr.rd(f), v) + (inv * inv) * acc);
    }
}

// special-vertex index of vertex j of segment s (-1 if it cannot be special): level-0 vertices are
// the identity table; an edge point born at m is special iff its level-(m-1) edge is listed
ALSUB_D int32_t sv_index(const VSegs &g, int s, int32_t j) {
    const int type = g.type[s];
    if (type == 0) return j;
    if (type == 1) return -1;
    const int m1 = g.birth[s] - 1;
    const int32_t idx = sp_index(g.spw[m1], g.spwpre[m1], j);
    return idx >= 0 ? g.nsvb[m1] + idx : -1;
}

template <int ORDER>
ALSUB_D void cc_vertex_smooth(const VtxCtx<ORDER> &x, const Frames &fr, const VSegs &g, int s, int32_t j, const VCr &cr);

// special (boundary / crease) vertex: the rule of crease_vertex_point, the smooth point only when
// it is blended in
template <int ORDER>
ALSUB_D void cc_vertex_special(const VtxCtx<ORDER> &x, const Frames &fr, const VSegs &g,
                                               const LevelDev &p, int32_t *csv_list, int s, int32_t j, int32_t i) {
    const int32_t v = g.start[s] + j;
    const VCr cr = vertex_crease(p, p.inherit ? csv_list : nullptr, i, v);
    if (cr.k >= 2 && cr.s >= 1.0f) {  // sharp: no smooth point needed
        for (int f = 0; f < fr.nb; ++f) st3(fr.wr(f), v, crease_vertex_point(cr, fr.rd(f), v, p3zero()));
        return;
    }
    if (s == g.hs_seg) {
        const int2 hh = __ldg(g.ehh[g.birth[s] - 1] + j);
        for (int f = 0; f < fr.nb; ++f) {
            const PR hs = fr.hsr(f);
            const P3 acc = ld3c(hs, hh.x) + ld3c(hs, hh.y);
            emit_vertex(fr, f, v, cr, 0.5f * ld3(fr.rd(f), v) + 0.0625f * acc);
        }
        return;
    }
    cc_vertex_smooth<ORDER>(x, fr, g, s, j, cr);
}

template <int ORDER, bool CR>
ALSUB_D void cc_vertex_one(const VtxCtx<ORDER> &x, const Frames &fr, const VSegs &g, const LevelDev &p,
                           int32_t *csv_list, int s, int32_t j) {
    if constexpr (CR) {
        const int32_t i = sv_index(g, s, j);
        if (i >= 0 && p.sv_off[i + 1] > p.sv_off[i]) {
            cc_vertex_special<ORDER>(x, fr, g, p, csv_list, s, j, i);
            return;
        }
    }
    cc_vertex_smooth<ORDER>(x, fr, g, s, j, VCr{0, 0.0f, -1, -1});
}

template <int ORDER>
ALSUB_D void cc_vertex_smooth(const VtxCtx<ORDER> &x, const Frames &fr, const VSegs &g, int s, int32_t j, const VCr &cr) {
    const int32_t v = g.start[s] + j;
    const int shift = 2 * (g.level - g.birth[s]);
    const int type = g.type[s];
    const int m1 = g.birth[s] - 1;
    if (fr.c0 && shift >= 2) {
        // faces = slots >> 2 = birth slots << (shift - 2)
        const int fs = shift - 2;
        if (type == 2) {
            const int2 hh = __ldg(g.ehh[m1] + j);
            if (hh.y < 0) { copy_point(fr, v, cr); return; }
            int32_t nh, nt;
            if (m1 == 0) {
                const Topo<0> t0{g.face_off0, g.slot_face0};
                nh = t0.next(hh.x);
                nt = t0.next(hh.y);
            } else {
                nh = (hh.x & ~3) | ((hh.x + 1) & 3);
                nt = (hh.y & ~3) | ((hh.y + 1) & 3);
            }
            const int32_t q[4] = {(4 * hh.x + 1) << fs, (4 * nh + 3) << fs, (4 * hh.y + 1) << fs, (4 * nt + 3) << fs};
            smooth_c0<4>(fr, v, q, cr);
        } else if (type == 1 && m1 > 0) {
            const int32_t q[4] = {(16 * j + 2) << fs, (16 * j + 6) << fs, (16 * j + 10) << fs, (16 * j + 14) << fs};
            smooth_c0<4>(fr, v, q, cr);
        } else {
            // level-0 vertex (its level-0 row) or face point of a level-0 face of any order
            int32_t o, cnt;
            const bool lv0 = type == 0;
            if (lv0) {
                if (__ldg(g.vbnd0 + j)) { copy_point(fr, v, cr); return; }
                o = __ldg(g.vtx_off0 + j);
                cnt = __ldg(g.vtx_off0 + j + 1) - o;
            } else {
                o = __ldg(g.face_off0 + j);
                cnt = __ldg(g.face_off0 + j + 1) - o;
            }
            for (int f = 0; f < fr.nb; ++f) {
                const PR c0 = fr.c0r(f);
                P3 acc = p3zero();
                for (int32_t k = 0; k < cnt; ++k) {
                    const int32_t b = lv0 ? __ldg(g.vtx_list0 + o + k) : 4 * (o + k) + 2;
                    acc = acc + ld3c(c0, (b << fs) >> fr.c0shift);
                }
                const P3 pv = ld3(fr.rd(f), v);
                if (cnt == 0) { st3(fr.wr(f), v, pv); continue; }
                const float inv = 1.0f / (float)cnt;
                emit_vertex(fr, f, v, cr, (1.0f - 2.0f * inv) * pv + (inv * inv) * acc);
            }
        }
        return;
    }
    if (type == 2) {  // edge point born at level m1 + 1
        const int2 hh = __ldg(g.ehh[m1] + j);
        if (hh.y < 0) { copy_point(fr, v, cr); return; }  // boundary (special, handled above)
        int32_t nh, nt;
        if (m1 == 0) {
            const Topo<0> t0{g.face_off0, g.slot_face0};
            nh = t0.next(hh.x);
            nt = t0.next(hh.y);
        } else {
            nh = (hh.x & ~3) | ((hh.x + 1) & 3);
            nt = (hh.y & ~3) | ((hh.y + 1) & 3);
        }
        const int32_t sl[4] = {(4 * hh.x + 1) << shift, (4 * nh + 3) << shift, (4 * hh.y + 1) << shift,
                               (4 * nt + 3) << shift};
        smooth_fixed<ORDER, 4>(x, fr, v, sl, cr);
    } else if (type == 1 && m1 > 0) {  // face point of a quad
        const int32_t sl[4] = {(16 * j + 2) << shift, (16 * j + 6) << shift, (16 * j + 10) << shift,
                               (16 * j + 14) << shift};
        smooth_fixed<ORDER, 4>(x, fr, v, sl, cr);
    } else if (type == 1) {  // face point of a level-0 face (any order)
        const int32_t off = __ldg(g.face_off0 + j), cnt = __ldg(g.face_off0 + j + 1) - off;
        smooth_list<ORDER>(x, fr, v, nullptr, cnt, shift, true, off, cr);
    } else {  // level-0 vertex
        if (__ldg(g.vbnd0 + j)) { copy_point(fr, v, cr); return; }
        const int32_t o = __ldg(g.vtx_off0 + j), cnt = __ldg(g.vtx_off0 + j + 1) - o;
        smooth_list<ORDER>(x, fr, v, g.vtx_list0 + o, cnt, shift, false, 0, cr);
    }
}

// ---- the fused-crease (small) levels: one smooth evaluation, then the crease rule ----
// At these sizes the kernel is a chain of dependent loads (and its code size matters: ncu showed
// a quarter of the level-1 stalls on instruction fetch while cc_vertex_special and its own copy of
// cc_vertex_smooth were inlined at every call site).  Here the smooth value is computed once per
// frame by smooth_value (cc_vertex_smooth's arithmetic and summation order, returning the value),
// its loads in flight together with the special test's, ring slots and their corner sums four at
// a time; special vertices then apply crease_vertex_point to it (sharp ones ignore it).
constexpr int kRingBatch = 4;

// ring of a level-0 vertex (list = its M^T row) or of the face point of a level-0 face (list =
// nullptr, slots 4 (off + k) + 2): c0 corner sums at levels >= 1, slot gathers at level 0
template <int ORDER>
ALSUB_D P3 ring_sum(const VtxCtx<ORDER> &x, const Frames &fr, int f, const int32_t *list, int32_t off, int32_t cnt,
                    int shift) {
    const PR P = fr.rd(f);
    const PW Pn = fr.wr(f);
    const bool c0p = fr.c0 && shift >= 2;
    P3 acc = p3zero();
    for (int32_t k0 = 0; k0 < cnt; k0 += kRingBatch) {
        int32_t b[kRingBatch];
#pragma unroll
        for (int u = 0; u < kRingBatch; ++u)
            b[u] = k0 + u >= cnt ? -1 : list ? __ldg(list + off + k0 + u) : 4 * (off + k0 + u) + 2;
        if (c0p) {
            const PR c0 = fr.c0r(f);
#pragma unroll
            for (int u = 0; u < kRingBatch; ++u)
                if (b[u] >= 0) acc = acc + ld3c(c0, (b[u] << (shift - 2)) >> fr.c0shift);
        } else {
            int32_t nbv[kRingBatch], fc[kRingBatch];
#pragma unroll
            for (int u = 0; u < kRingBatch; ++u) {
                nbv[u] = fc[u] = 0;
                if (b[u] >= 0) {
                    const int32_t sl = b[u] << shift;
                    fc[u] = x.V + x.tl.face(sl);
                    nbv[u] = __ldg(x.face_vtx + x.tl.next(sl));
                }
            }
#pragma unroll
            for (int u = 0; u < kRingBatch; ++u)
                if (b[u] >= 0) acc = acc + ld3(P, nbv[u]) + ld3c(Pn, fc[u]);
        }
    }
    return acc;
}

template <int ORDER>
ALSUB_D P3 smooth_value(const VtxCtx<ORDER> &x, const Frames &fr, const VSegs &g, int s, int32_t j, int f) {
    const int32_t v = g.start[s] + j;
    const int type = g.type[s];
    const int m1 = g.birth[s] - 1;
    const int shift = 2 * (g.level - g.birth[s]);
    const PR P = fr.rd(f);
    const PW Pn = fr.wr(f);
    const P3 pv = ld3(P, v);
    if (type == 2) {
        const int2 hh = __ldg(g.ehh[m1] + j);
        if (hh.y < 0) return pv;
        if (s == g.hs_seg) {  // edge point born at this level: the face kernel's two half sums
            const PR hs = fr.hsr(f);
            return 0.5f * pv + 0.0625f * (ld3c(hs, hh.x) + ld3c(hs, hh.y));
        }
        int32_t nh, nt;
        if (m1 == 0) {
            const Topo<0> t0{g.face_off0, g.slot_face0};
            nh = t0.next(hh.x);
            nt = t0.next(hh.y);
        } else {
            nh = (hh.x & ~3) | ((hh.x + 1) & 3);
            nt = (hh.y & ~3) | ((hh.y + 1) & 3);
        }
        const int32_t q[4] = {4 * hh.x + 1, 4 * nh + 3, 4 * hh.y + 1, 4 * nt + 3};
        P3 acc;
        if (fr.c0 && shift >= 2) {
            const PR c0 = fr.c0r(f);
            acc = ld3c(c0, (q[0] << (shift - 2)) >> fr.c0shift);
#pragma unroll
            for (int k = 1; k < 4; ++k) acc = acc + ld3c(c0, (q[k] << (shift - 2)) >> fr.c0shift);
        } else {
            int32_t nbv[4], fc[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                nbv[k] = __ldg(x.face_vtx + x.tl.next(q[k] << shift));
                fc[k] = x.V + x.tl.face(q[k] << shift);
            }
            acc = ld3(P, nbv[0]) + ld3c(Pn, fc[0]);
#pragma unroll
            for (int k = 1; k < 4; ++k) acc = acc + ld3(P, nbv[k]) + ld3c(Pn, fc[k]);
        }
        return 0.5f * pv + 0.0625f * acc;
    }
    int32_t off, cnt;
    const int32_t *list = nullptr;
    if (type == 1 && m1 > 0) {  // face point of a quad: slots 16 j + 2 + 4 t
        off = 4 * j;
        cnt = 4;
    } else if (type == 1) {  // face point of a level-0 face
        off = __ldg(g.face_off0 + j);
        cnt = __ldg(g.face_off0 + j + 1) - off;
    } else {  // level-0 vertex: its M^T row
        const int32_t o = __ldg(g.vtx_off0 + j), o1 = __ldg(g.vtx_off0 + j + 1);
        if (__ldg(g.vbnd0 + j)) return pv;
        off = o;
        cnt = o1 - o;
        list = g.vtx_list0;
    }
    if (cnt == 0) return pv;
    const P3 acc = ring_sum<ORDER>(x, fr, f, list, off, cnt, shift);
    const float inv = 1.0f / (float)cnt;
    return (1.0f - 2.0f * inv) * pv + (inv * inv) * acc;
}

template <int ORDER>
ALSUB_D void cc_vertex_cr(const VtxCtx<ORDER> &x, const Frames &fr, const VSegs &g, const LevelDev &p,
                          int32_t *csv_list, int s, int32_t j) {
    const int32_t v = g.start[s] + j;
    const int32_t i = sv_index(g, s, j);
    VCr cr{0, 0.0f, -1, -1};
    for (int f = 0; f < fr.nb; ++f) {
        const P3 sm = smooth_value<ORDER>(x, fr, g, s, j, f);
        if (f == 0 && i >= 0 && p.sv_off[i + 1] > p.sv_off[i]) cr = vertex_crease(p, p.inherit ? csv_list : nullptr, i, v);
        st3(fr.wr(f), v, cr.k >= 2 ? crease_vertex_point(cr, fr.rd(f), v, sm) : sm);
    }
}

// a long level-0 ring (n > kLongRing, not boundary, not special), summed by the whole warp; the
// same two forms as cc_vertex_smooth: c0 corner sums (levels >= 1) or slot gathers (level 0)
// level-0 vertex j is summed by k_cc_vertex_long: a long M^T row (the build's list, n > 16), not on
// a boundary, not special (those keep the per-lane path)
ALSUB_D bool cc_long_ring(const VSegs &g, const LevelDev &p, int32_t j, bool cr) {
    const int32_t n = __ldg(g.vtx_off0 + j + 1) - __ldg(g.vtx_off0 + j);
    if (n <= kLongRow || __ldg(g.vbnd0 + j)) return false;
    return !(cr && p.sv_off[j + 1] > p.sv_off[j]);
}

// The long rings, a warp per listed vertex (only launched when the mesh has long rows): kept out
// of k_cc_vertex, whose registers an inlined (or called) 8-wide gather loop raised from 40 to 64
// (config 3 0.685 -> 0.704 ms).  Same two forms as cc_vertex_smooth: c0 corner sums (levels >= 1)
// or slot gathers (level 0); lanes take slots k = lane, lane + 32, ..., warp_sum reduces.
template <int ORDER, bool CR>
__global__ void __launch_bounds__(kThreads) k_cc_vertex_long(LevelDev p, Frames fr, VSegs g) {
    ALSUB_GRID_WAIT();
    const int32_t w = (int32_t)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (w >= g.nlong) return;
    const int32_t j = __ldg(g.long_list + w);
    if (!cc_long_ring(g, p, j, CR)) return;
    const Topo<ORDER> tl{p.face_off, p.slot_face};
    const int shift = 2 * g.level;
    const int32_t o = __ldg(g.vtx_off0 + j), cnt = __ldg(g.vtx_off0 + j + 1) - o;
    const bool c0p = fr.c0 && shift >= 2;
    const float inv = 1.0f / (float)cnt;
    for (int f = 0; f < fr.nb; ++f) {
        P3 acc = p3zero();
        // 8 slots per lane in flight: the chain list -> (face_vtx ->) position is latency bound
        for (int32_t k0 = lane; k0 < cnt; k0 += 32 * 8) {
            int32_t b[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) b[u] = k0 + 32 * u < cnt ? __ldg(g.vtx_list0 + o + k0 + 32 * u) : -1;
            if (c0p) {
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (b[u] >= 0) acc = acc + ld3c(fr.c0r(f), (b[u] << (shift - 2)) >> fr.c0shift);
            } else {
                int32_t nbr[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) nbr[u] = b[u] >= 0 ? __ldg(p.face_vtx + tl.next(b[u] << shift)) : -1;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (b[u] >= 0) acc = acc + ld3(fr.rd(f), nbr[u]) + ld3c(fr.wr(f), p.V + tl.face(b[u] << shift));
            }
        }
        acc = warp_sum(acc);
        if (lane == 0) st3(fr.wr(f), j, (1.0f - 2.0f * inv) * ld3(fr.rd(f), j) + (inv * inv) * acc);
    }
}

template <int ORDER, int PL, bool CR>
__global__ void __launch_bounds__(kThreads, ORDER == 4 && !CR ? 8 : 0) k_cc_vertex(LevelDev p, Frames fr, VSegs g, int32_t *csv_list) {
    ALSUB_GRID_WAIT();
    constexpr int kVtxTask = 32 * PL;  // vertices per warp task (PL per lane)
    // Work unit = a warp task of 32 PL consecutive vertices of ONE segment (no divergence between
    // vertex classes inside a warp); block b takes the same fraction [b/NB, (b+1)/NB) of every
    // segment's tasks, so a block works on one spatial band of the mesh.
    __shared__ int32_t s_lo[kMaxSeg], s_pre[kMaxSeg + 1];
    const int64_t nblk = gridDim.x, b = blockIdx.x;
    // warp 0: this block's task range of every segment (nseg = 1 + 2 l <= 31 for l < 16 levels)
    // and their exclusive prefix by a shuffle scan -- one barrier; most blocks of a large level
    // have only a few tasks, so the prologue is a visible share of the kernel
    if (threadIdx.x < 32) {
        int32_t lo = 0, cnt = 0;
        if ((int)threadIdx.x < g.nseg) {
            const int64_t tasks = (g.len[threadIdx.x] + kVtxTask - 1) / kVtxTask;
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
    const VtxCtx<ORDER> x{p.face_vtx, Topo<ORDER>{p.face_off, p.slot_face}, p.V};
    const int32_t ntask = s_pre[g.nseg];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    int s = 0;
    for (int32_t task = warp; task < ntask; task += nwarp) {
        while (s_pre[s + 1] <= task) ++s;  // tasks ascend: the segment index only moves forward
        const int32_t j0 = (s_lo[s] + (task - s_pre[s])) * kVtxTask + lane;
        const int32_t len = g.len[s];
        if (CR) {
            for (int k = 0; k < PL; ++k) {
                const int32_t j = j0 + 32 * k;
                if (j >= len) continue;
                if (s != g.hs_seg && g.nlong > 0 && g.type[s] == 0 && cc_long_ring(g, p, j, CR)) continue;  // k_cc_vertex_long
                cc_vertex_cr<ORDER>(x, fr, g, p, csv_list, s, j);
            }
            continue;
        }
        if (s == g.hs_seg) {
            // edge points born at this level: two half sums from the face kernel
            const int m1 = g.birth[s] - 1;
            for (int k = 0; k < PL; ++k) {
                const int32_t j = j0 + 32 * k;
                if (j >= len) continue;
                const int32_t v = g.start[s] + j;
                const int2 hh = __ldg(g.ehh[m1] + j);  // (issued beside the special test's loads)
                if constexpr (CR) {
                    const int32_t i = sv_index(g, s, j);
                    if (i >= 0) {  // boundary / creased parent edge
                        cc_vertex_special<ORDER>(x, fr, g, p, csv_list, s, j, i);
                        continue;
                    }
                }
                for (int f = 0; f < fr.nb; ++f) {
                    // boundary edge points keep p (set by the separate crease/boundary pass)
                    if (hh.y < 0) { st3(fr.wr(f), v, ld3(fr.rd(f), v)); continue; }
                    const PR hs = fr.hsr(f);
                    const P3 acc = ld3c(hs, hh.x) + ld3c(hs, hh.y);
                    st3(fr.wr(f), v, 0.5f * ld3(fr.rd(f), v) + 0.0625f * acc);
                }
            }
            continue;
        }
        for (int k = 0; k < PL; ++k) {
            const int32_t j = j0 + 32 * k;
            if (j >= len) continue;
            if (g.nlong > 0 && g.type[s] == 0 && cc_long_ring(g, p, j, CR)) continue;  // k_cc_vertex_long
            if (s == g.gp_skip_seg) {
                // done by k_cc_edge_gp when the 4 child edges of interior edge j (ids base ..
                // base + 3) are in one of its blocks, and by the second of the two blocks
                // (gside) when they straddle two
                const int m1 = g.birth[s] - 1;
                if (__ldg(g.ehh[m1] + j).y >= 0) {
                    if (fr.gside) continue;
                    const int32_t base = 4 * j - (g.bw[m1] ? bprefix(g.bw[m1], g.bwp[m1], j) : 0);
                    if ((base & (kThreads - 1)) <= kThreads - 4) continue;
                }
            }
            cc_vertex_one<ORDER, CR>(x, fr, g, p, csv_list, s, j);
        }
    }
}

template <int ORDER, bool ADJ, bool BND>
static void cc_launch(const LevelDev &p, const ChildDev &c, const Frames &fr0, bool topo, const VSegs &g0,
                      const LevelDev *gp, cudaStream_t s, Launches &L) {
    const bool fpv = g0.level >= 2;  // face points born at this level are smoothed by the face kernel
    const bool one = fr0.nb == 1;
    const LevelDev gpd = gp ? *gp : LevelDev{};
    // levels >= 3 (quad kernel, c0 stored): the face points born at level l-1 are smoothed by the
    // face kernel too (a shuffle over the 4 faces around each); the vertex kernel skips them
    VSegs g = g0;
    int32_t fpo = -1;
    if (ORDER == 4 && g.level >= 3)
        for (int k = 0; k < g.nseg; ++k)
            if (g.type[k] == 1 && g.birth[k] == g.level - 1 && g.len[k] > 0) {
                fpo = g.start[k];
                g.len[k] = 0;
            }
    // the last level (grandparent path): the edge points born at l-1 come from the edge kernel's
    // block sums (the face points born at l-1 from the face kernel's shuffle, above); the older
    // vertices sum their faces' corner sums c0 (dropping c0 at this level and gathering their rings
    // directly was measured slower: 0.715 -> 0.731 ms on config 3)
    // last level >= 3: compact corner sums (fr.c0shift, set by the caller with the buffers)
    const Frames &fr = fr0;
    int32_t epo = -1;
    const int2 *ehh2 = nullptr;  // the level-(l-2) edges of those edge points
    if (gp) {
        for (int k = 0; k < g.nseg; ++k)
            if (g.type[k] == 2 && g.birth[k] == g.level - 1 && g.len[k] > 0) {
                epo = g.start[k];
                g.gp_skip_seg = k;
                ehh2 = g.ehh[g.birth[k] - 1];
            }
    }
    if (p.F > 0) {
        if constexpr (ORDER == 4) {
            // the last level recomputes its edge rows from the grandparent's (face_edge not
            // stored); a level before it with the grandparent edge kernel reads its own rows
            if (gp && p.face_edge == nullptr) {
                if (one) launch(L, "cc_face", k_cc_face_quad<ADJ, BND, 1, true>, dim3(grid_for(p.F)), dim3(kThreads), 0, s, p, c, fr, topo, fpv, gpd, fpo);
                else launch(L, "cc_face", k_cc_face_quad<ADJ, BND, 0, true>, dim3(grid_for(p.F)), dim3(kThreads), 0, s, p, c, fr, topo, fpv, gpd, fpo);
            } else {
                if (one) launch(L, "cc_face", k_cc_face_quad<ADJ, BND, 1, false>, dim3(grid_for(p.F)), dim3(kThreads), 0, s, p, c, fr, topo, fpv, gpd, fpo);
                else launch(L, "cc_face", k_cc_face_quad<ADJ, BND, 0, false>, dim3(grid_for(p.F)), dim3(kThreads), 0, s, p, c, fr, topo, fpv, gpd, fpo);
            }
        } else {
            if (one) launch(L, "cc_face", k_cc_face_gen<ORDER, ADJ, BND, 1>, dim3(grid_for(p.F)), dim3(kThreads), 0, s, p, c, fr, topo);
            else launch(L, "cc_face", k_cc_face_gen<ORDER, ADJ, BND, 0>, dim3(grid_for(p.F)), dim3(kThreads), 0, s, p, c, fr, topo);
        }
    }
    // the edge and vertex kernels only share read-only inputs: run them as parallel branches
    const bool fork = L.can_fork();
    cudaStream_t se = s;
    if (fork) {
        cudaEventRecord(L.ev_fork, s);
        cudaStreamWaitEvent(L.side, L.ev_fork, 0);
        se = L.side;
    }
    if (gp && gp->E > 0) {
        if (one) launch(L, "cc_edge", k_cc_edge_gp<1>, dim3(grid_for(gp->E)), dim3(kThreads), 0, se, p, gpd, c, fr, epo, ehh2);
        else launch(L, "cc_edge", k_cc_edge_gp<0>, dim3(grid_for(gp->E)), dim3(kThreads), 0, se, p, gpd, c, fr, epo, ehh2);
    } else if (p.E > 0) {
        constexpr int IT = 2;
        const unsigned gdim = grid_for(p.E, kThreads * IT);
        // p.crease: boundary/crease rules fused into the kernels (small levels, where a separate
        // pass costs a full dependent-kernel latency); otherwise crease.cu runs after this level.
        // Those small levels take one edge per thread (twice the CTAs: more latency hiding, less
        // wave quantisation; config 3 0.689 -> 0.684 ms -- two edges per thread stay better on the
        // large levels, 0.690 -> 0.698 ms with one)
        if (p.crease) {  // (static frames too: the same instantiation keeps them bitwise equal)
            const unsigned g1 = grid_for(p.E, kThreads);
            if (one) launch(L, "cc_edge", k_cc_edge<ORDER, ADJ, BND, 1, 1, true>, dim3(g1), dim3(kThreads), 0, se, p, c, fr, topo);
            else launch(L, "cc_edge", k_cc_edge<ORDER, ADJ, BND, 0, 1, true>, dim3(g1), dim3(kThreads), 0, se, p, c, fr, topo);
        } else {
            if (one) launch(L, "cc_edge", k_cc_edge<ORDER, ADJ, BND, 1, IT, false>, dim3(gdim), dim3(kThreads), 0, se, p, c, fr, topo);
            else launch(L, "cc_edge", k_cc_edge<ORDER, ADJ, BND, 0, IT, false>, dim3(gdim), dim3(kThreads), 0, se, p, c, fr, topo);
        }
    }
    if (L.build_open) {  // the level-0 build's special-list branch: read by the vertex kernel
        cudaStreamWaitEvent(s, L.ev_build, 0);
        L.build_open = false;
    }
    if (p.V > 0) {
        // 32-vertex warp tasks; >= 2 waves of 148 SMs for small levels, 4 tasks per warp for large
        // ones (128-vertex tasks with batched loads were measured slower)
        const unsigned nblk = (unsigned)std::max<int64_t>(grid_for(p.V, 4 * kThreads),
                                                          std::min<int64_t>(grid_for(p.V, kThreads), 2 * 148));
        // on the grandparent path, 128-thread vertex blocks (4096 registers) fit beside five
        // 256-thread edge blocks (61440) instead of taking an edge block's place (config 3
        // 0.5980 -> 0.5961 ms same-box)
        const bool half = gp && !p.crease;
        if (p.crease) launch(L, "cc_vertex", k_cc_vertex<ORDER == 4 ? 4 : 0, 1, true>, dim3(nblk), dim3(kThreads), 0, s, p, fr, g, c.sv_list);
        else if (half) launch(L, "cc_vertex", k_cc_vertex<ORDER == 4 ? 4 : 0, 1, false>, dim3(2 * nblk), dim3(kThreads / 2), 0, s, p, fr, g, c.sv_list);
        else launch(L, "cc_vertex", k_cc_vertex<ORDER == 4 ? 4 : 0, 1, false>, dim3(nblk), dim3(kThreads), 0, s, p, fr, g, c.sv_list);
        if (g.nlong > 0) {  // the poles' rings (reads what the vertex kernel reads, writes disjoint ids)
            const unsigned gl = grid_for(32 * (int64_t)g.nlong);
            if (p.crease) launch(L, "cc_vertex_long", k_cc_vertex_long<ORDER, true>, dim3(gl), dim3(kThreads), 0, s, p, fr, g);
            else launch(L, "cc_vertex_long", k_cc_vertex_long<ORDER, false>, dim3(gl), dim3(kThreads), 0, s, p, fr, g);
        }
    }
    if (fork) {
        cudaEventRecord(L.ev_join, L.side);
        cudaStreamWaitEvent(s, L.ev_join, 0);
    }
}

template <int ORDER>
static void cc_dispatch(const LevelDev &p, const ChildDev &c, const Frames &fr, bool topo, bool adj, const VSegs &g,
                        const LevelDev *gp, cudaStream_t s, Launches &L) {
    const bool bnd = p.B > 0;
    if (adj && topo) {
        if (bnd) cc_launch<ORDER, true, true>(p, c, fr, topo, g, gp, s, L);
        else cc_launch<ORDER, true, false>(p, c, fr, topo, g, gp, s, L);
    } else {
        cc_launch<ORDER, false, false>(p, c, fr, topo, g, gp, s, L);
    }
}

void cc_level(const LevelDev &p, const ChildDev &c, const Frames &fr, bool topo, bool adj, const VSegs &g,
              const LevelDev *gp, cudaStream_t s, Launches &L) {
    // level-0 meshes of uniform order use the generic kernels too (their M^T comes from the sort);
    // levels >= 1 are reduced quad matrices
    if (p.order == 4 && p.face_off == nullptr) cc_dispatch<4>(p, c, fr, topo, adj, g, gp, s, L);
    else cc_dispatch<0>(p, c, fr, topo, adj, g, gp, s, L);
}

}  // namespace alsub
