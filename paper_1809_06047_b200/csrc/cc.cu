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
#include "internal.h"

namespace alsub {

// base id of the child-edge block of parent edge e: sum_{e' < e} (4 - bnd_e')
template <bool BND>
ALSUB_D int32_t cc_base(const uint32_t *w, const int32_t *wp, int32_t e) {
    if constexpr (BND) return 4 * e - bprefix(w, wp, e);
    else return 4 * e;
}

// ---------------- face kernel: reduced quad matrix (levels >= 1, or all-quad input) --------
template <bool ADJ, bool BND>
__global__ void __launch_bounds__(kThreads) k_cc_face_quad(LevelDev p, ChildDev c, Frames fr, bool topo) {
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= p.F) return;
    const int4 fv = __ldg(reinterpret_cast<const int4 *>(p.face_vtx) + r);
    const int32_t v[4] = {fv.x, fv.y, fv.z, fv.w};
    const int32_t V = p.V, F = p.F;
    for (int f = 0; f < fr.nb; ++f) {
        const float *P = fr.P + f * fr.Pstride;
        P3 s = ld3(P, v[0]) + ld3(P, v[1]) + ld3(P, v[2]) + ld3(P, v[3]);
        st3(fr.Pn + f * fr.Pnstride, V + r, 0.25f * s);
    }
    if (!topo) return;
    const int4 fe = __ldg(reinterpret_cast<const int4 *>(p.face_edge) + r);
    const int32_t e[4] = {fe.x, fe.y, fe.z, fe.w};
    int4 *cfv = reinterpret_cast<int4 *>(c.face_vtx) + 4 * (int64_t)r;
#pragma unroll
    for (int t = 0; t < 4; ++t)
        cfv[t] = make_int4(v[t], V + F + e[t], V + r, V + F + e[(t + 3) & 3]);
    if constexpr (ADJ) {
        const int4 ft = __ldg(reinterpret_cast<const int4 *>(p.face_twin) + r);
        const int32_t tw[4] = {ft.x, ft.y, ft.z, ft.w};
        int32_t base[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) base[t] = cc_base<BND>(p.bnd_word, p.bnd_wpre, e[t]);
        int4 *cfe = reinterpret_cast<int4 *>(c.face_edge) + 4 * (int64_t)r;
        int4 *cft = reinterpret_cast<int4 *>(c.face_twin) + 4 * (int64_t)r;
        const int32_t h0 = 4 * r;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int tn = (t + 1) & 3, tp = (t + 3) & 3;
            const int32_t h = h0 + t, hp = h0 + tp;
            cfe[t] = make_int4(base[t] + (v[t] > v[tn]), base[t] + 2 + (tw[t] >= 0 && tw[t] < h),
                               base[tp] + 2 + (tw[tp] >= 0 && tw[tp] < hp), base[tp] + (v[t] > v[tp]));
            const int32_t twn = tw[t] >= 0 ? ((tw[t] & ~3) | ((tw[t] + 1) & 3)) : -1;
            cft[t] = make_int4(tw[t] >= 0 ? 4 * twn + 3 : -1, 4 * (h0 + tn) + 2, 4 * hp + 1,
                               tw[tp] >= 0 ? 4 * tw[tp] : -1);
        }
        c.vtx_slot0[V + r] = 4 * h0 + 2;
    }
}

// ---------------- face kernel: general matrix (level 0: mixed orders or triangles) ---------
template <int ORDER, bool ADJ, bool BND>
__global__ void __launch_bounds__(kThreads) k_cc_face_gen(LevelDev p, ChildDev c, Frames fr, bool topo) {
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= p.F) return;
    const Topo<ORDER> tp{p.face_off, p.slot_face};
    const int32_t o = tp.first(r), n = tp.order(r);
    const int32_t V = p.V, F = p.F;
    const float inv = 1.0f / (float)n;
    for (int f = 0; f < fr.nb; ++f) {
        const float *P = fr.P + f * fr.Pstride;
        P3 s = p3zero();
        for (int32_t t = 0; t < n; ++t) s = s + ld3(P, __ldg(p.face_vtx + o + t));
        st3(fr.Pn + f * fr.Pnstride, V + r, inv * s);
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
            reinterpret_cast<int4 *>(c.face_twin)[h] =
                make_int4(twt >= 0 ? 4 * tp.next(twt) + 3 : -1, 4 * hn + 2, 4 * hp + 1, twp >= 0 ? 4 * twp : -1);
        }
    }
    if constexpr (ADJ) c.vtx_slot0[V + r] = 4 * o + 2;
}

// ---------------- edge kernel ----------------
template <int ORDER, bool ADJ, bool BND>
__global__ void __launch_bounds__(kThreads) k_cc_edge(LevelDev p, ChildDev c, Frames fr, bool topo) {
    const int32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= p.E) return;
    const Topo<ORDER> tp{p.face_off, p.slot_face};
    const int32_t h = __ldg(p.edge_slot + e);
    const int32_t tw = __ldg(p.face_twin + h);
    const int32_t hn = tp.next(h);
    const int32_t va = __ldg(p.face_vtx + h), vb = __ldg(p.face_vtx + hn);
    const int32_t V = p.V, F = p.F;
    const int32_t fr_r = V + tp.face(h);
    const int32_t fr_s = tw >= 0 ? V + tp.face(tw) : -1;
    for (int f = 0; f < fr.nb; ++f) {
        const float *P = fr.P + f * fr.Pstride;
        float *Pn = fr.Pn + f * fr.Pnstride;
        const P3 ab = ld3(P, va) + ld3(P, vb);
        P3 out;
        if (tw < 0) out = 0.5f * ab;
        else out = 0.25f * (ab + ld3c(Pn, fr_r) + ld3c(Pn, fr_s));
        st3(Pn, (int64_t)V + F + e, out);
    }
    if constexpr (ADJ) {
        if (!topo) return;
        const int32_t base = cc_base<BND>(p.bnd_word, p.bnd_wpre, e);
        const int32_t h_ab = va < vb ? h : tw, h_ba = va < vb ? tw : h;
        int32_t o0 = INT32_MAX, o1 = INT32_MAX;
        if (h_ab >= 0) { o0 = 4 * h_ab; o1 = 4 * tp.next(h_ab) + 3; }
        if (h_ba >= 0) { o0 = min(o0, 4 * tp.next(h_ba) + 3); o1 = min(o1, 4 * h_ba); }
        c.edge_slot[base + 0] = o0;
        c.edge_slot[base + 1] = o1;
        c.edge_slot[base + 2] = min(4 * h + 1, 4 * hn + 2);
        if (tw >= 0) c.edge_slot[base + 3] = min(4 * tw + 1, 4 * tp.next(tw) + 2);
        c.vtx_slot0[V + F + e] = 4 * h + 1;
        if constexpr (BND) {
            if (tw < 0) {
                atomicOr(c.bnd_word + (base >> 5), 1u << (base & 31));
                atomicOr(c.bnd_word + ((base + 1) >> 5), 1u << ((base + 1) & 31));
            }
        }
    }
}

// ---------------- vertex kernel: 1-ring walk ----------------
template <int ORDER, bool ADJ>
__global__ void __launch_bounds__(kThreads) k_cc_vertex(LevelDev p, ChildDev c, Frames fr, bool topo) {
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= p.V) return;
    const Topo<ORDER> tp{p.face_off, p.slot_face};
    const int32_t h0 = __ldg(p.vtx_slot0 + v);
    if constexpr (ADJ) {
        if (topo) c.vtx_slot0[v] = h0 >= 0 ? 4 * h0 : -1;  // corner 0 of child face h0
    }
    const int32_t V = p.V;
    for (int f = 0; f < fr.nb; ++f) {
        const float *P = fr.P + f * fr.Pstride;
        float *Pn = fr.Pn + f * fr.Pnstride;
        const P3 pv = ld3(P, v);
        if (h0 < 0) { st3(Pn, v, pv); continue; }
        P3 acc = p3zero();
        int32_t h = h0, n = 0;
        bool bnd = false;
        do {
            acc = acc + ld3(P, __ldg(p.face_vtx + tp.next(h))) + ld3c(Pn, V + tp.face(h));
            ++n;
            h = __ldg(p.face_twin + tp.prev(h));
            if (h < 0) { bnd = true; break; }
        } while (h != h0 && n < p.S);
        if (bnd) { st3(Pn, v, pv); continue; }  // boundary: set by the crease/boundary override
        const float inv = 1.0f / (float)n;
        st3(Pn, v, (1.0f - 2.0f * inv) * pv + (inv * inv) * acc);
    }
}

// ------------------------------------------------------------------------------------------
template <int ORDER, bool ADJ, bool BND>
static void cc_launch(const LevelDev &p, const ChildDev &c, const Frames &fr, bool topo, cudaStream_t s,
                      Launches &L) {
    if (p.F > 0) {
        if constexpr (ORDER == 4) k_cc_face_quad<ADJ, BND><<<grid_for(p.F), kThreads, 0, s>>>(p, c, fr, topo);
        else k_cc_face_gen<ORDER, ADJ, BND><<<grid_for(p.F), kThreads, 0, s>>>(p, c, fr, topo);
        L.done("cc_face", s);
    }
    if (p.E > 0) {
        k_cc_edge<ORDER, ADJ, BND><<<grid_for(p.E), kThreads, 0, s>>>(p, c, fr, topo);
        L.done("cc_edge", s);
    }
    if (p.V > 0) {
        k_cc_vertex<ORDER, ADJ><<<grid_for(p.V), kThreads, 0, s>>>(p, c, fr, topo);
        L.done("cc_vertex", s);
    }
}

template <int ORDER>
static void cc_dispatch(const LevelDev &p, const ChildDev &c, const Frames &fr, bool topo, bool adj, cudaStream_t s,
                        Launches &L) {
    const bool bnd = p.B > 0;
    if (adj && topo) {
        if (bnd) cc_launch<ORDER, true, true>(p, c, fr, topo, s, L);
        else cc_launch<ORDER, true, false>(p, c, fr, topo, s, L);
    } else {
        cc_launch<ORDER, false, false>(p, c, fr, topo, s, L);
    }
}

void cc_level(const LevelDev &p, const ChildDev &c, const Frames &fr, bool topo, bool adj, void *scratch,
              cudaStream_t s, Launches &L) {
    (void)scratch;
    const bool need_mask = adj && topo && p.B > 0;
    if (need_mask) {
        const int32_t nw = (int32_t)ceil_div(c.E > 0 ? c.E : 1, 32);
        cudaMemsetAsync(c.bnd_word, 0, sizeof(uint32_t) * nw, s);
    }
    if (p.order == 4) cc_dispatch<4>(p, c, fr, topo, adj, s, L);
    else if (p.order == 3) cc_dispatch<3>(p, c, fr, topo, adj, s, L);
    else cc_dispatch<0>(p, c, fr, topo, adj, s, L);
    if (need_mask) {
        const int32_t nw = (int32_t)ceil_div(c.E > 0 ? c.E : 1, 32);
        bnd_prefix(c.bnd_word, c.bnd_wcnt, c.bnd_wpre, nw, scratch, s, L);
    }
}

}  // namespace alsub
