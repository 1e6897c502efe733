// crease_fused.cuh -- the boundary/crease module of PAPER.md §3.3 evaluated INSIDE the
// Catmull-Clark edge and vertex kernels (no separate crease pass).
//
// A level's special edges (boundary = inf crease, reading R6, and creased edges) form a list in
// edge-id order whose entry j has children 2j, 2j+1 at the next level (dead children keep
// sigma = 0).  Bit e of `spw` says whether edge e is on the list; its index is the per-word
// prefix `spwpre` plus a popcount.  Child bits / prefixes are closed-form (children base+0, base+1
// of every listed edge), exactly like the boundary words.
// Special vertices: identity table over the level-0 vertices, then one entry per listed edge (its
// edge point) per level; sv_list holds each special vertex's incident special edges (ascending).
#pragma once
#include "internal.h"

namespace alsub {

ALSUB_D int32_t sp_index(const uint32_t *__restrict__ w, const int32_t *__restrict__ wp, int32_t e) {
    const uint32_t word = __ldg(w + (e >> 5)), bit = 1u << (e & 31);
    if (!(word & bit)) return -1;
    return __ldg(wp + (e >> 5)) + __popc(word & (bit - 1u));
}
ALSUB_D int32_t sp_prefix(const uint32_t *__restrict__ w, const int32_t *__restrict__ wp, int32_t e) {
    return __ldg(wp + (e >> 5)) + __popc(__ldg(w + (e >> 5)) & ((1u << (e & 31)) - 1u));
}

// edge rule (reading R7): sigma >= 1 midpoint, 0 < sigma < 1 blend, 0 smooth
ALSUB_D P3 crease_edge_point(float sg, P3 smooth, P3 mid) {
    if (sg >= 1.0f) return mid;
    if (sg > 0.0f) return (1.0f - sg) * smooth + sg * mid;
    return smooth;
}

// mean of the OTHER finite non-boundary creases at special vertex ix (reading R8); shared by the
// fused crease rules and the separate crease pass (crease.cu)
ALSUB_D float sigma_bar(const LevelDev &p, int32_t ix, int32_t j, float se) {
    float sum = 0.0f;
    int n = 0;
    for (int32_t q = p.sv_off[ix]; q < p.sv_off[ix + 1]; ++q) {
        const int32_t k = p.sv_list[q];
        if (k == j) continue;
        const SpEdge o = p.sp[k];
        if (!(o.sigma > 0.0f) || isinf(o.sigma) || (o.flags & kSpBoundary)) continue;
        sum += o.sigma;
        ++n;
    }
    return n > 0 ? sum / (float)n : se;
}

// crease inheritance of special edge j (Eqs. sigma_ij / sigma_jk): children 2j (at
// endpoint a) and 2j+1 (at b) with child edge ids base+0 / base+1, and the table entries of the
// new special vertex (the edge point ep)
ALSUB_D void fused_inherit(const LevelDev &p, const ChildDev &c, int32_t j, const SpEdge &se, int32_t base,
                           int32_t ep) {
    float ca = 0.0f, cb = 0.0f;
    if (se.sigma > 0.0f) {
        if ((se.flags & kSpBoundary) || isinf(se.sigma)) {
            ca = cb = se.sigma;
        } else {
            ca = fmaxf(0.25f * (sigma_bar(p, se.ia, j, se.sigma) + 3.0f * se.sigma) - 1.0f, 0.0f);
            cb = fmaxf(0.25f * (sigma_bar(p, se.ib, j, se.sigma) + 3.0f * se.sigma) - 1.0f, 0.0f);
        }
    }
    const int32_t iep = p.nsv + j;
    c.sp[2 * j] = SpEdge{base + 0, se.a, ep, se.ia, iep, ca, se.flags, 0};
    c.sp[2 * j + 1] = SpEdge{base + 1, se.b, ep, se.ib, iep, cb, se.flags, 0};
    const int32_t tot = 2 * p.nsp;  // = parent sv_off[nsv]
    c.sv_vtx[iep] = ep;
    c.sv_off[iep] = tot + 2 * j;
    *reinterpret_cast<int2 *>(c.sv_list + tot + 2 * j) = make_int2(2 * j, 2 * j + 1);  // (tot even: 8-B aligned)
    if (j == p.nsp - 1) c.sv_off[iep + 1] = tot + 2 * p.nsp;
}

// child special-edge bits (children base, base+1 of a listed edge) and, for the child words that
// start inside this edge's child block [base, base + nch), their prefix 2 ip(e) + listed * min(k, 2)
ALSUB_D void fused_child_words(const ChildDev &c, int32_t base, int32_t nch, int32_t ip, bool listed) {
    if (listed) {
        atomicOr(c.spw + (base >> 5), 1u << (base & 31));
        atomicOr(c.spw + ((base + 1) >> 5), 1u << ((base + 1) & 31));
    }
    const int32_t w = (base + 31) >> 5;
    if (32 * w < base + nch) c.spwpre[w] = 2 * ip + (listed ? min(32 * w - base, 2) : 0);
}

// crease valency k = C1, sharpness s = mean sigma (Eqs. CC_crease_valency / _vsharpness, fused as in
// P:L676-681) and the first two sharp neighbours of special vertex i (= v); transforms i's list
// for the child level (entry k -> 2k + [v is b_k])
struct VCr {
    int k;
    float s;
    int32_t nb0, nb1;
};
ALSUB_D VCr vertex_crease(const LevelDev &p, int32_t *child_list, int32_t i, int32_t v) {
    VCr r{0, 0.0f, -1, -1};
    int inf = 0;
    float sum = 0.0f;
    for (int32_t q = p.sv_off[i]; q < p.sv_off[i + 1]; ++q) {
        const int32_t kk = p.sv_list[q];
        const SpEdge o = p.sp[kk];
        if (child_list) child_list[q] = 2 * kk + (o.b == v ? 1 : 0);
        if (!(o.sigma > 0.0f)) continue;
        const int32_t other = o.a == v ? o.b : o.a;
        if (r.k == 0) r.nb0 = other;
        else if (r.k == 1) r.nb1 = other;
        ++r.k;
        if (isinf(o.sigma)) inf = 1;
        else sum += o.sigma;
    }
    r.s = r.k == 0 ? 0.0f : (inf ? __int_as_float(0x7f800000) : sum / (float)r.k);
    return r;
}

// vertex rule (reading R7): crease 3/4 p + 1/8 (p_a + p_b) for k = 2 (= Eq. CC_boundary on
// boundaries), corner p for k >= 3, (1 - s) smooth + s sharp for s < 1; k <= 1: smooth
ALSUB_D P3 crease_vertex_point(const VCr &cr, PR P, int32_t v, P3 smooth) {
    if (cr.k < 2) return smooth;
    const P3 pv = ld3(P, v);
    const P3 sh = cr.k == 2 ? 0.75f * pv + 0.125f * (ld3(P, cr.nb0) + ld3(P, cr.nb1)) : pv;
    if (cr.s >= 1.0f) return sh;
    return (1.0f - cr.s) * smooth + cr.s * sh;
}

}  // namespace alsub
