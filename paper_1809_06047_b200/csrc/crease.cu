// crease.cu -- boundary and crease module (§3.3).
//
// A level's special edges are its boundary edges (E value 1) and its creased edges
// (non-zeros of C); boundary edges are treated as infinitely sharp creases (reading R6).
// The whole module -- edge overrides, vertex overrides, crease inheritance -- is one
// gather kernel per level over the special-edge list and the special-vertex CSR (common.cuh).
#include "crease_fused.cuh"
#include "internal.h"

namespace alsub {

__device__ __forceinline__ bool is_inf(float x) { return isinf(x); }

// One kernel per level, no atomics, no grid-wide dependency:
//   threads [0, nsp)        special edge j: edge-point override (midpoint for sigma >= 1, blend
//                           below) and -- inherit -- its two children 2j, 2j+1 with
//                           Chaikin sharpness (Eqs. sigma_ij / sigma_jk, reading R8)
//                           and the table entries of its edge point;
//   threads [nsp, nsp+nsv)  special vertex i: crease valency k = C1 and sharpness s = mean sigma
//                           (Eqs. CC_crease_valency / _vsharpness, fused as in P:L676-681) from its
//                           incident-special-edge list, then the vertex override: crease
//                           3/4,1/8,1/8 for k = 2 (= Eq. CC_boundary on boundaries), corner for
//                           k >= 3, (1-s) smooth + s sharp for s < 1; -- inherit -- its child list.
// Sums run over each list in ascending edge id, the oracle's order, so they are bit-identical.
struct CreaseArgs {
    LevelDev p;
    ChildDev c;
    Frames fr;
    int32_t ep_base;
    int32_t scheme;   // 0 CC (child ids from the boundary prefix), 1 Loop (loop_base)
    int32_t inherit;  // build the child special lists
};

__global__ void __launch_bounds__(kThreads) k_crease(CreaseArgs A) {
    ALSUB_GRID_WAIT();
    const LevelDev &p = A.p;
    const Frames &fr = A.fr;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < p.nsp) {
        const int32_t j = (int32_t)t;
        const SpEdge se = p.sp[j];
        const float sg = se.sigma;
        if (sg > 0.0f) {
            for (int f = 0; f < fr.nb; ++f) {
                const PR P = fr.rd(f);
                const PW Pn = fr.wr(f);
                const P3 mid = 0.5f * (ld3(P, se.a) + ld3(P, se.b));
                const int64_t o = (int64_t)A.ep_base + se.e;
                if (sg >= 1.0f) st3(Pn, o, mid);  // includes +inf (boundary)
                else st3(Pn, o, (1.0f - sg) * ld3c(Pn, o) + sg * mid);
            }
        }
        if (!A.inherit) return;
        float ca = 0.0f, cb = 0.0f;
        if (sg > 0.0f) {
            if ((se.flags & kSpBoundary) || is_inf(sg)) {
                ca = cb = sg;
            } else {
                ca = fmaxf(0.25f * (sigma_bar(p, se.ia, j, sg) + 3.0f * sg) - 1.0f, 0.0f);
                cb = fmaxf(0.25f * (sigma_bar(p, se.ib, j, sg) + 3.0f * sg) - 1.0f, 0.0f);
            }
        }
        int32_t base;
        if (A.scheme == 0) base = (p.B > 0) ? 4 * se.e - bprefix(p.bnd_word, p.bnd_wpre, se.e) : 4 * se.e;
        else base = __ldg(p.loop_base + se.e);
        const ChildDev &c = A.c;
        const int32_t ep = A.ep_base + se.e, iep = p.nsv + j;
        c.sp[2 * j] = SpEdge{base + 0, se.a, ep, se.ia, iep, ca, se.flags, 0};
        c.sp[2 * j + 1] = SpEdge{base + 1, se.b, ep, se.ib, iep, cb, se.flags, 0};
        // the edge point joins the special-vertex table with entries {2j, 2j+1}
        const int32_t tot = 2 * p.nsp;  // = parent sv_off[nsv]
        c.sv_vtx[iep] = ep;
        c.sv_off[iep] = tot + 2 * j;
        *reinterpret_cast<int2 *>(c.sv_list + tot + 2 * j) = make_int2(2 * j, 2 * j + 1);  // (tot even: 8-B aligned)
        if (j == p.nsp - 1) c.sv_off[iep + 1] = tot + 2 * p.nsp;
        return;
    }
    const int64_t i64 = t - p.nsp;
    if (i64 >= p.nsv) return;
    const int32_t i = (int32_t)i64;
    const int32_t v = p.sv_vtx[i];
    const int32_t q0 = p.sv_off[i], q1 = p.sv_off[i + 1];
    int k = 0, inf = 0;
    float sum = 0.0f;
    int32_t nb0 = -1, nb1 = -1;
    for (int32_t q = q0; q < q1; ++q) {
        const int32_t kk = p.sv_list[q];
        const SpEdge o = p.sp[kk];
        if (A.inherit) A.c.sv_list[q] = 2 * kk + (o.b == v ? 1 : 0);
        if (!(o.sigma > 0.0f)) continue;
        const int32_t other = o.a == v ? o.b : o.a;
        if (k == 0) nb0 = other;
        else if (k == 1) nb1 = other;
        ++k;
        if (is_inf(o.sigma)) inf = 1;
        else sum += o.sigma;
    }
    if (k < 2) return;
    const float s = inf ? __int_as_float(0x7f800000) : sum / (float)k;
    for (int f = 0; f < fr.nb; ++f) {
        const PR P = fr.rd(f);
        const PW Pn = fr.wr(f);
        const P3 pv = ld3(P, v);
        const P3 sh = k == 2 ? 0.75f * pv + 0.125f * (ld3(P, nb0) + ld3(P, nb1)) : pv;
        if (s >= 1.0f) st3(Pn, v, sh);
        else st3(Pn, v, (1.0f - s) * ld3c(Pn, v) + s * sh);
    }
}

void crease_level(const LevelDev &p, const ChildDev &c, const Frames &fr, int32_t ep_base, int scheme, bool inherit,
                  cudaStream_t s, Launches &L) {
    const int64_t work = (int64_t)p.nsp + p.nsv;
    if (work <= 0) return;
    CreaseArgs A{p, c, fr, ep_base, scheme, inherit ? 1 : 0};
    launch(L, "crease", k_crease, dim3(grid_for(work)), dim3(kThreads), 0, s, A);
}

// ---------------- topology export ----------------
template <int ORDER>
__global__ void k_export_edges(LevelDev p, int32_t *edge_vtx, int32_t *edge_face) {
    ALSUB_GRID_WAIT();
    const int32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= p.E) return;
    const Topo<ORDER> tp{p.face_off, p.slot_face};
    const int2 hh = p.edge_hh[e];
    const int32_t h = hh.x, tw = hh.y;
    const int32_t va = p.face_vtx[h], vb = p.face_vtx[tp.next(h)];
    const int32_t fh = tp.face(h), ft = tw >= 0 ? tp.face(tw) : -1;
    if (edge_vtx) {
        edge_vtx[2 * e] = min(va, vb);
        edge_vtx[2 * e + 1] = max(va, vb);
    }
    if (edge_face) {
        edge_face[2 * e] = va < vb ? fh : ft;
        edge_face[2 * e + 1] = va < vb ? ft : fh;
    }
}

void export_edges(const LevelDev &p, int32_t *edge_vtx, int32_t *edge_face, cudaStream_t s, Launches &L) {
    if (p.E <= 0) return;
    if (p.order == 4) launch(L, "export_edges", k_export_edges<4>, dim3(grid_for(p.E)), dim3(kThreads), 0, s, p, edge_vtx, edge_face);
    else if (p.order == 3) launch(L, "export_edges", k_export_edges<3>, dim3(grid_for(p.E)), dim3(kThreads), 0, s, p, edge_vtx, edge_face);
    else launch(L, "export_edges", k_export_edges<0>, dim3(grid_for(p.E)), dim3(kThreads), 0, s, p, edge_vtx, edge_face);
}

}  // namespace alsub
