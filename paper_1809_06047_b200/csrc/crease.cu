// crease.cu -- boundary and crease module (§3.3).
//
// A level's special edges are its boundary edges (E value 1) and its creased edges
// (non-zeros of C); boundary edges are treated as infinitely sharp creases (reading R6).
//   k_sp_edge  per special edge: edge-point override (midpoint for sigma >= 1, blend below) and,
//              fused as in P:L676-681, the crease valency k = C1 and sharpness sums at both
//              endpoints (accumulated into the small special-vertex table, not V-sized arrays).
//   k_sp_vert  per special vertex: s = (sum sigma)/k (Eq. CC_crease_vsharpness) and the vertex
//              override (crease 3/4,1/8,1/8 for k = 2 -- = Eq. CC_boundary on boundaries --,
//              corner for k >= 3, semi-sharp blend for s < 1).
//   k_sp_count / scan / k_sp_fill  the paper's two-stage crease inheritance:
//              count surviving children per crease, scan, fill the child list in edge-id order.
#include "internal.h"

namespace alsub {

__device__ __forceinline__ bool is_inf(float x) { return isinf(x); }

__global__ void __launch_bounds__(kThreads) k_sp_edge(LevelDev p, Frames fr, int32_t ep_base, bool accumulate) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= p.sp_cap || j >= *p.sp_count) return;
    const SpEdge se = p.sp[j];
    const float sg = se.sigma;
    const bool sharp = sg >= 1.0f;  // includes +inf
    for (int f = 0; f < fr.nb; ++f) {
        const float *P = fr.P + f * fr.Pstride;
        float *Pn = fr.Pn + f * fr.Pnstride;
        const P3 mid = 0.5f * (ld3(P, se.a) + ld3(P, se.b));
        const int64_t o = (int64_t)ep_base + se.e;
        if (sharp) st3(Pn, o, mid);
        else st3(Pn, o, (1.0f - sg) * ld3c(Pn, o) + sg * mid);
    }
    if (!accumulate) return;
    const int32_t ends[2] = {se.ia, se.ib}, other[2] = {se.b, se.a};
    const bool inf = is_inf(sg);
    const bool fin_crease = !inf && !(se.flags & kSpBoundary);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        SvAcc *a = p.sva + ends[k];
        const int slot = atomicAdd(&a->k, 1);
        if (slot == 0) a->nb0 = other[k];
        else if (slot == 1) a->nb1 = other[k];
        if (inf) atomicOr(&a->inf, 1);
        else atomicAdd(&a->sum, sg);
        if (fin_crease) {
            atomicAdd(&a->nfin, 1);
            atomicAdd(&a->finsum, sg);
        }
    }
}

__global__ void __launch_bounds__(kThreads) k_sp_vert(LevelDev p, Frames fr, bool accumulate) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p.sv_cap || i >= *p.sv_count) return;
    SvAcc a = p.sva[i];
    float s;
    if (accumulate) {
        s = a.k == 0 ? 0.0f : (a.inf ? __int_as_float(0x7f800000) : a.sum / (float)a.k);
        p.sva[i].s = s;
    } else {
        s = a.s;
    }
    if (a.k < 2) return;
    const int32_t v = p.sv_vtx[i];
    for (int f = 0; f < fr.nb; ++f) {
        const float *P = fr.P + f * fr.Pstride;
        float *Pn = fr.Pn + f * fr.Pnstride;
        const P3 pv = ld3(P, v);
        const P3 sh = a.k == 2 ? 0.75f * pv + 0.125f * (ld3(P, a.nb0) + ld3(P, a.nb1)) : pv;
        if (s >= 1.0f) st3(Pn, v, sh);
        else st3(Pn, v, (1.0f - s) * ld3c(Pn, v) + s * sh);
    }
}

void crease_eval(const LevelDev &p, const Frames &fr, int32_t ep_base, bool accumulate, cudaStream_t s, Launches &L) {
    if (p.sp_cap <= 0) return;
    if (accumulate && p.sv_cap > 0) cudaMemsetAsync(p.sva, 0, sizeof(SvAcc) * (size_t)p.sv_cap, s);
    k_sp_edge<<<grid_for(p.sp_cap), kThreads, 0, s>>>(p, fr, ep_base, accumulate);
    L.done("sp_edge", s);
    if (p.sv_cap > 0) {
        k_sp_vert<<<grid_for(p.sv_cap), kThreads, 0, s>>>(p, fr, accumulate);
        L.done("sp_vert", s);
    }
}

// ---------------- inheritance ----------------
// Child sharpness of crease e = (a, b) at endpoint x (Eqs. sigma_ij / sigma_jk, with
// reading R8: sigma_bar = mean of the OTHER finite creases at x, sigma_e itself at a chain end).
__device__ __forceinline__ float child_sigma(const SpEdge &se, const SvAcc &ax) {
    if ((se.flags & kSpBoundary) || is_inf(se.sigma)) return se.sigma;
    const float sbar = ax.nfin > 1 ? (ax.finsum - se.sigma) / (float)(ax.nfin - 1) : se.sigma;
    const float c = 0.25f * (sbar + 3.0f * se.sigma) - 1.0f;
    return c > 0.0f ? c : 0.0f;
}

__global__ void __launch_bounds__(kThreads) k_sp_count(LevelDev p, int32_t *__restrict__ cnt) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= p.sp_cap) return;
    if (j >= *p.sp_count) { cnt[j] = 0; return; }
    const SpEdge se = p.sp[j];
    const float ca = child_sigma(se, p.sva[se.ia]), cb = child_sigma(se, p.sva[se.ib]);
    cnt[j] = (ca > 0.0f) + (cb > 0.0f);
}

template <int SCHEME>
__global__ void __launch_bounds__(kThreads) k_sp_fill(LevelDev p, ChildDev c, int32_t ep_base,
                                                    const int32_t *__restrict__ off) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    const int32_t count = *p.sp_count, nsv = *p.sv_count;
    if (j == 0) *c.sv_count = nsv + count;
    if (j >= p.sp_cap || j >= count) return;
    const SpEdge se = p.sp[j];
    const int32_t ep = ep_base + se.e;
    c.sv_vtx[nsv + j] = ep;  // the edge point joins the special-vertex table
    int32_t base;
    if constexpr (SCHEME == 0) base = (p.B > 0) ? 4 * se.e - bprefix(p.bnd_word, p.bnd_wpre, se.e) : 4 * se.e;
    else base = p.loop_base[se.e];
    const float ca = child_sigma(se, p.sva[se.ia]), cb = child_sigma(se, p.sva[se.ib]);
    int32_t o = off[j];
    if (ca > 0.0f) {
        SpEdge ch{base + 0, se.a, ep, se.ia, nsv + j, ca, se.flags, 0};
        c.sp[o++] = ch;
    }
    if (cb > 0.0f) {
        SpEdge ch{base + 1, se.b, ep, se.ib, nsv + j, cb, se.flags, 0};
        c.sp[o++] = ch;
    }
}

void crease_inherit(const LevelDev &p, const ChildDev &c, int scheme, int32_t ep_base, int32_t *cnt, int32_t *off,
                    void *scratch, cudaStream_t s, Launches &L) {
    if (p.sp_cap <= 0) {
        cudaMemsetAsync(c.sp_count, 0, sizeof(int32_t), s);
        cudaMemcpyAsync(c.sv_count, p.sv_count, sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
        return;
    }
    k_sp_count<<<grid_for(p.sp_cap), kThreads, 0, s>>>(p, cnt);
    L.done("sp_count", s);
    scan_exclusive(cnt, off, p.sp_cap, c.sp_count, scratch, s, L);
    if (scheme == 0) k_sp_fill<0><<<grid_for(p.sp_cap), kThreads, 0, s>>>(p, c, ep_base, off);
    else k_sp_fill<1><<<grid_for(p.sp_cap), kThreads, 0, s>>>(p, c, ep_base, off);
    L.done("sp_fill", s);
}

// ---------------- boundary-word prefix ----------------
__global__ void k_popc_words(const uint32_t *__restrict__ w, int32_t n, int32_t *__restrict__ c) {
    int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) c[i] = __popc(w[i]);
}

void bnd_prefix(uint32_t *words, int32_t *wcnt, int32_t *wpre, int32_t nwords, void *scratch, cudaStream_t s,
                Launches &L) {
    k_popc_words<<<grid_for(nwords), kThreads, 0, s>>>(words, nwords, wcnt);
    L.done("popc_words", s);
    scan_exclusive(wcnt, wpre, nwords, nullptr, scratch, s, L);
}

// ---------------- topology export ----------------
template <int ORDER>
__global__ void k_export_edges(LevelDev p, int32_t *edge_vtx, int32_t *edge_face) {
    const int32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= p.E) return;
    const Topo<ORDER> tp{p.face_off, p.slot_face};
    const int32_t h = p.edge_slot[e], tw = p.face_twin[h];
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
    if (p.order == 4) k_export_edges<4><<<grid_for(p.E), kThreads, 0, s>>>(p, edge_vtx, edge_face);
    else if (p.order == 3) k_export_edges<3><<<grid_for(p.E), kThreads, 0, s>>>(p, edge_vtx, edge_face);
    else k_export_edges<0><<<grid_for(p.E), kThreads, 0, s>>>(p, edge_vtx, edge_face);
    L.done("export_edges", s);
}

}  // namespace alsub
