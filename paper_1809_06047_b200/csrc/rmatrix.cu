// rmatrix.cu -- the refinement matrix R = R_{L-1} ... R_0 of a fixed topology (SURVEY.md 8(f)
// NEXT-1; "a single SpMV"; static mode P:L525-529).
//
// Row i of R holds the weights of the level-L vertex i on the control vertices.  By locality,
// vertex i lies in (the closure of) some control face f, and its row is supported on the 1-ring
// vertex set S_f of f (the vertices of the faces sharing a vertex with f): every subdivision rule
// reads a one-ring.  Construction without symbolic sparse products:
//   owner(i)   smallest control face among the control ancestors of the level-L faces around i
//   S_f        1-ring vertex set of f, ascending (host, from the control mesh)
//   colours    greedy colouring of the control vertices such that no S_f holds two vertices of one
//              colour (host)
//   probe      one 3-channel frame per three colours: channel c of probe p is the indicator of
//              colour 3p + c; the verified static path (alsub_eval_frames) refines the probes
//   assemble   R[i, j] = probe value of colour(j) at row i, for j in S_owner(i): the only vertex of
//              that colour in the support, so the probe reads exactly one weight
// Rows are stored in CSR (exact zeros dropped) in output-vertex order.
//
// Evaluation: P_L = R P_0 for batches of 32 frames.  A warp owns 8 consecutive rows;
// lane = frame, the control positions are frame-interleaved ([V0][32][3]: one 384-B row per
// non-zero), results are staged in shared memory and written frame by frame as full sectors.
#include "internal.h"

namespace alsub {

// owner(i) = min control face over the level-L faces g around i; ctrl(g) = control face of g
//   CC   : g descends from level-1 face g >> 2(L-1) = control slot h, face slot_face[h]
//   Loop : g >> 2L
__global__ void k_rm_owner(const int32_t *__restrict__ face_vtx, int32_t FL, int order, int shift,
                           const int32_t *__restrict__ slot_face, int32_t *__restrict__ owner) {
    ALSUB_GRID_WAIT();
    const int32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= FL) return;
    const int32_t a = g >> shift;
    const int32_t f = slot_face ? __ldg(slot_face + a) : a;
    for (int t = 0; t < order; ++t) atomicMin(owner + __ldg(face_vtx + (int64_t)order * g + t), f);
}

// pass 1 (fill = false): row lengths; pass 2 (fill = true): (col, weight) entries.  Unowned rows
// (isolated control vertices, i < V0) are the identity.
__global__ void k_rm_assemble(int32_t VL, const int32_t *__restrict__ owner, const int32_t *__restrict__ sup_off,
                              const int32_t *__restrict__ sup, const int32_t *__restrict__ colour,
                              const float *__restrict__ probe, int64_t probe_stride, bool fill,
                              int32_t *__restrict__ row_len, const int32_t *__restrict__ row_off,
                              int2 *__restrict__ ent) {
    ALSUB_GRID_WAIT();
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= VL) return;
    const int32_t f = owner[i];
    if (f == INT32_MAX) {
        if (fill) ent[row_off[i]] = make_int2(i, __float_as_int(1.0f));
        else row_len[i] = 1;
        return;
    }
    int32_t n = 0, o = fill ? row_off[i] : 0;
    for (int32_t k = __ldg(sup_off + f); k < __ldg(sup_off + f + 1); ++k) {
        const int32_t j = __ldg(sup + k), c = __ldg(colour + j);
        const float w = __ldg(probe + (c / 3) * probe_stride + 3 * (int64_t)i + (c % 3));
        if (w == 0.0f) continue;
        if (fill) ent[o + n] = make_int2(j, __float_as_int(w));
        ++n;
    }
    if (!fill) row_len[i] = n;
}

// probe frames: channel c of frame p = indicator of colour 3p + c
__global__ void k_rm_probes(int32_t V0, const int32_t *__restrict__ colour, int32_t nprobe, float *__restrict__ out) {
    ALSUB_GRID_WAIT();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)nprobe * V0 * 3) return;
    const int64_t p = t / (3 * (int64_t)V0), r = t - p * 3 * V0, v = r / 3;
    const int c = (int)(r - 3 * v);
    out[t] = colour[v] == 3 * p + c ? 1.0f : 0.0f;
}

// [nb][V0][3] frame-major -> [V0][32][3] frame-interleaved (lanes >= nb repeat frame nb - 1)
__global__ void k_rm_interleave(const float *__restrict__ in, int32_t V0, int32_t nb, float *__restrict__ out) {
    ALSUB_GRID_WAIT();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)V0 * kRmLanes * 3) return;
    const int64_t v = t / (kRmLanes * 3);
    const int r = (int)(t - v * kRmLanes * 3), f = r / 3, c = r - 3 * f;
    const int ff = f < nb ? f : nb - 1;
    out[t] = in[((int64_t)ff * V0 + v) * 3 + c];
}

// P_L = R P_0: a row of P_0 for the batch is 96 contiguous floats (32 frames x 3), so each
// non-zero is a 96-float axpy: lanes 0..23 own one float4 of it (one 16-B load per lane, the
// whole 384-B row in 3 cache lines), lanes 24..31 idle.  A warp owns 8 consecutive rows; results
// are staged in shared memory and written frame by frame (8 rows x 12 B = 3 full sectors).
constexpr int kRmWarps = 8, kRmRows = 8;
__global__ void __launch_bounds__(32 * kRmWarps) k_rm_spmm(int32_t VL, const int32_t *__restrict__ row_off,
                                                         const int2 *__restrict__ ent,
                                                         const float4 *__restrict__ P0i, int32_t nb,
                                                         float *__restrict__ out) {
    ALSUB_GRID_WAIT();
    // rows padded to 25 float4 so the per-frame read-back (row stride 100 floats) is conflict-free
    __shared__ float4 s_out[kRmWarps][kRmRows][kRmLanes * 3 / 4 + 1];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const bool act = lane < kRmLanes * 3 / 4;
    const int q = act ? lane : 0;
    // each block walks one contiguous range of tiles: consecutive output vertices are spatial
    // neighbours within a class segment, so the block's control rows stay in L1
    const int64_t ntile = ((int64_t)VL + kRmRows - 1) / kRmRows;
    const int64_t per = (ntile + gridDim.x - 1) / gridDim.x;
    const int64_t t_end = min(ntile, per * (blockIdx.x + 1));
    for (int64_t tile = per * blockIdx.x + w; tile < t_end; tile += kRmWarps) {
        const int32_t r0 = (int32_t)(tile * kRmRows);
        const int32_t nr = min(kRmRows, VL - r0);
        for (int r = 0; r < nr; ++r) {
            const int32_t a = __ldg(row_off + r0 + r), b = __ldg(row_off + r0 + r + 1);
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            int32_t k = a;
            for (; k + 4 <= b; k += 4) {
                int2 e[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) e[u] = __ldg(ent + k + u);
                float4 p[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) p[u] = __ldg(P0i + (int64_t)e[u].x * (kRmLanes * 3 / 4) + q);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float wt = __int_as_float(e[u].y);
                    acc.x = fmaf(wt, p[u].x, acc.x);
                    acc.y = fmaf(wt, p[u].y, acc.y);
                    acc.z = fmaf(wt, p[u].z, acc.z);
                    acc.w = fmaf(wt, p[u].w, acc.w);
                }
            }
            for (; k < b; ++k) {
                const int2 e = __ldg(ent + k);
                const float4 p = __ldg(P0i + (int64_t)e.x * (kRmLanes * 3 / 4) + q);
                const float wt = __int_as_float(e.y);
                acc.x = fmaf(wt, p.x, acc.x);
                acc.y = fmaf(wt, p.y, acc.y);
                acc.z = fmaf(wt, p.z, acc.z);
                acc.w = fmaf(wt, p.w, acc.w);
            }
            if (act) s_out[w][r][lane] = acc;
        }
        __syncwarp();
        // frame f: rows r0 .. r0+nr-1 are 3 nr contiguous floats of out[f]
        if (lane < 3 * nr) {
            const int r = lane / 3, c = lane - 3 * r;
            const float *src = reinterpret_cast<const float *>(s_out[w][r]);
            for (int f = 0; f < nb; ++f) out[((int64_t)f * VL + r0) * 3 + lane] = src[3 * f + c];
        }
        __syncwarp();
    }
}

void rm_owner(const int32_t *face_vtx, int32_t FL, int order, int shift, const int32_t *slot_face, int32_t *owner,
              cudaStream_t s, Launches &L) {
    if (FL > 0) launch(L, "rm_owner", k_rm_owner, dim3(grid_for(FL)), dim3(kThreads), 0, s, face_vtx, FL, order, shift, slot_face, owner);
}
void rm_probes(int32_t V0, const int32_t *colour, int32_t nprobe, float *out, cudaStream_t s, Launches &L) {
    const int64_t n = (int64_t)nprobe * V0 * 3;
    if (n > 0) launch(L, "rm_probes", k_rm_probes, dim3(grid_for(n)), dim3(kThreads), 0, s, V0, colour, nprobe, out);
}
void rm_assemble(int32_t VL, const int32_t *owner, const int32_t *sup_off, const int32_t *sup, const int32_t *colour,
                 const float *probe, int64_t probe_stride, bool fill, int32_t *row_len, const int32_t *row_off,
                 int2 *ent, cudaStream_t s, Launches &L) {
    if (VL > 0) launch(L, "rm_assemble", k_rm_assemble, dim3(grid_for(VL)), dim3(kThreads), 0, s, VL, owner, sup_off, sup, colour,
                       probe, probe_stride, fill, row_len, row_off, ent);
}
void rm_interleave(const float *in, int32_t V0, int32_t nb, float *out, cudaStream_t s, Launches &L) {
    const int64_t n = (int64_t)V0 * kRmLanes * 3;
    if (n > 0) launch(L, "rm_interleave", k_rm_interleave, dim3(grid_for(n)), dim3(kThreads), 0, s, in, V0, nb, out);
}
void rm_spmm(int32_t VL, const int32_t *row_off, const int2 *ent, const float *P0i, int32_t nb, float *out,
             cudaStream_t s, Launches &L) {
    if (VL <= 0) return;
    const int64_t ntile = ((int64_t)VL + kRmRows - 1) / kRmRows;
    // occupancy beats L1 capacity here: a smaller shared-memory carve-out (25-50 %) was measured
    // 1.3-1.8x slower (profiles/r01_rmatrix.json)
    const unsigned grid = (unsigned)std::min<int64_t>((ntile + kRmWarps - 1) / kRmWarps, 148 * 8);
    launch(L, "rm_spmm", k_rm_spmm, dim3(grid), dim3(32 * kRmWarps), 0, s, VL, row_off, ent,
           reinterpret_cast<const float4 *>(P0i), nb, out);
}

}  // namespace alsub
