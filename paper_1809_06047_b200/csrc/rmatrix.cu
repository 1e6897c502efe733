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
// Evaluation: P_L = R P_0 for batches of 32 frames, in a blocked form of R (below): the
// rows of one owner face share its support, so R restricted to them is a small dense block
// W_c [|S_c|][rows_c] -- a warp stages the batch's control positions of S_c in shared memory once
// and every row is a dense |S_c|-term dot product per frame with its weights in registers.
#include <algorithm>

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
                              int2 *__restrict__ ent, int64_t *nnz64) {
    ALSUB_GRID_WAIT();
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    int32_t n = 0;
    if (i < VL) {
        const int32_t f = owner[i];
        if (f == INT32_MAX) {
            if (fill) ent[row_off[i]] = make_int2(i, __float_as_int(1.0f));
            n = 1;
        } else {
            const int32_t o = fill ? row_off[i] : 0;
            for (int32_t k = __ldg(sup_off + f); k < __ldg(sup_off + f + 1); ++k) {
                const int32_t j = __ldg(sup + k), c = __ldg(colour + j);
                const float w = __ldg(probe + (c / 3) * probe_stride + 3 * (int64_t)i + (c % 3));
                if (w == 0.0f) continue;
                if (fill) ent[o + n] = make_int2(j, __float_as_int(w));
                ++n;
            }
        }
        if (!fill) row_len[i] = n;
    }
    if (!fill) {  // the total in 64 bits (the int32 row offsets are only valid if it fits)
        unsigned long long t = (unsigned long long)n;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if ((threadIdx.x & 31) == 0 && t) atomicAdd(reinterpret_cast<unsigned long long *>(nnz64), t);
    }
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

// ------------------------------------------------------------------------------------------
// Blocked R.  Chunk c = owner face c (c < F0), or an isolated control vertex (identity row).
//   row_off [C+1]   rows of chunk c = rows[row_off[c] .. row_off[c+1]), ascending row ids
//   sup_off [C+1]   support S_c = sup[sup_off[c] ..), ascending control vertex ids
//   w_off   [C+1]   W_c at W + w_off[c]: [|S_c|][R64_c] floats, R64_c = rows_c rounded up to 64,
//                   W_c[k][r] = R[rows[row_off[c] + r], S_c[k]] (zero padded)
// ------------------------------------------------------------------------------------------
// chunk of row i: its owner face, or (unowned rows = isolated control vertices, i < V0) the chunk
// iso_chunk[i] the host gave that vertex
__global__ void k_rb_hist(int32_t VL, const int32_t *__restrict__ owner, const int32_t *__restrict__ iso_chunk,
                          int32_t *__restrict__ chunk, int32_t *__restrict__ cnt) {
    ALSUB_GRID_WAIT();
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= VL) return;
    const int32_t o = owner[i];
    const int32_t c = o == INT32_MAX ? iso_chunk[i] : o;
    chunk[i] = c;
    atomicAdd(cnt + c, 1);
}

__global__ void k_rb_scatter(int32_t VL, const int32_t *__restrict__ chunk, const int32_t *__restrict__ row_off,
                             int32_t *__restrict__ cur, int32_t *__restrict__ rows) {
    ALSUB_GRID_WAIT();
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= VL) return;
    const int32_t c = chunk[i];
    rows[row_off[c] + atomicAdd(cur + c, 1)] = i;
}

// rows of every chunk sorted ascending (block per chunk, shared-memory bitonic up to kRbSortCap
// rows; longer chunks -- very high-order control faces -- by one thread), then pos[row] = its index
// in the chunk and the chunk's W length |S_c| x R64_c
constexpr int kRbSortCap = 4096;
__global__ void __launch_bounds__(256) k_rb_sort(int32_t C, const int32_t *__restrict__ row_off,
                                               const int32_t *__restrict__ sup_off, int32_t *__restrict__ rows,
                                               int32_t *__restrict__ pos, int64_t *__restrict__ wlen) {
    ALSUB_GRID_WAIT();
    __shared__ int32_t sk[kRbSortCap];
    for (int32_t c = blockIdx.x; c < C; c += gridDim.x) {
        const int32_t r0 = row_off[c], n = row_off[c + 1] - r0;
        if (threadIdx.x == 0)
            wlen[c] = (int64_t)(sup_off[c + 1] - sup_off[c]) * (int64_t)((n + 63) & ~63);
        if (n <= 1) {
            if (n == 1 && threadIdx.x == 0) pos[rows[r0]] = 0;
            continue;
        }
        if (n <= kRbSortCap) {
            int32_t P = 1;
            while (P < n) P <<= 1;
            for (int32_t i = threadIdx.x; i < P; i += blockDim.x) sk[i] = i < n ? rows[r0 + i] : INT32_MAX;
            __syncthreads();
            for (int32_t k = 2; k <= P; k <<= 1)
                for (int32_t jj = k >> 1; jj > 0; jj >>= 1) {
                    for (int32_t i = threadIdx.x; i < P; i += blockDim.x) {
                        const int32_t l = i ^ jj;
                        if (l > i) {
                            const int32_t x = sk[i], y = sk[l];
                            if ((x > y) == ((i & k) == 0)) { sk[i] = y; sk[l] = x; }
                        }
                    }
                    __syncthreads();
                }
            for (int32_t i = threadIdx.x; i < n; i += blockDim.x) {
                rows[r0 + i] = sk[i];
                pos[sk[i]] = i;
            }
            __syncthreads();
        } else if (threadIdx.x == 0) {
            int32_t *r = rows + r0;
            for (int32_t a = 1; a < n; ++a) {
                const int32_t x = r[a];
                int32_t b = a - 1;
                while (b >= 0 && r[b] > x) { r[b + 1] = r[b]; --b; }
                r[b + 1] = x;
            }
            for (int32_t a = 0; a < n; ++a) pos[r[a]] = a;
        }
    }
}

// exclusive int64 scan of wlen [C] -> w_off [C+1] by one block (build time only)
__global__ void __launch_bounds__(1024) k_rb_scan64(int32_t C, const int64_t *__restrict__ wlen, int64_t *__restrict__ w_off) {
    ALSUB_GRID_WAIT();
    __shared__ int64_t s_part[1024];
    const int32_t per = (C + blockDim.x - 1) / blockDim.x;
    const int32_t lo = min(C, (int32_t)threadIdx.x * per), hi = min(C, lo + per);
    int64_t acc = 0;
    for (int32_t c = lo; c < hi; ++c) acc += wlen[c];
    s_part[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int k = 0; k < (int)blockDim.x; ++k) {
            const int64_t v = s_part[k];
            s_part[k] = t;
            t += v;
        }
        w_off[C] = t;
    }
    __syncthreads();
    acc = s_part[threadIdx.x];
    for (int32_t c = lo; c < hi; ++c) {
        w_off[c] = acc;
        acc += wlen[c];
    }
}

// W_c[k][pos(i)] = probe value of colour(S_c[k]) at row i (the only support vertex of its colour)
__global__ void k_rb_fill(int32_t VL, const int32_t *__restrict__ chunk, const int32_t *__restrict__ pos,
                          const int32_t *__restrict__ row_off, const int32_t *__restrict__ sup_off,
                          const int32_t *__restrict__ sup, const int64_t *__restrict__ w_off,
                          const int32_t *__restrict__ colour, const float *__restrict__ probe, int64_t probe_stride,
                          float *__restrict__ W) {
    ALSUB_GRID_WAIT();
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= VL) return;
    const int32_t c = chunk[i], r = pos[i];
    const int32_t n = row_off[c + 1] - row_off[c];
    const int64_t R64 = (n + 63) & ~63;
    float *Wc = W + w_off[c] + r;
    for (int32_t k = sup_off[c]; k < sup_off[c + 1]; ++k) {
        const int32_t cl = __ldg(colour + __ldg(sup + k));
        Wc[(k - sup_off[c]) * R64] = __ldg(probe + (cl / 3) * probe_stride + 3 * (int64_t)i + (cl % 3));
    }
}

// one batch of nb <= 32 frames [nb][V0][3] -> XT [V0][3][32] (frames innermost, zero padded)
__global__ void k_rb_xt(const float *__restrict__ in, int32_t V0, int32_t nb, float *__restrict__ XT,
                        int32_t *__restrict__ next_chunk) {
    ALSUB_GRID_WAIT();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t == 0) *next_chunk = 0;
    if (t >= (int64_t)V0 * 3 * kRmLanes) return;
    const int f = (int)(t % kRmLanes);
    const int64_t vc = t / kRmLanes;  // 3 v + c
    XT[t] = f < nb ? __ldg(in + (int64_t)f * V0 * 3 + vc) : 0.0f;
}

// P_L = R P_0 over the chunks: one CTA per chunk (taken in order from a counter), warp w on its row
// groups w, w + 4, ... (64 rows: lane = rows r and r + 32, their |S_c| weights in registers).  The
// batch's control positions of S_c are staged once per chunk in shared memory ([k][coord][32
// frames]) and read as warp-wide broadcasts, 4 frames per float4: per support vertex 3 broadcast
// loads feed 24 FMAs.  With the whole chunk in flight at once and neighbouring chunks on
// neighbouring CTAs, the output runs that share a boundary sector are written within a few
// microseconds of each other and merge in L2 (one warp per chunk, processed over ~100 us, left
// those sectors to be evicted half written: DRAM read-modify-write, +40 % traffic).  Chunks with
// |S_c| > kRbTK run the same product over kRbTK-wide support tiles (positions restaged per tile
// and frame group in the warp's quarter of the buffer, weights from L1).
constexpr int kRbWarps = 4, kRbTK = 24;
constexpr int kRbXf4 = 3 * kRmLanes / 4;  // float4 per support vertex in XT / shared memory (24)

// results of one row group (64 rows) for 4 frames -> the chunk's output rows.  The lanes' values
// (row r and r + 32, 4 frames x 3 coords) go through shared memory so that each store instruction
// writes 32 consecutive floats of one frame (float t of the group = coord t % 3 of its row t / 3):
// contiguous row runs become full 128-B lines instead of 12-B-strided partial sectors.
// the frame's summary record (alsub_frame_summary) folded in from the lane's two rows: float
// index 3 row + c, bbox over the ordered-int images, checksum sum bits (2 idx + 1) mod 2^64; warp
// reductions by redux.sync (the 64-bit sum as three exact 32-bit partial sums), one lane's shared
// atomics into the CTA's record
// row r's checksum term sum_c bits(x_c) (6 r + 2 c + 1) = (6 r + 1)(b0 + b1 + b2) + 2 b1 + 4 b2
// (mod 2^64: the distributive law holds in the ring, so the value is the same as term by term)
ALSUB_D unsigned long long rb_row_sum(int32_t r, const float (&v)[3]) {
    const unsigned long long b0 = (uint32_t)__float_as_int(v[0]), b1 = (uint32_t)__float_as_int(v[1]),
                             b2 = (uint32_t)__float_as_int(v[2]);
    return (6ull * (unsigned long long)r + 1ull) * (b0 + b1 + b2) + 2ull * b1 + 4ull * b2;
}
// FULL: both rows of every lane exist (all but a chunk's last row group): no per-row predicates
template <bool FULL>
ALSUB_D void rb_fold(SummaryRec &acc, int f, int32_t ra, int32_t rb, const float (&a)[3], const float (&b)[3]) {
    int32_t lo[3], hi[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int32_t oa = f2ord(a[c]), ob = f2ord(b[c]);
        if constexpr (FULL) {
            lo[c] = min(oa, ob);
            hi[c] = max(oa, ob);
        } else {
            lo[c] = min(ra >= 0 ? oa : INT32_MAX, rb >= 0 ? ob : INT32_MAX);
            hi[c] = max(ra >= 0 ? oa : INT32_MIN, rb >= 0 ? ob : INT32_MIN);
        }
    }
    unsigned long long sum;
    if constexpr (FULL) sum = rb_row_sum(ra, a) + rb_row_sum(rb, b);
    else sum = (ra >= 0 ? rb_row_sum(ra, a) : 0ull) + (rb >= 0 ? rb_row_sum(rb, b) : 0ull);
    const unsigned m = 0xffffffffu;
    const uint32_t s0 = __reduce_add_sync(m, (uint32_t)(sum & 0xffffu));
    const uint32_t s1 = __reduce_add_sync(m, (uint32_t)((sum >> 16) & 0xffffu));
    const uint32_t s2 = __reduce_add_sync(m, (uint32_t)(sum >> 32));
    int32_t l[3], h[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        l[c] = __reduce_min_sync(m, lo[c]);
        h[c] = __reduce_max_sync(m, hi[c]);
    }
    // frame f's running record lives in lane f's registers (flushed once per warp at the end of
    // the kernel) instead of eight shared-memory atomics per frame and row group
    if ((threadIdx.x & 31) == f) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            acc.lo[c] = min(acc.lo[c], l[c]);
            acc.hi[c] = max(acc.hi[c], h[c]);
        }
        acc.sum += (unsigned long long)s0 + ((unsigned long long)s1 << 16) + ((unsigned long long)s2 << 32);
    }
}

ALSUB_D void rb_store(float *so, const int32_t (&rid)[6], float *out, int64_t VL, int f0, int nb, int lane,
                      const float (&a)[4][3], const float (&b)[4][3], SummaryRec *acc, int32_t rowa, int32_t rowb) {
    if (acc) {
        if (__all_sync(0xffffffffu, rowb >= 0)) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (f0 + u < nb) rb_fold<true>(*acc, f0 + u, rowa, rowb, a[u], b[u]);
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (f0 + u < nb) rb_fold<false>(*acc, f0 + u, rowa, rowb, a[u], b[u]);
        }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            so[u * 192 + 3 * lane + c] = a[u][c];
            so[u * 192 + 96 + 3 * lane + c] = b[u][c];
        }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        if (f0 + u >= nb) break;
        float *o = out + (int64_t)(f0 + u) * VL * 3;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            const int t = lane + 32 * i;
            if (rid[i] >= 0) o[3 * (int64_t)rid[i] + (t % 3)] = so[u * 192 + t];
        }
    }
    __syncwarp();
}

ALSUB_D void rb_fma(float (&a)[4][3], float w, const float4 (&x)[3]) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        a[0][c] = fmaf(w, x[c].x, a[0][c]);
        a[1][c] = fmaf(w, x[c].y, a[1][c]);
        a[2][c] = fmaf(w, x[c].z, a[2][c]);
        a[3][c] = fmaf(w, x[c].w, a[3][c]);
    }
}

__global__ void __launch_bounds__(32 * kRbWarps) k_rb_eval(int32_t C, int32_t *__restrict__ next_chunk,
                                                         const int32_t *__restrict__ row_off,
                                                         const int32_t *__restrict__ sup_off,
                                                         const int64_t *__restrict__ w_off,
                                                         const int32_t *__restrict__ rows,
                                                         const int32_t *__restrict__ sup, const float *__restrict__ W,
                                                         const float4 *__restrict__ XT, int32_t nb, int64_t VL,
                                                         float *__restrict__ out, SummaryRec *__restrict__ rec) {
    ALSUB_GRID_WAIT();
    extern __shared__ float4 s_dyn[];  // kRbTK x 24 float4 of positions (the CTA's), then per warp 4 x 192 floats
    __shared__ int32_t s_c;
    // per-frame summary records of this CTA's rows (rec != nullptr), flushed to rec at the end
    __shared__ SummaryRec s_rec[kRmLanes];
    SummaryRec racc;  // lane f: the running record of frame f over this warp's rows
    for (int c = 0; c < 3; ++c) {
        racc.lo[c] = INT32_MAX;
        racc.hi[c] = INT32_MIN;
    }
    racc.sum = 0ull;
    SummaryRec *srec = rec ? &racc : nullptr;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (rec && threadIdx.x < kRmLanes) {
        SummaryRec r;
        for (int c = 0; c < 3; ++c) {
            r.lo[c] = INT32_MAX;
            r.hi[c] = INT32_MIN;
        }
        r.sum = 0ull;
        s_rec[threadIdx.x] = r;
    }
    float4 *sx = s_dyn;
    float *so = reinterpret_cast<float *>(s_dyn + kRbTK * kRbXf4) + w * 4 * 192;
    for (;;) {
        if (threadIdx.x == 0) s_c = atomicAdd(next_chunk, 1);
        __syncthreads();
        const int32_t c = s_c;
        if (c >= C) break;
        const int32_t r0 = __ldg(row_off + c), nr = __ldg(row_off + c + 1) - r0;
        const int32_t s0 = __ldg(sup_off + c), S = __ldg(sup_off + c + 1) - s0;
        const int32_t R64 = (nr + 63) & ~63;
        const float *Wc = W + __ldg(w_off + c);
        if (S <= kRbTK) {
            for (int32_t q = threadIdx.x; q < S * kRbXf4; q += blockDim.x) {
                const int32_t k = q / kRbXf4, u = q - k * kRbXf4;
                sx[q] = __ldg(XT + (int64_t)__ldg(sup + s0 + k) * kRbXf4 + u);
            }
            __syncthreads();
            for (int32_t g = 64 * w; g < nr; g += 64 * kRbWarps) {
                const int32_t ra = g + lane, rb = ra + 32;
                float wa[kRbTK], wb[kRbTK];
#pragma unroll
                for (int k = 0; k < kRbTK; ++k) {
                    wa[k] = k < S ? __ldg(Wc + (int64_t)k * R64 + ra) : 0.0f;
                    wb[k] = k < S ? __ldg(Wc + (int64_t)k * R64 + rb) : 0.0f;
                }
                int32_t rid[6];
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    const int32_t r = g + (lane + 32 * i) / 3;
                    rid[i] = r < nr ? __ldg(rows + r0 + r) : -1;
                }
                const int32_t rowa = ra < nr ? __ldg(rows + r0 + ra) : -1, rowb = rb < nr ? __ldg(rows + r0 + rb) : -1;
                for (int f0 = 0; f0 < nb; f0 += 4) {
                    float a[4][3] = {}, b[4][3] = {};
#pragma unroll
                    for (int k = 0; k < kRbTK; ++k) {
                        if (k >= S) break;
                        float4 x[3];
#pragma unroll
                        for (int cc = 0; cc < 3; ++cc) x[cc] = sx[k * kRbXf4 + cc * (kRmLanes / 4) + (f0 >> 2)];
                        rb_fma(a, wa[k], x);
                        rb_fma(b, wb[k], x);
                    }
                    rb_store(so, rid, out, VL, f0, nb, lane, a, b, srec, rowa, rowb);
                }
            }
        } else {
            // wide support: kRbTK-wide tiles, positions of one frame group per tile, in this warp's
            // quarter of the position buffer
            float4 *sw = sx + w * (kRbTK * kRbXf4 / kRbWarps);
            for (int32_t g = 64 * w; g < nr; g += 64 * kRbWarps) {
                const int32_t ra = g + lane, rb = ra + 32;
                int32_t rid[6];
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    const int32_t r = g + (lane + 32 * i) / 3;
                    rid[i] = r < nr ? __ldg(rows + r0 + r) : -1;
                }
                const int32_t rowa = ra < nr ? __ldg(rows + r0 + ra) : -1, rowb = rb < nr ? __ldg(rows + r0 + rb) : -1;
                for (int f0 = 0; f0 < nb; f0 += 4) {
                    float a[4][3] = {}, b[4][3] = {};
                    for (int32_t t0 = 0; t0 < S; t0 += kRbTK) {
                        const int32_t St = min(kRbTK, S - t0);
                        __syncwarp();
                        for (int32_t q = lane; q < 3 * St; q += 32) {
                            const int32_t k = q / 3, cc = q - 3 * k;
                            sw[q] = __ldg(XT + (int64_t)__ldg(sup + s0 + t0 + k) * kRbXf4 + cc * (kRmLanes / 4) + (f0 >> 2));
                        }
                        __syncwarp();
                        for (int32_t k = 0; k < St; ++k) {
                            const float4 x[3] = {sw[3 * k], sw[3 * k + 1], sw[3 * k + 2]};
                            rb_fma(a, __ldg(Wc + (int64_t)(t0 + k) * R64 + ra), x);
                            rb_fma(b, __ldg(Wc + (int64_t)(t0 + k) * R64 + rb), x);
                        }
                    }
                    rb_store(so, rid, out, VL, f0, nb, lane, a, b, srec, rowa, rowb);
                }
            }
        }
        __syncthreads();  // the positions and s_c are reused by the next chunk
    }
    if (rec && lane < nb) {  // the warps' records into the CTA's (the loop ended with a barrier)
        SummaryRec &r = s_rec[lane];
        for (int c = 0; c < 3; ++c) {
            atomicMin(&r.lo[c], racc.lo[c]);
            atomicMax(&r.hi[c], racc.hi[c]);
        }
        atomicAdd(&r.sum, racc.sum);
    }
    if (rec) __syncthreads();
    if (rec && threadIdx.x < nb) {
        const SummaryRec &r = s_rec[threadIdx.x];
        SummaryRec &g = rec[threadIdx.x];
        for (int c = 0; c < 3; ++c) {
            atomicMin(&g.lo[c], r.lo[c]);
            atomicMax(&g.hi[c], r.hi[c]);
        }
        atomicAdd(&g.sum, r.sum);
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
                 int2 *ent, int64_t *nnz64, cudaStream_t s, Launches &L) {
    if (VL > 0) launch(L, "rm_assemble", k_rm_assemble, dim3(grid_for(VL)), dim3(kThreads), 0, s, VL, owner, sup_off, sup, colour,
                       probe, probe_stride, fill, row_len, row_off, ent, nnz64);
}
void rb_hist(int32_t VL, const int32_t *owner, const int32_t *iso_chunk, int32_t *chunk, int32_t *cnt, cudaStream_t s,
             Launches &L) {
    if (VL > 0) launch(L, "rb_hist", k_rb_hist, dim3(grid_for(VL)), dim3(kThreads), 0, s, VL, owner, iso_chunk, chunk, cnt);
}
void rb_scatter(int32_t VL, const int32_t *chunk, const int32_t *row_off, int32_t *cur, int32_t *rows, cudaStream_t s,
                Launches &L) {
    if (VL > 0) launch(L, "rb_scatter", k_rb_scatter, dim3(grid_for(VL)), dim3(kThreads), 0, s, VL, chunk, row_off, cur, rows);
}
void rb_sort(int32_t C, const int32_t *row_off, const int32_t *sup_off, int32_t *rows, int32_t *pos, int64_t *wlen,
             int64_t *w_off, cudaStream_t s, Launches &L) {
    if (C <= 0) return;
    launch(L, "rb_sort", k_rb_sort, dim3((unsigned)std::min<int32_t>(C, 148 * 8)), dim3(256), 0, s, C, row_off, sup_off,
           rows, pos, wlen);
    launch(L, "rb_scan64", k_rb_scan64, dim3(1), dim3(1024), 0, s, C, (const int64_t *)wlen, w_off);
}
void rb_fill(int32_t VL, const int32_t *chunk, const int32_t *pos, const int32_t *row_off, const int32_t *sup_off,
             const int32_t *sup, const int64_t *w_off, const int32_t *colour, const float *probe, int64_t probe_stride,
             float *W, cudaStream_t s, Launches &L) {
    if (VL > 0) launch(L, "rb_fill", k_rb_fill, dim3(grid_for(VL)), dim3(kThreads), 0, s, VL, chunk, pos, row_off, sup_off,
                       sup, w_off, colour, probe, probe_stride, W);
}
void rb_eval(int32_t C, const int32_t *row_off, const int32_t *sup_off, const int64_t *w_off, const int32_t *rows,
             const int32_t *sup, const float *W, const float *in, int32_t V0, int32_t nb, float *XT, int64_t VL,
             float *out, SummaryRec *rec, cudaStream_t s, Launches &L) {
    if (nb <= 0) return;
    const int64_t n = (int64_t)V0 * 3 * kRmLanes;
    int32_t *next_chunk = reinterpret_cast<int32_t *>(XT + n);  // one int after the batch
    launch(L, "rb_xt", k_rb_xt, dim3(grid_for(n)), dim3(kThreads), 0, s, in, V0, nb, XT, next_chunk);
    if (C <= 0) return;
    const size_t smem = (size_t)kRbTK * kRbXf4 * 16 + (size_t)kRbWarps * 4 * 192 * 4;
    static bool attr = [smem] {
        return cudaFuncSetAttribute(k_rb_eval, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess;
    }();
    (void)attr;
    int max_blocks = 4;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_blocks, k_rb_eval, 32 * kRbWarps, smem);
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(C, kRbWarps), 148 * std::max(max_blocks, 1));
    launch(L, "rb_eval", k_rb_eval, dim3(grid), dim3(32 * kRbWarps), smem, s, C, next_chunk, row_off, sup_off, w_off, rows, sup, W,
           reinterpret_cast<const float4 *>(XT), nb, VL, out, rec);
}

}  // namespace alsub
