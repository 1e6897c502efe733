// build0.cu -- level-0 topology from arbitrary face lists.
//
// a1  mesh matrix M (CSC: face_off / face_vtx) + validation
// a2  M^T by a counting sort of the slots by vertex (histogram = row lengths, scan, scatter, rows
//     sorted by slot); vertex valence n = M 1 (Eq. vo) = row length
// a3  the implicit mapped SpGEMMs E = M M^T {Q_c + Q_c^{c-1}}[lambda] and F = M M^T {Q_c}[gamma]
//      evaluated as in the paper's implicit SpGEMM: every collision of
//     vertex j with its face neighbours next(h) = Q_c and prev(h) = Q_c^{c-1} is visited from j's
//     incident slots; a symbolic pass counts the distinct neighbours i < j (the upper-triangular
//     non-zeros of column j of E), a scan turns the counts into ids -- edge id = rank of (j, i) in
//     column-major order (reading R1) -- and a numeric pass fills face_edge / face_twin
//     (F(i,j) and F(j,i)) and the multiplicity checks (E(i,j) in {1, 2}).
// Then the crease matrix C is attached to edge ids and the special-edge list
// (boundary edges = infinitely sharp creases, reading R6) and special-vertex table are built.
#include <algorithm>

#include "internal.h"

namespace alsub {


// a1 + the input of a2: validation, slot -> face and the row
// lengths of M^T (vertex valences n = M 1, Eq. vo).
__global__ void __launch_bounds__(kThreads) k_b0_prep(const int32_t *__restrict__ face_off,
                                                    const int32_t *__restrict__ face_vtx, int32_t F, int32_t V,
                                                    int32_t *__restrict__ slot_face, int32_t *__restrict__ vtx_cnt,
                                                    int32_t *flags) {
    ALSUB_GRID_WAIT();
    const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= F) return;
    const int32_t o = face_off[r], c = face_off[r + 1] - o;
    if (c < 3) atomicOr(flags, kFlagMesh);
    for (int32_t t = 0; t < c; ++t) {
        const int32_t v = face_vtx[o + t];
        slot_face[o + t] = r;
        if (v < 0 || v >= V) { atomicOr(flags, kFlagMesh); continue; }
        atomicAdd(vtx_cnt + v, 1);
        for (int32_t u = 0; u < t; ++u)
            if (face_vtx[o + u] == v) atomicOr(flags, kFlagMesh);
    }
}

// a2: M^T by a counting sort -- the histogram is the row lengths (prep), their scan the row
// offsets, and every slot is scattered into its vertex's row through a per-row cursor.  The rows
// come out in arbitrary order; k_edge_count sorts each one by slot (ascending, as a stable sort by
// vertex would leave them) before anything reads them.
__global__ void __launch_bounds__(kThreads) k_b0_scatter(const int32_t *__restrict__ face_vtx, int32_t S, int32_t V,
                                                       const int32_t *__restrict__ vtx_off,
                                                       int32_t *__restrict__ cur, int32_t *__restrict__ vtx_slot) {
    ALSUB_GRID_WAIT();
    const int32_t h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= S) return;
    const int32_t v = __ldg(face_vtx + h);
    if (v < 0 || v >= V) return;
    vtx_slot[vtx_off[v] + atomicAdd(cur + v, 1)] = h;
}

// Warp-per-vertex collision processing: lane q < 2n holds candidate q of vertex j (slot q/2,
// neighbour next (q even) or prev (q odd)); duplicates are found with __match_any_sync and the
// rank of a distinct neighbour among the distinct neighbours < j with a ballot per lane.
// Vertices with more than 16 incident faces are listed for k_long_rows (block per row).
struct WarpCand {
    int32_t x;     // neighbour vertex (INT32_MAX = none)
    int32_t slot;  // the slot of the directed edge (j -> x for next, x -> j for prev)
    bool first;    // first occurrence of x among the candidates
    unsigned peers;
};

template <int ORDER, bool NC = true>
ALSUB_D WarpCand warp_cand(const int32_t *face_vtx, const int32_t *vtx_slot, Topo<ORDER> tp, int32_t o0, int32_t n, int lane) {
    WarpCand c{INT32_MAX, -1, false, 0u};
    if (lane < 2 * n) {
        const int32_t h = NC ? __ldg(vtx_slot + o0 + (lane >> 1)) : vtx_slot[o0 + (lane >> 1)];
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
template <int ORDER>
__global__ void k_edge_count(const int32_t *__restrict__ face_vtx, const int32_t *__restrict__ vtx_off,
                             const int32_t *vtx_slot, Topo<ORDER> tp, int32_t V, int32_t *__restrict__ cnt,
                             int32_t *__restrict__ long_list, int32_t *long_cnt) {
    ALSUB_GRID_WAIT();
    const int32_t j = (int32_t)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (j >= V) return;
    const int32_t o0 = vtx_off[j], n = vtx_off[j + 1] - o0;
    int32_t *row = const_cast<int32_t *>(vtx_slot) + o0;
    if (n <= kLongRow) {
        // sort the row by slot: lane q moves its slot to its rank (slots are distinct)
        const int32_t sq = lane < n ? row[lane] : INT32_MAX;
        int32_t rank = 0;
        for (int p = 0; p < n; ++p) rank += __shfl_sync(0xffffffffu, sq, p) < sq;  // (n warp-uniform)
        __syncwarp();
        if (lane < n) row[rank] = sq;
        __syncwarp();
        const WarpCand c = warp_cand<ORDER, false>(face_vtx, vtx_slot, tp, o0, n, lane);
        // unsigned: an out-of-range (negative) id of an invalid mesh is never an edge
        const unsigned b = __ballot_sync(0xffffffffu, c.first && (uint32_t)c.x < (uint32_t)j);
        if (lane == 0) cnt[j] = __popc(b);
        return;
    }
    // long rows (poles, fan caps): one block per row in k_long_rows (sorted in shared memory)
    if (lane == 0) long_list[atomicAdd(long_cnt, 1)] = j;
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
template <int ORDER>
__global__ void k_edge_fill(const int32_t *__restrict__ face_vtx, const int32_t *__restrict__ vtx_off,
                            const int32_t *__restrict__ vtx_slot, Topo<ORDER> tp, int32_t V,
                            const int32_t *__restrict__ edge_off, int32_t *__restrict__ face_edge,
                            int32_t *__restrict__ face_twin, int2 *__restrict__ edge_hh,
                            uint32_t *__restrict__ bnd_word, int32_t *__restrict__ vbnd,
                            int32_t *__restrict__ scalars, int32_t *flags, int32_t *__restrict__ slot0) {
    ALSUB_GRID_WAIT();
    const int32_t j = (int32_t)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (j >= V) return;
    const int32_t o0 = vtx_off[j], n = vtx_off[j + 1] - o0;
    if (lane == 0) slot0[j] = n > 0 ? vtx_slot[o0] : -1;
    if (n <= kLongRow) {
        const WarpCand c = warp_cand(face_vtx, vtx_slot, tp, o0, n, lane);
        const bool mine = c.first && (uint32_t)c.x < (uint32_t)j;
        // the rank of each edge this vertex owns among its distinct smaller neighbours: only the
        // owning lanes need one (about half the distinct neighbours), so the loop visits those
        int32_t rank = 0;
        for (unsigned mm = __ballot_sync(0xffffffffu, mine); mm; mm &= mm - 1) {
            const int k = __ffs(mm) - 1;
            const int32_t xk = __shfl_sync(0xffffffffu, c.x, k);
            const unsigned b = __ballot_sync(0xffffffffu, c.first && (uint32_t)c.x < (uint32_t)xk);
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
    // long rows: k_long_rows<..., true>
}

// ------------------------------------------------------------------------------------------
// Long rows of M^T (n > 16 incident slots: poles, fan caps).  One block per listed row: the row
// and its 2n collision candidates (key = neighbour << 32 | candidate index) are sorted with a
// block-wide bitonic network, so equal neighbours are adjacent, the first of each run is the
// first occurrence, a run's length and parity give E(i,j) and the directed slots, and the rank of
// a distinct neighbour is an exclusive count of run starts -- O(n log^2 n) work spread over the
// block instead of the warp path's 32 candidate lanes.  Rows of up to kLongFast / 2 slots sort in
// registers (count pass; the sorted candidates are kept in a global scratch, 4 keys per slot, for
// the fill pass); longer rows run the same steps as a plain bitonic network in that scratch.
// count pass (FILL = false): sort the row in place + number of distinct neighbours i < j;
// fill pass (FILL = true): ids, twins, multiplicity checks, boundary bits (rows already sorted).
// ------------------------------------------------------------------------------------------
constexpr int kLongThreads = 512;
constexpr int kLongFast = 4 * kLongThreads;  // keys sorted in registers (4 per thread)

ALSUB_D int32_t pow2_at_least(int32_t n) {
    int32_t p = 1;
    while (p < n) p <<= 1;
    return p;
}

// ascending bitonic sort of a[0, n), n a power of two, by the whole block (rows > kLongFast / 2)
ALSUB_D void block_bitonic(uint64_t *a, int32_t n) {
    for (int32_t k = 2; k <= n; k <<= 1)
        for (int32_t jj = k >> 1; jj > 0; jj >>= 1) {
            for (int32_t i = threadIdx.x; i < n; i += blockDim.x) {
                const int32_t l = i ^ jj;
                if (l > i) {
                    const uint64_t x = a[i], y = a[l];
                    if ((x > y) == ((i & k) == 0)) { a[i] = y; a[l] = x; }
                }
            }
            __syncthreads();
        }
}

// ascending bitonic sort of kLongFast keys, element 4 tid + r in v[r]: partners inside the thread
// (stride < 4) in registers, inside the warp (< 128) by shuffles, across warps through s_x --
// 10 of the 66 stages touch shared memory
ALSUB_D void block_sort4(uint64_t (&v)[4], uint64_t *s_x) {
    const int tid = threadIdx.x;
    for (int k = 2; k <= kLongFast; k <<= 1) {
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            if (jj >= 128) {
#pragma unroll
                for (int r = 0; r < 4; ++r) s_x[4 * tid + r] = v[r];
                __syncthreads();
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int i = 4 * tid + r;
                    const uint64_t o = s_x[i ^ jj];
                    v[r] = (((i & jj) == 0) == ((i & k) == 0)) ? min(v[r], o) : max(v[r], o);
                }
                __syncthreads();
            } else if (jj >= 4) {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int i = 4 * tid + r;
                    const uint64_t o = __shfl_xor_sync(0xffffffffu, v[r], jj >> 2);
                    v[r] = (((i & jj) == 0) == ((i & k) == 0)) ? min(v[r], o) : max(v[r], o);
                }
            } else {  // strides 2 and 1 inside the thread (constant register indices)
                const bool a01 = ((4 * tid) & k) == 0, a23 = ((4 * tid + 2) & k) == 0;  // differ only for k = 2
                auto cs = [](uint64_t &a, uint64_t &b, bool asc) {
                    const uint64_t lo = min(a, b), hi = max(a, b);
                    a = asc ? lo : hi;
                    b = asc ? hi : lo;
                };
                if (jj == 2) { cs(v[0], v[2], a01); cs(v[1], v[3], a01); }
                else { cs(v[0], v[1], a01); cs(v[2], v[3], a23); }
            }
        }
    }
}

// exclusive block scan of one flag per thread; returns the prefix, *total = the round's sum
ALSUB_D int32_t block_excl_scan(bool flag, int32_t *s_w, int32_t *total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const unsigned b = __ballot_sync(0xffffffffu, flag);
    if (lane == 0) s_w[w] = __popc(b);
    __syncthreads();
    int32_t before = 0, all = 0;
    for (int k = 0; k < nw; ++k) {
        const int32_t c = s_w[k];
        before += k < w ? c : 0;
        all += c;
    }
    __syncthreads();
    *total = all;
    return before + __popc(b & ((1u << lane) - 1u));
}

// candidate key q of row j: even q = next(h) (slot h carries j -> x), odd = prev(h) (x -> j)
template <int ORDER>
ALSUB_D uint64_t cand_key(const int32_t *face_vtx, const int32_t *row, Topo<ORDER> tp, int32_t q, int32_t nq) {
    if (q >= nq) return ~0ull;
    const int32_t h = row[q >> 1];
    const int32_t x = __ldg(face_vtx + ((q & 1) ? tp.prev(h) : tp.next(h)));
    return ((uint64_t)(uint32_t)x << 32) | (uint32_t)q;
}

template <int ORDER, bool FILL>
__global__ void __launch_bounds__(kLongThreads) k_long_rows(const int32_t *__restrict__ face_vtx,
                                                          const int32_t *__restrict__ vtx_off, int32_t *vtx_slot,
                                                          Topo<ORDER> tp, const int32_t *__restrict__ long_list,
                                                          const int32_t *long_cnt, uint64_t *__restrict__ g_keys,
                                                          int32_t *__restrict__ cnt, const int32_t *__restrict__ edge_off,
                                                          int32_t *__restrict__ face_edge, int32_t *__restrict__ face_twin,
                                                          int2 *__restrict__ edge_hh, uint32_t *__restrict__ bnd_word,
                                                          int32_t *__restrict__ vbnd, int32_t *__restrict__ scalars,
                                                          int32_t *flags) {
    ALSUB_GRID_WAIT();
    __shared__ uint64_t s_key[kLongFast];
    __shared__ int32_t s_w[kLongThreads / 32];
    const int32_t nl = *long_cnt;
    const int tid = threadIdx.x;
    for (int32_t idx = blockIdx.x; idx < nl; idx += gridDim.x) {
        const int32_t j = long_list[idx];
        const int32_t o0 = vtx_off[j], n = vtx_off[j + 1] - o0;
        const int32_t nq = 2 * n;
        int32_t *row = vtx_slot + o0;
        uint64_t *gk = g_keys + 4 * (int64_t)o0;  // 4 n keys of room (>= the padded 2 n)
        const bool fast = nq <= kLongFast;
        const int32_t P2 = fast ? kLongFast : pow2_at_least(nq);
        const uint64_t *key = fast ? s_key : gk;
        if (fast) {
            uint64_t v[4];
            if constexpr (!FILL) {  // sort the row by slot, then its candidates; keep them for the fill pass
#pragma unroll
                for (int r = 0; r < 4; ++r) v[r] = 4 * tid + r < n ? (uint64_t)row[4 * tid + r] : ~0ull;
                block_sort4(v, s_key);
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    if (4 * tid + r < n) row[4 * tid + r] = (int32_t)v[r];
                __syncthreads();
#pragma unroll
                for (int r = 0; r < 4; ++r) v[r] = cand_key(face_vtx, row, tp, 4 * tid + r, nq);
                block_sort4(v, s_key);
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    s_key[4 * tid + r] = v[r];
                    if (4 * tid + r < nq) gk[4 * tid + r] = v[r];
                }
            } else {
#pragma unroll
                for (int r = 0; r < 4; ++r) s_key[4 * tid + r] = 4 * tid + r < nq ? gk[4 * tid + r] : ~0ull;
            }
            __syncthreads();
        } else {  // long rows beyond the register sort: the same steps in global memory
            if constexpr (!FILL) {
                const int32_t P1 = pow2_at_least(n);
                for (int32_t i = tid; i < P1; i += blockDim.x) gk[i] = i < n ? (uint64_t)row[i] : ~0ull;
                __syncthreads();
                block_bitonic(gk, P1);
                for (int32_t i = tid; i < n; i += blockDim.x) row[i] = (int32_t)gk[i];
                __syncthreads();
            }
            for (int32_t q = tid; q < P2; q += blockDim.x) gk[q] = cand_key(face_vtx, row, tp, q, nq);
            __syncthreads();
            block_bitonic(gk, P2);
        }
        // run starts with x < j (padding keys have x = 0xffffffff > any j); rank = exclusive count
        int32_t base = 0;
        for (int32_t p0 = 0; p0 < P2; p0 += blockDim.x) {
            const int32_t p = p0 + tid;
            const uint32_t x = p < P2 ? (uint32_t)(key[p] >> 32) : 0xffffffffu;
            const bool start = p < P2 && x < (uint32_t)j && (p == 0 || (uint32_t)(key[p - 1] >> 32) != x);
            int32_t total;
            const int32_t rank = base + block_excl_scan(start, s_w, &total);
            if constexpr (FILL) {
                if (start) {
                    int32_t s_ij = -1, s_ji = -1, m_ij = 0, m_ji = 0;
                    for (int32_t r = p; r < nq && (uint32_t)(key[r] >> 32) == x; ++r) {
                        const int32_t q = (int32_t)(uint32_t)key[r];
                        const int32_t h = row[q >> 1];
                        if (q & 1) { s_ij = tp.prev(h); ++m_ij; }
                        else { s_ji = h; ++m_ji; }
                    }
                    if (m_ij > 1 || m_ji > 1) atomicOr(flags, kFlagNonManifold);
                    emit_edge(edge_off[j] + rank, s_ij, s_ji, (int32_t)x, j, face_edge, face_twin, edge_hh, bnd_word,
                              vbnd, scalars);
                }
            }
            base += total;
        }
        if constexpr (!FILL) {
            if (tid == 0) cnt[j] = base;
        }
        __syncthreads();
    }
}

// a vertex whose interior faces form a closed fan that misses some incident face is non-manifold
// (reading R18); open fans (bowties) are allowed and end up as corners.
template <int ORDER>
__global__ void k_check_fans(const int32_t *__restrict__ face_twin, const int32_t *__restrict__ vtx_off,
                             const int32_t *__restrict__ slot0, Topo<ORDER> tp, int32_t V, int32_t *flags) {
    ALSUB_GRID_WAIT();
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









// ------------------------------------------------------------------------------------------
// Level-0 special lists.  The level-0 special-vertex table is the identity over all V0 vertices
// (sv_vtx[v] = v; non-special vertices get empty lists), so no vertex compaction is needed.
// ------------------------------------------------------------------------------------------
// crease matrix C: pairs -> edge ids and the special flags (boundary = inf crease,
// reading R6); also the popcounts of the boundary words
template <int ORDER>
__global__ void __launch_bounds__(kThreads) k_b0_flags(const int32_t *__restrict__ crease, const float *__restrict__ sigma,
                                                     int32_t K, const int32_t *__restrict__ face_vtx,
                                                     const int32_t *__restrict__ vtx_off,
                                                     const int32_t *__restrict__ vtx_slot,
                                                     const int32_t *__restrict__ face_edge, const int2 *__restrict__ edge_hh,
                                                     Topo<ORDER> tp, int32_t V, int32_t E, const uint32_t *__restrict__ bnd_word,
                                                     int32_t nw, float *__restrict__ edge_sigma,
                                                     int32_t *__restrict__ edge_cidx, int32_t *__restrict__ flag,
                                                     int32_t *__restrict__ wcnt, int32_t *flags, int32_t lenient,
                                                     const int32_t *__restrict__ Edev, int32_t *__restrict__ sv_cnt) {
    ALSUB_GRID_WAIT();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // inside alsub_mesh_create the arrays are sized by an upper bound and E is only on the device
    if (Edev) E = min(E, *Edev);
    // every special edge is flagged exactly once (here if boundary, below if creased), so the
    // special-vertex list lengths (incident special edges) are counted where the flag is set
    if (t < E) {
        const int2 hh = edge_hh[t];
        if (hh.y < 0) {
            atomicOr(flag + t, 1);
            atomicAdd(sv_cnt + face_vtx[hh.x], 1);
            atomicAdd(sv_cnt + face_vtx[tp.next(hh.x)], 1);
        }
    }
    if (t < nw) wcnt[t] = __popc(bnd_word[t]);
    // one warp per crease pair: the lanes test the incident slots of max(a, b) in parallel
    const int64_t k = t >> 5;
    const int lane = threadIdx.x & 31;
    if (k >= K) return;
    const int32_t a = crease[2 * k], b = crease[2 * k + 1];
    const float sg = sigma[k];
    if (a < 0 || a >= V || b < 0 || b >= V || a == b || !(sg >= 0.0f)) {
        if (lane == 0) atomicOr(flags, kFlagCrease);
        return;
    }
    const int32_t j = max(a, b), i = min(a, b);
    const int32_t o0 = vtx_off[j], n = vtx_off[j + 1] - o0;
    int32_t e = -1;
    for (int32_t q0 = 0; q0 < n; q0 += 32) {
        int32_t cand = -1;
        if (q0 + lane < n) {
            const int32_t h = vtx_slot[o0 + q0 + lane];
            if (face_vtx[tp.next(h)] == i) cand = face_edge[h];
            else {
                const int32_t hp = tp.prev(h);
                if (face_vtx[hp] == i) cand = face_edge[hp];
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, cand >= 0);
        if (m) { e = __shfl_sync(0xffffffffu, cand, __ffs(m) - 1); break; }
    }
    if (lane != 0) return;
    if (e < 0) {
        if (!lenient) atomicOr(flags, kFlagCrease);
        return;
    }
    if (atomicCAS(edge_cidx + e, -1, (int32_t)k) != -1) { atomicOr(flags, kFlagCrease); return; }
    if (sg > 0.0f && edge_hh[e].y >= 0) {  // boundary edges are infinitely sharp anyway (R19)
        edge_sigma[e] = sg;
        atomicOr(flag + e, 1);
        atomicAdd(sv_cnt + a, 1);
        atomicAdd(sv_cnt + b, 1);
    }
}

// One launch after the two scans (special flags -> list offsets, list lengths -> CSR offsets):
//   threads [0, E32)       special edge list in ascending edge id (compaction by the scanned
//                          flags), its bitmask words and per-word prefixes (E32 = E rounded up to
//                          whole warps: a warp is one bitmask word);
//   threads [E32, E32 + V) vertex v's special-vertex row: its incident special edges (each once:
//                          the edge leaving v in every incident face, the edge entering v where it
//                          is a boundary edge) as list indices, ascending (= the oracle's edge-id
//                          order, so crease sums match bit for bit); identity table sv_vtx[v] = v.
// (Replaces a special-edge kernel, an atomic list scatter and a per-row sort: three launches on
// the chain the level-0 edge and vertex kernels wait for.)
template <int ORDER>
__global__ void __launch_bounds__(kThreads) k_b0_special_fill(const int2 *__restrict__ edge_hh,
                                                            const int32_t *__restrict__ face_vtx,
                                                            const float *__restrict__ edge_sigma,
                                                            const int32_t *__restrict__ flag,
                                                            const int32_t *__restrict__ off, Topo<ORDER> tp, int32_t E,
                                                            SpEdge *__restrict__ sp, uint32_t *__restrict__ spw,
                                                            int32_t *__restrict__ spwpre, int32_t V,
                                                            const int32_t *__restrict__ vtx_off,
                                                            const int32_t *__restrict__ vtx_slot,
                                                            const int32_t *__restrict__ face_edge,
                                                            const int32_t *__restrict__ face_twin,
                                                            const int32_t *__restrict__ sv_off, int32_t *__restrict__ sv_list,
                                                            int32_t *__restrict__ sv_vtx, int32_t *__restrict__ scalars,
                                                            int32_t cap) {
    ALSUB_GRID_WAIT();
    const int32_t E32 = (E + 31) & ~31;
    const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < E32) {
        const int32_t e = t;
        // the special-edge bitmask word of these 32 edges (one warp = one word) and its prefix
        const int fl = e < E ? flag[e] : 0;
        const unsigned word = __ballot_sync(0xffffffffu, fl != 0);
        if ((threadIdx.x & 31) == 0 && e < E) {
            spw[e >> 5] = word;
            spwpre[e >> 5] = off[e];
        }
        if (e >= E || !fl) return;
        const int2 hh = edge_hh[e];
        const int32_t va = face_vtx[hh.x], vb = face_vtx[tp.next(hh.x)];
        const bool bnd = hh.y < 0;
        SpEdge x;
        x.e = e;
        x.a = min(va, vb);
        x.b = max(va, vb);
        x.ia = x.a;  // identity special-vertex table at level 0
        x.ib = x.b;
        x.sigma = bnd ? __int_as_float(0x7f800000) : edge_sigma[e];
        x.flags = bnd ? kSpBoundary : 0;
        x.pad = 0;
        sp[off[e]] = x;
        return;
    }
    const int32_t v = t - E32;
    if (v >= V) return;
    if (v == 0) scalars[3] = V;
    sv_vtx[v] = v;
    const int32_t o = sv_off[v], n = sv_off[v + 1] - o;
    const int32_t r0 = vtx_off[v], r1 = vtx_off[v + 1];  // (beside the list bounds)
    if (n == 0 || o + n > cap) return;
    int32_t m = 0;
    // the row's slots kSvBatch at a time, each stage's loads issued together (slot -> its two edges
    // and the twin test -> flags -> list indices), then inserted into the ascending row
    constexpr int kSvBatch = 8;
    for (int32_t q0 = r0; q0 < r1 && m < n; q0 += kSvBatch) {
        int32_t ea[kSvBatch], eb[kSvBatch];
#pragma unroll
        for (int u = 0; u < kSvBatch; ++u) {
            ea[u] = eb[u] = -1;
            if (q0 + u < r1) {
                const int32_t h = vtx_slot[q0 + u], hp = tp.prev(h);
                ea[u] = face_edge[h];
                eb[u] = face_twin[hp] < 0 ? face_edge[hp] : -1;
            }
        }
#pragma unroll
        for (int u = 0; u < kSvBatch; ++u) {  // flag and offset loaded side by side
            const int32_t fa = ea[u] >= 0 ? flag[ea[u]] : 0, oa = ea[u] >= 0 ? off[ea[u]] : 0;
            const int32_t fb = eb[u] >= 0 ? flag[eb[u]] : 0, ob = eb[u] >= 0 ? off[eb[u]] : 0;
            ea[u] = fa ? oa : -1;
            eb[u] = fb ? ob : -1;
        }
        if (r1 - r0 <= kSvBatch) {
            // the whole row in this batch: each entry's place is its rank among the row's entries
            // (distinct list indices), counted in registers -- no read-back of the list
#pragma unroll
            for (int u = 0; u < 2 * kSvBatch; ++u) {
                const int32_t x = u < kSvBatch ? ea[u] : eb[u - kSvBatch];
                if (x < 0) continue;
                int32_t r = 0;
#pragma unroll
                for (int w = 0; w < kSvBatch; ++w) r += (ea[w] >= 0 && ea[w] < x) + (eb[w] >= 0 && eb[w] < x);
                if (r < n) sv_list[o + r] = x;
            }
            break;
        }
#pragma unroll
        for (int u = 0; u < 2 * kSvBatch; ++u) {
            const int32_t x = u < kSvBatch ? ea[u] : eb[u - kSvBatch];
            if (x < 0 || m >= n) continue;
            int32_t b = m - 1;  // insertion into the ascending row
            while (b >= 0 && sv_list[o + b] > x) { sv_list[o + b + 1] = sv_list[o + b]; --b; }
            sv_list[o + b + 1] = x;
            ++m;
        }
    }
}

// ------------------------------------------------------------------------------------------
// scratch arena: 5 scan status regions, each 256-byte aligned, so a single k_zero launch can
// initialise all of them for a refine
static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }
static size_t region_bytes(int32_t V, int32_t S) { return al(scan_scratch_bytes(std::max(V, S) + 1)); }
static void *region(const Build0 &b, int k) {
    if (!b.zeroed) return b.scratch;  // create: one region reused (memset before every use)
    return (char *)b.scratch + (size_t)(k - 1) * region_bytes(b.V, b.S);
}
size_t build0_scratch_bytes(int32_t V, int32_t S) { return 5 * region_bytes(V, S); }

void build0_zero_segments(Build0 &b, ZeroSegs &z) {
    const int32_t E = b.E, nw = (int32_t)ceil_div(E > 0 ? E : 1, 32);
    z.add(b.vtx_cnt, (int64_t)b.V + 1);
    z.add(b.vtx_cur, b.V);
    z.add(b.scalars + 1, 5);  // B, K, NSV, -, long-row count
    z.add(b.bnd_word, nw);
    z.add(b.vbnd, b.V);
    z.add(b.edge_sigma, E);
    z.add(b.edge_cidx, E, -1);
    z.add(b.sp_flag, E);
    z.add(b.sv_cnt, b.V);
    z.add(b.scratch, (int64_t)(build0_scratch_bytes(b.V, b.S) / 4));
    b.zeroed = true;
}

// a1: validation + M^T row lengths
void build0_validate(Build0 &b, cudaStream_t s, Launches &L) {
    if (!b.zeroed) cudaMemsetAsync(b.vtx_cnt, 0, sizeof(int32_t) * ((size_t)b.V + 1), s);
    if (b.F > 0)
        launch(L, "b0_prep", k_b0_prep, dim3(grid_for(b.F)), dim3(kThreads), 0, s, b.face_off, b.face_vtx, b.F, b.V,
               b.slot_face, b.vtx_cnt, b.flags);
}

// long rows: launched when the create found some (nlong > 0) or does not know yet (nlong < 0)
template <int ORDER, bool FILL>
static void long_rows(Build0 &b, Topo<ORDER> tp, cudaStream_t s, Launches &L) {
    if (b.V == 0 || b.nlong == 0) return;
    const unsigned grid = (unsigned)(b.nlong < 0 ? 148 : std::min<int32_t>(b.nlong, 148));
    launch(L, FILL ? "b0_long_fill" : "b0_long_count", k_long_rows<ORDER, FILL>, dim3(grid), dim3(kLongThreads), 0, s,
           b.face_vtx, b.vtx_off, b.vtx_slot, tp, b.long_list, b.scalars + 5, b.long_keys, b.edge_cnt, b.edge_off,
           b.face_edge, b.face_twin, b.edge_hh, b.bnd_word, b.vbnd, b.scalars, b.flags);
}

// a2 + symbolic a3: M^T (row lengths scanned into vtx_off, slots scattered into their rows, rows
// sorted inside k_edge_count), then the per-vertex upper-triangle counts of E
template <int ORDER>
static void count_edges(Build0 &b, cudaStream_t s, Launches &L) {
    const Topo<ORDER> tp{b.face_off, b.slot_face};
    scan_exclusive(b.vtx_cnt, b.vtx_off, (int64_t)b.V + 1, nullptr, region(b, 1), s, L, b.zeroed);
    if (!b.zeroed && b.V > 0) cudaMemsetAsync(b.vtx_cur, 0, sizeof(int32_t) * b.V, s);
    if (b.S > 0)
        launch(L, "b0_scatter", k_b0_scatter, dim3(grid_for(b.S)), dim3(kThreads), 0, s, b.face_vtx, b.S, b.V, b.vtx_off,
               b.vtx_cur, b.vtx_slot);
    if (b.V > 0)
        launch(L, "b0_edge_count", k_edge_count<ORDER>, dim3(grid_for(32 * (int64_t)b.V)), dim3(kThreads), 0, s, b.face_vtx,
               b.vtx_off, b.vtx_slot, tp, b.V, b.edge_cnt, b.long_list, b.scalars + 5);
    long_rows<ORDER, false>(b, tp, s, L);
    scan_exclusive(b.edge_cnt, b.edge_off, b.V, b.scalars + 0, region(b, 2), s, L, b.zeroed);
}
void build0_count_edges(Build0 &b, cudaStream_t s, Launches &L) {
    if (b.order == 3) count_edges<3>(b, s, L);
    else if (b.order == 4) count_edges<4>(b, s, L);
    else count_edges<0>(b, s, L);
}

// numeric a3 + crease matrix + special lists
template <int ORDER>
static void fill(Build0 &b, bool check_fans, cudaStream_t s, Launches &L) {
    const Topo<ORDER> tp{b.face_off, b.slot_face};
    const int32_t E = b.E;
    const int32_t nw = (int32_t)ceil_div(E > 0 ? E : 1, 32);
    if (!b.zeroed) {
        cudaMemsetAsync(b.scalars + 1, 0, 3 * sizeof(int32_t), s);
        cudaMemsetAsync(b.bnd_word, 0, sizeof(uint32_t) * nw, s);
        if (b.V > 0) cudaMemsetAsync(b.vbnd, 0, sizeof(int32_t) * b.V, s);
    }
    if (b.V > 0) {
        launch(L, "b0_edge_fill", k_edge_fill<ORDER>, dim3(grid_for(32 * (int64_t)b.V)), dim3(kThreads), 0, s, b.face_vtx, b.vtx_off, b.vtx_slot, tp, b.V,
                                                                       b.edge_off, b.face_edge, b.face_twin, b.edge_hh,
                                                                       b.bnd_word, b.vbnd, b.scalars, b.flags,
                                                                       b.vtx_slot0);
        long_rows<ORDER, true>(b, tp, s, L);
        if (check_fans) {
            launch(L, "b0_check_fans", k_check_fans<ORDER>, dim3(grid_for(b.V)), dim3(kThreads), 0, s, b.face_twin, b.vtx_off, b.vtx_slot0, tp, b.V, b.flags);
        }
    }
    if (E > 0 && !b.zeroed) {
        cudaMemsetAsync(b.edge_sigma, 0, sizeof(float) * E, s);
        cudaMemsetAsync(b.edge_cidx, 0xff, sizeof(int32_t) * E, s);
        cudaMemsetAsync(b.sp_flag, 0, sizeof(int32_t) * E, s);
    }
    if (b.V > 0 && !b.zeroed) {
        cudaMemsetAsync(b.sv_cnt, 0, sizeof(int32_t) * b.V, s);
    }
    if (b.zeroed && b.no_special) return;  // closed and crease-free: no special lists, no boundary words
    const int64_t nf = std::max<int64_t>(std::max<int64_t>(E, 32 * (int64_t)b.K_in), nw);
    launch(L, "b0_flags", k_b0_flags<ORDER>, dim3(grid_for(nf)), dim3(kThreads), 0, s, b.crease_in, b.sigma_in, b.K_in, b.face_vtx, b.vtx_off, b.vtx_slot,
                                                 b.face_edge, b.edge_hh, tp, b.V, E, b.bnd_word, nw, b.edge_sigma,
                                                 b.edge_cidx, b.sp_flag, b.bnd_wcnt, b.flags, b.crease_lenient,
                                                 b.zeroed ? nullptr : b.scalars + 0, b.sv_cnt);
    // the special-list chain (special edges, special-vertex CSR) is only read by the crease rules of
    // the level kernels: with a side stream it runs as a parallel branch beside the boundary-word
    // prefix scan and the level-0 face kernel, and stays open (L.build_open) until the level-0
    // vertex kernel, the first reader on the main stream, waits for L.ev_build (the edge kernel
    // follows it on the side stream itself)
    const bool fork = L.can_fork() && b.zeroed && L.ev_build;
    cudaStream_t sc = s;
    if (fork) {
        cudaEventRecord(L.ev_fork, s);
        cudaStreamWaitEvent(L.side, L.ev_fork, 0);
        sc = L.side;
    }
    scan_exclusive(b.bnd_wcnt, b.bnd_wpre, nw, nullptr, region(b, 3), s, L, b.zeroed);
    if (b.zeroed) {
        scan_exclusive2(b.sp_flag, b.sp_off, E, b.scalars + 2, region(b, 4), b.sv_cnt, b.sv_off, b.V, b.sv_off + b.V,
                        region(b, 5), sc, L, true);
    } else {  // create: one scratch region, reused by scans in sequence
        scan_exclusive(b.sp_flag, b.sp_off, E, b.scalars + 2, region(b, 4), sc, L, false);
        scan_exclusive(b.sv_cnt, b.sv_off, b.V, b.sv_off + b.V, region(b, 5), sc, L, false);
    }
    const int64_t nt = (int64_t)((E + 31) & ~31) + b.V;
    if (nt > 0) {
        launch(L, "b0_special", k_b0_special_fill<ORDER>, dim3(grid_for(nt)), dim3(kThreads), 0, sc, b.edge_hh, b.face_vtx,
               b.edge_sigma, b.sp_flag, b.sp_off, tp, E, b.sp, b.spw, b.spwpre, b.V, b.vtx_off, b.vtx_slot, b.face_edge,
               b.face_twin, b.sv_off, b.sv_list, b.sv_vtx, b.scalars, 2 * b.S);
    }
    if (fork) {
        cudaEventRecord(L.ev_build, L.side);
        L.build_open = true;
    }
}

void build0_fill(Build0 &b, bool check_fans, cudaStream_t s, Launches &L) {
    if (b.order == 3) fill<3>(b, check_fans, s, L);
    else if (b.order == 4) fill<4>(b, check_fans, s, L);
    else fill<0>(b, check_fans, s, L);
}

}  // namespace alsub
