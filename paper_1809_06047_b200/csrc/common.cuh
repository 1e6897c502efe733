// common.cuh -- device-side helpers shared by the AlSub sm_100a kernels.
//
// Mesh representation on the device:
//   slot h = one non-zero of the mesh matrix M: vertex face_vtx[h] of face face(h)
//   at cyclic position h - off(face).  Reduced matrices (all quads / all triangles)
//   have no column pointer: face(h) = h / c.  Level 0 with mixed orders keeps face_off[F+1]
//   and a slot_face[S] table.
//   face_edge[h]  id of the edge v(h) -> v(next(h))       (E's enumeration)
//   face_twin[h]  slot of the reverse directed edge or -1 (F(j,i) of Eq. F)
//   edge_hh[e]    (smallest slot carrying edge e, the other slot or -1 on a boundary)
//   vtx_slot0[v]  (Loop / sqrt3) one slot at vertex v; the 1-ring is walked with
//                 next-around(h) = twin(prev(h)).  CC derives each vertex's row of M in closed
//                 form from the level the vertex was born at (VSegs in internal.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define ALSUB_HD __host__ __device__ __forceinline__
#define ALSUB_D __device__ __forceinline__
// first statement of every kernel: wait for the predecessor grid (programmatic dependent launch).
// Small grids (at most kEarlyTriggerBlocks CTAs, i.e. the latency-bound small levels) then let the
// next kernel in the stream launch at once: its CTAs take free SM slots and wait in their own
// griddepcontrol.wait, which hides the dependent-launch latency.  The trigger comes after the
// wait, so at most one grid runs ahead.  Large grids do not trigger (waiting CTAs would take
// slots from a bandwidth-bound kernel).
#ifndef ALSUB_EARLY_TRIGGER_BLOCKS
#define ALSUB_EARLY_TRIGGER_BLOCKS 296
#endif
#define ALSUB_GRID_WAIT()                                                                  \
    do {                                                                                  \
        asm volatile("griddepcontrol.wait;" ::: "memory");                                \
        if (gridDim.x * gridDim.y * gridDim.z <= ALSUB_EARLY_TRIGGER_BLOCKS)              \
            asm volatile("griddepcontrol.launch_dependents;" ::: "memory");                \
    } while (0)
// let the next kernel in the stream begin launching (its blocks wait in ALSUB_GRID_WAIT)
#define ALSUB_GRID_LAUNCH_NEXT() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")

namespace alsub {

constexpr int kThreads = 256;

// Topology accessors for a face order known at compile time (3, 4) or mixed (0).
template <int ORDER>
struct Topo {
    const int32_t *face_off;   // [F+1]   (ORDER == 0 only)
    const int32_t *slot_face;  // [S]     (ORDER == 0 only)
    ALSUB_D int32_t face(int32_t h) const {
        if constexpr (ORDER == 0) return __ldg(slot_face + h);
        else return h / ORDER;
    }
    ALSUB_D int32_t first(int32_t f) const {
        if constexpr (ORDER == 0) return __ldg(face_off + f);
        else return f * ORDER;
    }
    ALSUB_D int32_t order(int32_t f) const {
        if constexpr (ORDER == 0) return __ldg(face_off + f + 1) - __ldg(face_off + f);
        else return ORDER;
    }
    ALSUB_D int32_t next(int32_t h) const {
        if constexpr (ORDER == 4) return (h & ~3) | ((h + 1) & 3);
        else if constexpr (ORDER == 3) { int32_t t = h % 3; return t == 2 ? h - 2 : h + 1; }
        else { int32_t f = face(h); int32_t o = first(f); int32_t c = order(f); return h + 1 == o + c ? o : h + 1; }
    }
    ALSUB_D int32_t prev(int32_t h) const {
        if constexpr (ORDER == 4) return (h & ~3) | ((h + 3) & 3);
        else if constexpr (ORDER == 3) { int32_t t = h % 3; return t == 0 ? h + 2 : h - 1; }
        else { int32_t f = face(h); int32_t o = first(f); int32_t c = order(f); return h == o ? o + c - 1 : h - 1; }
    }
};

// fp32 [V][3] positions (the API layout).  12-byte gathers; the write side is coalesced
// across a warp because consecutive threads own consecutive items.
struct P3 {
    float x, y, z;
};
ALSUB_D P3 ld3(const float *__restrict__ P, int64_t v) {
    const float *p = P + 3 * v;
    return P3{__ldg(p), __ldg(p + 1), __ldg(p + 2)};
}
// plain (coherent) load: for data written earlier in the same stream by another kernel
ALSUB_D P3 ld3c(const float *P, int64_t v) {
    const float *p = P + 3 * v;
    return P3{p[0], p[1], p[2]};
}
ALSUB_D void st3(float *P, int64_t v, P3 a) {
    float *p = P + 3 * v;
    p[0] = a.x;
    p[1] = a.y;
    p[2] = a.z;
}
// strided views of one frame's positions: element v at p + vs * v (vs = 3 for the API layout
// [V][3]; vs = 3 nb for the frame-interleaved batches [V][nb][3] of alsub_eval_frames)
struct PR {
    const float *p;
    int32_t vs;
};
struct PW {
    float *p;
    int32_t vs;
};
ALSUB_D P3 ld3(PR P, int64_t v) {
    const float *q = P.p + P.vs * v;
    return P3{__ldg(q), __ldg(q + 1), __ldg(q + 2)};
}
ALSUB_D P3 ld3c(PR P, int64_t v) {
    const float *q = P.p + P.vs * v;
    return P3{q[0], q[1], q[2]};
}
ALSUB_D P3 ld3c(PW P, int64_t v) {
    const float *q = P.p + P.vs * v;
    return P3{q[0], q[1], q[2]};
}
// wide gather: a 12-byte element as one 8-byte and one 4-byte load (whichever half is 8-byte
// aligned) instead of three 4-byte loads -- scattered gathers are bound by the L1 data pipe's
// wavefronts (one per load instruction and line touched).  Costs registers: used where measured
// faster (sqrt3 kernels); on the CC and Loop kernels it raised spills and was slower
ALSUB_D P3 ld3w(PR P, int64_t v) {
    const float *q = P.p + P.vs * v;
    const bool odd = (reinterpret_cast<uintptr_t>(q) & 4) != 0;
    const float2 d = __ldg(reinterpret_cast<const float2 *>(q + (odd ? 1 : 0)));
    const float s = __ldg(q + (odd ? 0 : 2));
    return odd ? P3{s, d.x, d.y} : P3{d.x, d.y, s};
}
ALSUB_D void st3(PW P, int64_t v, P3 a) {
    float *q = P.p + P.vs * v;
    q[0] = a.x;
    q[1] = a.y;
    q[2] = a.z;
}
ALSUB_D P3 operator+(P3 a, P3 b) { return P3{a.x + b.x, a.y + b.y, a.z + b.z}; }
ALSUB_D P3 operator*(float s, P3 a) { return P3{s * a.x, s * a.y, s * a.z}; }
ALSUB_D P3 p3zero() { return P3{0.f, 0.f, 0.f}; }

// Per-frame summary record (alsub_frame_summary, include/alsub.h): bbox lo.xyz / hi.xyz and the
// wrapping checksum sum_i bits(x_i) (2 i + 1).  While accumulating, lo / hi hold the ordered-int
// image of the floats (f2ord: the same total order as the floats, so atomicMin / atomicMax on ints
// apply); a decode pass turns them back into float bits.
struct SummaryRec {
    int32_t lo[3], hi[3];
    unsigned long long sum;
};
ALSUB_D int32_t f2ord(float f) {
    const int32_t i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
ALSUB_D float ord2f(int32_t i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

// Long rings (level-0 vertices with more than kLongRing incident slots, e.g. poles): the vertex
// kernels skip them in their per-lane pass and then sum each one's ring with the whole warp --
// lanes take slots k = lane, lane + 32, ...; warp_sum is a fixed xor butterfly, so the result is
// deterministic (and identical between refine and eval_frames, which share the kernels).
constexpr int32_t kLongRing = 32;
constexpr int32_t kLongRow = 16;  // M^T rows longer than this are listed by the level-0 build
ALSUB_D P3 warp_sum(P3 a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
        a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
        a.z += __shfl_xor_sync(0xffffffffu, a.z, o);
    }
    return a;
}

// Boundary-edge prefix: bprefix(e) = number of boundary edges with id < e, from a bitmask and
// per-word exclusive prefix.
ALSUB_D int32_t bprefix(const uint32_t *__restrict__ words, const int32_t *__restrict__ wpre, int32_t e) {
    int32_t w = e >> 5;
    uint32_t m = __ldg(words + w) & ((1u << (e & 31)) - 1u);
    return __ldg(wpre + w) + __popc(m);
}

// Special (boundary or creased) edge of a level: boundary edges are infinitely sharp creases
// (reading R6).  Level l's list has K_l = 2^l K_0 entries in edge-id order; entry j's children
// are entries 2j (endpoint a) and 2j + 1 (endpoint b) of the next level -- dead children keep
// sigma = 0, so the list never needs compaction and every index is closed-form.
struct alignas(16) SpEdge {
    int32_t e, a, b;   // edge id, endpoints a < b
    int32_t ia, ib;    // special-vertex indices of a and b
    float sigma;       // 0 = dead, > 0, +inf for boundary / infinitely sharp
    int32_t flags;     // bit 0: boundary
    int32_t pad;
};
constexpr int32_t kSpBoundary = 1;

// Special-vertex table of a level: vertex ids sv_vtx[i] with their incident special edges
// sv_list[sv_off[i] .. sv_off[i+1]) (CSR).  The next level keeps the same vertices with the same
// list lengths (entry j -> 2j + (vertex is b_j)) and appends one vertex per special edge (its edge
// point) with the two entries {2j, 2j + 1}.
// Device-side status flags written by the level-0 build (read back by alsub_mesh_create).
enum : int32_t {
    kFlagMesh = 1, kFlagNonManifold = 2, kFlagCrease = 4, kFlagOrder = 8,
};

}  // namespace alsub
