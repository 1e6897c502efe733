// scan.cuh -- the single-pass decoupled look-back exclusive scan, templated on its input so a
// producer (e.g. the Loop child-edge counts) can be fused into the scan's load phase.
#pragma once
#include "internal.h"

namespace alsub {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

constexpr unsigned long long kStatAgg = 1ull << 62;
constexpr unsigned long long kStatInc = 2ull << 62;
constexpr unsigned long long kStatMask = (1ull << 62) - 1;

inline size_t scan_scratch_bytes_impl(int64_t n) {
    int64_t tiles = ceil_div(n > 0 ? n : 1, kScanTile);
    return (size_t)(tiles + 2) * sizeof(unsigned long long);
}

__device__ __forceinline__ int warp_incl_scan(int v) {
    const unsigned lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int o = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= (unsigned)d) v += o;
    }
    return v;
}

// Src: int32_t operator()(int64_t i) -- the value of element i (i < n)
template <class Src>
__device__ __forceinline__ void scan_tile(Src in, int32_t *__restrict__ out, int64_t n, unsigned long long *status,
                                          int32_t *total) {
    __shared__ int s_tile;
    __shared__ int s_data[kScanTile + kScanTile / 32];
    __shared__ int s_warp[kScanThreads / 32];
    __shared__ long long s_prefix;
    unsigned *counter = reinterpret_cast<unsigned *>(status);  // word 0 = tile counter
    unsigned long long *stat = status + 2;
    const int tid = threadIdx.x;
    if (tid == 0) s_tile = (int)atomicAdd(counter, 1u);
    __syncthreads();
    const int tile = s_tile;
    const int64_t base = (int64_t)tile * kScanTile;
    // striped, coalesced load into padded smem
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int i = k * kScanThreads + tid;
        int64_t g = base + i;
        s_data[i + (i >> 5)] = g < n ? in(g) : 0;
    }
    __syncthreads();
    int v[kScanItems];
    int sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int i = tid * kScanItems + k;
        v[k] = s_data[i + (i >> 5)];
        sum += v[k];
    }
    int incl = warp_incl_scan(sum);
    const int warp = tid >> 5, lane = tid & 31;
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int w = lane < kScanThreads / 32 ? s_warp[lane] : 0;
        w = warp_incl_scan(w);
        if (lane < kScanThreads / 32) s_warp[lane] = w;
    }
    __syncthreads();
    const int block_total = s_warp[kScanThreads / 32 - 1];
    int excl = incl - sum + (warp > 0 ? s_warp[warp - 1] : 0);
    if (warp == 0) {
        // warp-wide look-back: lane l inspects predecessor tile - 1 - l (32 status words per round)
        long long prefix = 0;
        if (tile == 0) {
            if (lane == 0) atomicExch(&stat[0], kStatInc | (unsigned long long)block_total);
        } else {
            if (lane == 0) atomicExch(&stat[tile], kStatAgg | (unsigned long long)block_total);
            int p0 = tile - 1;
            while (true) {
                const int p = p0 - lane;
                unsigned long long w = 0;
                if (p >= 0) {
                    do {
                        w = *(volatile unsigned long long *)&stat[p];
                    } while ((w >> 62) == 0);
                }
                // nearest inclusive predecessor among the 32 (tile 0 is always inclusive)
                const unsigned inc = __ballot_sync(0xffffffffu, p >= 0 && (w >> 62) == 2);
                const int stop = inc ? __ffs(inc) - 1 : 31;
                long long v = (p >= 0 && lane <= stop) ? (long long)(w & kStatMask) : 0;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
                prefix += v;
                if (inc) break;
                p0 -= 32;
            }
            if (lane == 0) atomicExch(&stat[tile], kStatInc | (unsigned long long)(prefix + block_total));
        }
        if (lane == 0) s_prefix = prefix;
    }
    __syncthreads();
    int run = (int)s_prefix + excl;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int i = tid * kScanItems + k;
        s_data[i + (i >> 5)] = run;
        run += v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int i = k * kScanThreads + tid;
        int64_t g = base + i;
        if (g < n) out[g] = s_data[i + (i >> 5)];
    }
    if (total && tid == 0 && base + kScanTile >= n) *total = (int)(s_prefix + block_total);
}

template <class Src>
__global__ void __launch_bounds__(kScanThreads) k_scan(Src in, int32_t *__restrict__ out, int64_t n,
                                                     unsigned long long *status, int32_t *total) {
    ALSUB_GRID_WAIT();
    scan_tile(in, out, n, status, total);
}

// two independent scans in one launch: blocks [0, tilesA) scan A, the rest B (each array keeps
// its own status words and tile counter, so the look-back order stays per array)
template <class Src>
__global__ void __launch_bounds__(kScanThreads) k_scan2(Src ina, int32_t *__restrict__ outa, int64_t na,
                                                      unsigned long long *sta, int32_t *tota, Src inb,
                                                      int32_t *__restrict__ outb, int64_t nb,
                                                      unsigned long long *stb, int32_t *totb, int32_t tilesa) {
    ALSUB_GRID_WAIT();
    if ((int32_t)blockIdx.x < tilesa) scan_tile(ina, outa, na, sta, tota);
    else scan_tile(inb, outb, nb, stb, totb);
}

struct ArraySrc {
    const int32_t *p;
    ALSUB_D int32_t operator()(int64_t i) const { return p[i]; }
};

}  // namespace alsub
