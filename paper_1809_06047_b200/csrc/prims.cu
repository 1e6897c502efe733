// prims.cu -- device-wide primitives for the level-0 mesh-matrix build
// and the count -> scan -> fill stages of the paper's two-stage constructions.
//
//  * scan_exclusive: single-pass decoupled look-back scan (one read + one write of the array).
//  * zero_segments: one launch initialising up to 32 arrays (instead of memset graph nodes).
//  * pack_channels / unpack_channels: vertex channels <-> 3-float frames.
#include <algorithm>

#include "internal.h"

namespace alsub {

// ------------------------------------------------------------------------------------------
// decoupled look-back scan
// ------------------------------------------------------------------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

constexpr unsigned long long kStatAgg = 1ull << 62;
constexpr unsigned long long kStatInc = 2ull << 62;
constexpr unsigned long long kStatMask = (1ull << 62) - 1;

size_t scan_scratch_bytes(int64_t n) {
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

__global__ void __launch_bounds__(kScanThreads) k_scan(const int32_t *__restrict__ in, int32_t *__restrict__ out,
                                                     int64_t n, unsigned long long *status, int32_t *total) {
    ALSUB_GRID_WAIT();
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
        s_data[i + (i >> 5)] = g < n ? in[g] : 0;
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

void scan_exclusive(const int32_t *in, int32_t *out, int64_t n, int32_t *total, void *scratch, cudaStream_t s,
                    Launches &L, bool prezeroed) {
    if (n <= 0) {
        if (total) cudaMemsetAsync(total, 0, sizeof(int32_t), s);
        return;
    }
    if (!prezeroed) cudaMemsetAsync(scratch, 0, scan_scratch_bytes(n), s);
    int64_t tiles = ceil_div(n, kScanTile);
    launch(L, "scan", k_scan, dim3((unsigned)tiles), dim3(kScanThreads), 0, s, in, out, n, (unsigned long long *)scratch, total);
}

// ------------------------------------------------------------------------------------------
// one launch that initialises many small arrays (replaces a chain of memset graph nodes)
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_zero(ZeroSegs z) {
    ALSUB_GRID_WAIT();
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    for (int k = 0; k < z.n; ++k)
        for (int64_t i = tid; i < z.words[k]; i += nth) z.ptr[k][i] = z.value[k];
}

void zero_segments(const ZeroSegs &z, cudaStream_t s, Launches &L) {
    int64_t mx = 0;
    for (int k = 0; k < z.n; ++k) mx = std::max(mx, z.words[k]);
    if (mx == 0) return;
    launch(L, "zero", k_zero, dim3((unsigned)std::min<int64_t>(ceil_div(mx, kThreads), 4 * 148)), dim3(kThreads), 0, s, z);
}

}  // namespace alsub

namespace alsub {
// ---------------- vertex channels <-> 3-float frames (alsub_eval_attributes) ----------------
// [V][C] channel rows <-> ceil(C/3) frames [g][V][3]; channel 3g + k of vertex v is component k
// of frame g (the padding components of the last frame are zero)
__global__ void k_pack_channels(const float *__restrict__ in, int64_t V, int32_t C, float *__restrict__ out) {
    ALSUB_GRID_WAIT();
    const int32_t ng = (C + 2) / 3;
    const int64_t n = V * 3 * ng;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = i / (3 * V), r = i - g * 3 * V, v = r / 3;
        const int32_t ch = (int32_t)(3 * g + (r - 3 * v));
        out[i] = ch < C ? in[v * C + ch] : 0.0f;
    }
}
__global__ void k_unpack_channels(const float *__restrict__ in, int64_t V, int32_t C, float *__restrict__ out) {
    ALSUB_GRID_WAIT();
    const int64_t n = V * C;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / C;
        const int32_t ch = (int32_t)(i - v * C), g = ch / 3;
        out[i] = in[(int64_t)g * 3 * V + 3 * v + (ch - 3 * g)];
    }
}
void pack_channels(const float *in, int64_t V, int32_t C, float *out, cudaStream_t s, Launches &L) {
    const int64_t n = V * 3 * ((C + 2) / 3);
    if (n > 0) launch(L, "pack_channels", k_pack_channels, dim3((unsigned)std::min<int64_t>(grid_for(n), 148 * 16)), dim3(kThreads), 0, s, in, V, C, out);
}
void unpack_channels(const float *in, int64_t V, int32_t C, float *out, cudaStream_t s, Launches &L) {
    const int64_t n = V * C;
    if (n > 0) launch(L, "unpack_channels", k_unpack_channels, dim3((unsigned)std::min<int64_t>(grid_for(n), 148 * 16)), dim3(kThreads), 0, s, in, V, C, out);
}
}  // namespace alsub
