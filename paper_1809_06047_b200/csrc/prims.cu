// prims.cu -- device-wide primitives for the level-0 mesh-matrix build
// and the count -> scan -> fill stages of the paper's two-stage constructions.
//
//  * scan_exclusive: single-pass decoupled look-back scan (one read + one write of the array).
//  * radix_sort_pairs: stable LSD radix sort, 8-bit digits, histogram -> scan -> scatter per pass;
//    the scatter ranks keys with warp match (__match_any_sync) so equal digits keep their order.
//  * offsets_from_sorted: CSR column pointer of sorted keys ("segmented scan / run-length").
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
    if (tid == 0) {
        long long prefix = 0;
        if (tile == 0) {
            atomicExch(&stat[0], kStatInc | (unsigned long long)block_total);
        } else {
            atomicExch(&stat[tile], kStatAgg | (unsigned long long)block_total);
            int p = tile - 1;
            while (true) {
                unsigned long long w;
                do {
                    w = atomicAdd(&stat[p], 0ull);
                } while ((w >> 62) == 0);
                prefix += (long long)(w & kStatMask);
                if ((w >> 62) == 2) break;
                --p;
            }
            atomicExch(&stat[tile], kStatInc | (unsigned long long)(prefix + block_total));
        }
        s_prefix = prefix;
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
// LSD radix sort (stable), 8-bit digits
// ------------------------------------------------------------------------------------------
constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;

static int64_t sort_blocks(int64_t n) { return ceil_div(n > 0 ? n : 1, kSortTile); }

size_t sort_scratch_bytes(int64_t n) {
    int64_t cnt = 256 * sort_blocks(n);
    return (size_t)(2 * cnt + 16) * sizeof(int32_t) + scan_scratch_bytes(cnt) + 256;
}

__global__ void __launch_bounds__(kSortThreads) k_rs_hist(const int32_t *__restrict__ keys, int64_t n, int shift,
                                                        int32_t *__restrict__ counts, int nblocks) {
    ALSUB_GRID_WAIT();
    __shared__ int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kSortTile;
    for (int k = 0; k < kSortItems; ++k) {
        int64_t i = base + k * kSortThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[((uint32_t)keys[i] >> shift) & 255u], 1);
    }
    __syncthreads();
    counts[threadIdx.x * nblocks + blockIdx.x] = h[threadIdx.x];  // digit-major
}

__global__ void __launch_bounds__(kSortThreads) k_rs_scatter(const int32_t *__restrict__ keys,
                                                           const int32_t *__restrict__ vals, int64_t n, int shift,
                                                           const int32_t *__restrict__ offs, int nblocks,
                                                           int32_t *__restrict__ okeys, int32_t *__restrict__ ovals) {
    ALSUB_GRID_WAIT();
    __shared__ int run[256];
    __shared__ int wc[kSortThreads / 32][256];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    run[tid] = offs[tid * nblocks + blockIdx.x];
    const int64_t base = (int64_t)blockIdx.x * kSortTile;
    for (int k = 0; k < kSortItems; ++k) {
        for (int w = 0; w < kSortThreads / 32; ++w) wc[w][tid] = 0;
        __syncthreads();
        int64_t i = base + k * kSortThreads + tid;
        bool valid = i < n;
        int32_t key = valid ? keys[i] : 0;
        int32_t val = valid ? vals[i] : 0;
        unsigned d = valid ? (((uint32_t)key >> shift) & 255u) : 256u;  // 256 = invalid bucket
        unsigned peers = __match_any_sync(0xffffffffu, d);
        int rank = __popc(peers & ((1u << lane) - 1u));
        int leader = __ffs(peers) - 1;
        if (valid && lane == leader) wc[warp][d] = __popc(peers);
        __syncthreads();
        if (valid) {
            int pos = run[d] + rank;
            for (int w = 0; w < warp; ++w) pos += wc[w][d];
            okeys[pos] = key;
            ovals[pos] = val;
        }
        __syncthreads();
        int add = 0;
        for (int w = 0; w < kSortThreads / 32; ++w) add += wc[w][tid];
        run[tid] += add;
        __syncthreads();
    }
}

void radix_sort_pairs(int32_t *keys, int32_t *vals, int32_t *keys_alt, int32_t *vals_alt, int64_t n, int bits,
                      void *scratch, cudaStream_t s, Launches &L) {
    if (n <= 1) return;
    const int nblocks = (int)sort_blocks(n);
    const int64_t cnt = 256 * (int64_t)nblocks;
    int32_t *counts = (int32_t *)scratch;
    int32_t *offs = counts + cnt;
    void *scan_scratch = (void *)(((uintptr_t)(offs + cnt + 16) + 255) & ~(uintptr_t)255);
    int passes = (bits + 7) / 8;
    if (passes < 1) passes = 1;
    int32_t *ka = keys, *va = vals, *kb = keys_alt, *vb = vals_alt;
    for (int p = 0; p < passes; ++p) {
        int shift = 8 * p;
        launch(L, "rs_hist", k_rs_hist, dim3(nblocks), dim3(kSortThreads), 0, s, ka, n, shift, counts, nblocks);
        scan_exclusive(counts, offs, cnt, nullptr, scan_scratch, s, L);
        launch(L, "rs_scatter", k_rs_scatter, dim3(nblocks), dim3(kSortThreads), 0, s, ka, va, n, shift, offs, nblocks, kb, vb);
        int32_t *t;
        t = ka; ka = kb; kb = t;
        t = va; va = vb; vb = t;
    }
    if (ka != keys) {
        cudaMemcpyAsync(keys, ka, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(vals, va, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
    }
}

// ------------------------------------------------------------------------------------------
// One-sweep LSD radix sort: digit histograms of every pass are computed up front (by the caller's
// fused kernel or k_os_hist), then ONE kernel per pass ranks each tile stably (warp match) and
// gets its per-digit offset by a decoupled look-back over the previous tiles (256 digits looked
// back in parallel, one per thread).
// ------------------------------------------------------------------------------------------
constexpr int kOsThreads = 256;
constexpr int kOsItems = 4;
constexpr int kOsTile = kOsThreads * kOsItems;

static int64_t os_tiles(int64_t n) { return ceil_div(n > 0 ? n : 1, kOsTile); }

size_t onesweep_scratch_bytes(int64_t n, int passes) {
    // per pass: tile counter (4 B, padded to 64) + ntiles x 256 status words
    return (size_t)passes * (64 + (size_t)os_tiles(n) * 256 * 4);
}

__global__ void __launch_bounds__(kOsThreads) k_os_hist(const int32_t *__restrict__ keys, int64_t n, int passes,
                                                      int32_t *__restrict__ counts) {
    ALSUB_GRID_WAIT();
    __shared__ int h[4][256];
    for (int p = 0; p < passes; ++p) h[p][threadIdx.x] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = (uint32_t)keys[i];
        for (int p = 0; p < passes; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 255u], 1);
    }
    __syncthreads();
    for (int p = 0; p < passes; ++p)
        if (h[p][threadIdx.x]) atomicAdd(counts + 256 * p + threadIdx.x, h[p][threadIdx.x]);
}

constexpr uint32_t kOsAgg = 1u << 30, kOsInc = 2u << 30, kOsMask = (1u << 30) - 1;

__global__ void __launch_bounds__(kOsThreads) k_os_pass(const int32_t *__restrict__ keys, const int32_t *__restrict__ vals,
                                                      int64_t n, int shift, const int32_t *__restrict__ counts,
                                                      uint32_t *status, unsigned *counter, int32_t *__restrict__ okeys,
                                                      int32_t *__restrict__ ovals) {
    ALSUB_GRID_WAIT();
    __shared__ int s_tile;
    __shared__ int s_base[256];       // global exclusive prefix of the digit + this tile's look-back
    __shared__ int s_cnt[256];        // this tile's digit counts
    __shared__ int wc[kOsThreads / 32][257];
    __shared__ int s_run[256];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) s_tile = (int)atomicAdd(counter, 1u);
    // global digit prefix (exclusive scan of the 256 pass counts; one warp-free serial-in-smem pass)
    s_cnt[tid] = counts[tid];
    __syncthreads();
    if (tid == 0) {
        int acc = 0;
        for (int d = 0; d < 256; ++d) { const int c = s_cnt[d]; s_cnt[d] = acc; acc += c; }
    }
    __syncthreads();
    s_base[tid] = s_cnt[tid];
    s_run[tid] = 0;
    s_cnt[tid] = 0;
    __syncthreads();
    const int tile = s_tile;
    const int64_t base = (int64_t)tile * kOsTile;
    int32_t key[kOsItems], val[kOsItems], rank[kOsItems];
    unsigned dig[kOsItems];
    // load the whole tile first (all loads in flight together), then rank from registers
#pragma unroll
    for (int k = 0; k < kOsItems; ++k) {
        const int64_t i = base + k * kOsThreads + tid;
        const bool valid = i < n;
        key[k] = valid ? keys[i] : 0;
        val[k] = valid ? vals[i] : 0;
        dig[k] = valid ? (((uint32_t)key[k] >> shift) & 255u) : 256u;
    }
    // stable local ranks, round by round (element order = base + k * 256 + tid)
#pragma unroll
    for (int k = 0; k < kOsItems; ++k) {
        for (int w = 0; w < kOsThreads / 32; ++w) wc[w][tid] = 0;
        __syncthreads();
        const bool valid = dig[k] < 256u;
        const unsigned peers = __match_any_sync(0xffffffffu, dig[k]);
        const int r = __popc(peers & ((1u << lane) - 1u));
        if (valid && (__ffs(peers) - 1) == lane) wc[warp][dig[k]] = __popc(peers);
        __syncthreads();
        if (valid) {
            int pos = s_run[dig[k]] + r;
            for (int w = 0; w < warp; ++w) pos += wc[w][dig[k]];
            rank[k] = pos;
        }
        __syncthreads();
        int add = 0;
        for (int w = 0; w < kOsThreads / 32; ++w) add += wc[w][tid];
        s_run[tid] += add;
        __syncthreads();
    }
    // decoupled look-back, one digit per thread
    {
        const int d = tid;
        const uint32_t mine = (uint32_t)s_run[d];
        uint32_t *st = status + (int64_t)tile * 256 + d;
        if (tile == 0) {
            atomicExch(st, kOsInc | mine);
        } else {
            atomicExch(st, kOsAgg | mine);
            uint32_t prefix = 0;
            for (int p = tile - 1; p >= 0; --p) {
                uint32_t w;
                do {
                    w = atomicAdd(status + (int64_t)p * 256 + d, 0u);
                } while ((w >> 30) == 0);
                prefix += w & kOsMask;
                if ((w >> 30) == 2) break;
            }
            atomicExch(st, kOsInc | (prefix + mine));
            s_base[d] += (int)prefix;
        }
    }
    __syncthreads();
    for (int k = 0; k < kOsItems; ++k) {
        const int64_t i = base + k * kOsThreads + tid;
        if (i < n) {
            const int pos = s_base[dig[k]] + rank[k];
            okeys[pos] = key[k];
            ovals[pos] = val[k];
        }
    }
}

void radix_sort_onesweep(int32_t *keys, int32_t *vals, int32_t *keys_alt, int32_t *vals_alt, int64_t n, int bits,
                         int32_t *counts, bool counts_ready, void *scratch, cudaStream_t s, Launches &L,
                         bool prezeroed) {
    int passes = (bits + 7) / 8;
    if (passes < 1) passes = 1;
    if (n <= 1) return;
    if (!counts_ready) {
        cudaMemsetAsync(counts, 0, sizeof(int32_t) * 256 * passes, s);
        launch(L, "os_hist", k_os_hist, dim3((unsigned)std::min<int64_t>(ceil_div(n, kOsThreads), 4 * 148)), dim3(kOsThreads), 0, s, keys, n, passes, counts);
    }
    if (!prezeroed) cudaMemsetAsync(scratch, 0, onesweep_scratch_bytes(n, passes), s);
    const int64_t tiles = os_tiles(n);
    int32_t *ka = keys, *va = vals, *kb = keys_alt, *vb = vals_alt;
    for (int p = 0; p < passes; ++p) {
        char *base = (char *)scratch + (size_t)p * (64 + (size_t)tiles * 256 * 4);
        launch(L, "os_pass", k_os_pass, dim3((unsigned)tiles), dim3(kOsThreads), 0, s, ka, va, n, 8 * p, counts + 256 * p, (uint32_t *)(base + 64),
                                                         (unsigned *)base, kb, vb);
        int32_t *t;
        t = ka; ka = kb; kb = t;
        t = va; va = vb; vb = t;
    }
    if (ka != keys) {
        cudaMemcpyAsync(keys, ka, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(vals, va, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
    }
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

// ------------------------------------------------------------------------------------------
// CSR offsets of sorted keys (run-length of the sorted key array)
// ------------------------------------------------------------------------------------------
__global__ void k_offsets(const int32_t *__restrict__ keys, int64_t n, int32_t *__restrict__ off, int32_t nkeys) {
    ALSUB_GRID_WAIT();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t k = keys[i];
    int32_t kp = i == 0 ? -1 : keys[i - 1];
    for (int32_t v = kp + 1; v <= k; ++v) off[v] = (int32_t)i;
    if (i == n - 1)
        for (int32_t v = k + 1; v <= nkeys; ++v) off[v] = (int32_t)n;
}

__global__ void k_fill_i32(int32_t *p, int64_t n, int32_t val) {
    ALSUB_GRID_WAIT();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = val;
}

void offsets_from_sorted(const int32_t *keys, int64_t n, int32_t *off, int32_t nkeys, cudaStream_t s, Launches &L) {
    if (n == 0) {
        cudaMemsetAsync(off, 0, sizeof(int32_t) * ((size_t)nkeys + 1), s);
        return;
    }
    launch(L, "offsets", k_offsets, dim3(grid_for(n)), dim3(kThreads), 0, s, keys, n, off, nkeys);
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
