// prims.cu -- device-wide primitives for the level-0 mesh-matrix build
// and the count -> scan -> fill stages of the paper's two-stage constructions.
//
//  * scan_exclusive: single-pass decoupled look-back scan (one read + one write of the array).
//  * zero_segments: one launch initialising up to 32 arrays (instead of memset graph nodes).
//  * pack_channels / unpack_channels: vertex channels <-> 3-float frames.
#include <algorithm>

#include "internal.h"
#include "scan.cuh"

namespace alsub {

// ------------------------------------------------------------------------------------------
// decoupled look-back scan
// ------------------------------------------------------------------------------------------
size_t scan_scratch_bytes(int64_t n) { return scan_scratch_bytes_impl(n); }

void scan_exclusive(const int32_t *in, int32_t *out, int64_t n, int32_t *total, void *scratch, cudaStream_t s,
                    Launches &L, bool prezeroed) {
    if (n <= 0) {
        if (total) cudaMemsetAsync(total, 0, sizeof(int32_t), s);
        return;
    }
    if (!prezeroed) cudaMemsetAsync(scratch, 0, scan_scratch_bytes(n), s);
    int64_t tiles = ceil_div(n, kScanTile);
    launch(L, "scan", k_scan<ArraySrc>, dim3((unsigned)tiles), dim3(kScanThreads), 0, s, ArraySrc{in}, out, n,
           (unsigned long long *)scratch, total);
}

void scan_exclusive2(const int32_t *ina, int32_t *outa, int64_t na, int32_t *tota, void *scra,
                     const int32_t *inb, int32_t *outb, int64_t nb, int32_t *totb, void *scrb, cudaStream_t s,
                     Launches &L, bool prezeroed) {
    if (na <= 0 || nb <= 0) {  // (degenerate inputs: the plain scans)
        scan_exclusive(ina, outa, na, tota, scra, s, L, prezeroed);
        scan_exclusive(inb, outb, nb, totb, scrb, s, L, prezeroed);
        return;
    }
    if (!prezeroed) {
        cudaMemsetAsync(scra, 0, scan_scratch_bytes(na), s);
        cudaMemsetAsync(scrb, 0, scan_scratch_bytes(nb), s);
    }
    const int64_t ta = ceil_div(na, kScanTile), tb = ceil_div(nb, kScanTile);
    launch(L, "scan2", k_scan2<ArraySrc>, dim3((unsigned)(ta + tb)), dim3(kScanThreads), 0, s, ArraySrc{ina}, outa, na,
           (unsigned long long *)scra, tota, ArraySrc{inb}, outb, nb, (unsigned long long *)scrb, totb, (int32_t)ta);
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
