// micro-benchmark: HBM bandwidth on B200 for read-only, write-only, copy (1:1) and 1:2 / 1:3
// read:write float4 streams (grid = 148 SMs x 8 blocks, grid-stride), 1 GiB per array.
// Used to bound the write-heavy last-level CC face kernel (~0.35 GB read, ~0.74 GB written).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/micro/bw tools/micro/bw.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_read(const float4 *a, size_t n, float *sink) {
    float acc = 0.f;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        float4 v = __ldg(a + i);
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 12345.f) *sink = acc;
}
__global__ void k_write(float4 *b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = make_float4(1.f, 2.f, 3.f, (float)i);
}
__global__ void k_copy(const float4 *a, float4 *b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = __ldg(a + i);
}
// read n, write W * n (W output arrays)
template <int W>
__global__ void k_rw(const float4 *a, float4 *b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        float4 v = __ldg(a + i);
#pragma unroll
        for (int w = 0; w < W; ++w) b[w * n + i] = make_float4(v.x + w, v.y, v.z, v.w);
    }
}

int main() {
    const size_t bytes = 1ull << 30, n = bytes / 16;
    float4 *a, *b;
    float *sink;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, 3 * bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(a, 0, bytes);
    cudaMemset(b, 0, 3 * bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = 148 * 8, blk = 256;
    auto time = [&](const char *name, double gb, auto fn) {
        float best = 1e30f;
        for (int r = 0; r < 10; ++r) {
            cudaEventRecord(e0);
            fn();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r > 0 && ms < best) best = ms;
        }
        printf("%-12s %8.3f ms  %7.1f GB/s\n", name, best, gb / (best * 1e-3));
    };
    const double G = bytes / 1e9;
    time("read", G, [&] { k_read<<<grid, blk>>>(a, n, sink); });
    time("write", G, [&] { k_write<<<grid, blk>>>(b, n); });
    time("copy 1:1", 2 * G, [&] { k_copy<<<grid, blk>>>(a, b, n); });
    time("r:w 1:2", 3 * G, [&] { k_rw<2><<<grid, blk>>>(a, b, n); });
    time("r:w 1:3", 4 * G, [&] { k_rw<3><<<grid, blk>>>(a, b, n); });
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
