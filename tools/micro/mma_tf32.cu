// Legacy-path TF32 tensor throughput on this GPU: mma.sync.m16n8k8 (tf32 in, fp32 accumulate),
// 8 independent accumulators per warp, vs plain FP32 FFMA.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_mma(float *out, int iters) {
    uint32_t a0 = __float_as_uint(1.0f + threadIdx.x), a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 ^ 5, b1 = a0 ^ 7;
    float c[8][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[k][0]), "+f"(c[k][1]), "+f"(c[k][2]), "+f"(c[k][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma(float *out, int iters) {
    float c[16];
    for (int k = 0; k < 16; ++k) c[k] = threadIdx.x + k;
    const float a = 1.0001f, b = 0.5f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int k = 0; k < 16; ++k) c[k] = fmaf(c[k], a, b);
    }
    float s = 0;
    for (int k = 0; k < 16; ++k) s += c[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float *out;
    cudaMalloc(&out, 148 * 8 * 256 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096, blocks = 148 * 8, threads = 256;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k_mma<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 16 * 8 * 8 * 8.0 * iters * (blocks * threads / 32);
        printf("mma.sync tf32 m16n8k8: %.1f TFLOP/s (%.3f ms)\n", flops / (ms * 1e9), ms);
        cudaEventRecord(e0);
        k_ffma<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double f2 = 2.0 * 8 * 16 * (double)iters * blocks * threads;
        printf("ffma fp32: %.1f TFLOP/s (%.3f ms)\n", f2 / (ms * 1e9), ms);
    }
    return 0;
}
