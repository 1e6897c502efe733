// micro-benchmark: cost of cooperative_groups grid.sync() and of a custom atomic barrier on B200
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_sync(int n, int *x) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < n; ++i) {
        if (threadIdx.x == 0 && blockIdx.x == 0) x[0] += 1;
        g.sync();
    }
}

// sense-reversing barrier on one global counter
__device__ __forceinline__ void bar(unsigned *count, unsigned *gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g = *(volatile unsigned *)gen;
        __threadfence();
        if (atomicAdd(count, 1) == nblocks - 1) {
            *count = 0;
            __threadfence();
            atomicAdd(gen, 1);
        } else {
            while (*(volatile unsigned *)gen == g) {}
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void k_bar(int n, unsigned *cnt, unsigned *gen) {
    for (int i = 0; i < n; ++i) bar(cnt, gen, gridDim.x);
}

__global__ void k_empty() {}

int main() {
    int *x;
    unsigned *c;
    cudaMalloc(&x, 64);
    cudaMalloc(&c, 64);
    cudaMemset(x, 0, 64);
    cudaMemset(c, 0, 64);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int blocks : {16, 148, 296, 592}) {
        for (int n : {0, 100}) {
            void *args[] = {&n, &x};
            cudaLaunchCooperativeKernel((void *)k_sync, blocks, 256, args, 0, 0);
            cudaEventRecord(a);
            for (int r = 0; r < 10; ++r) cudaLaunchCooperativeKernel((void *)k_sync, blocks, 256, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("grid.sync blocks=%d n=%d: %.2f us per launch\n", blocks, n, ms * 100);
            unsigned *cnt = c, *gen = c + 16;
            cudaEventRecord(a);
            for (int r = 0; r < 10; ++r) k_bar<<<blocks, 256>>>(n, cnt, gen);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("atomic bar blocks=%d n=%d: %.2f us per launch\n", blocks, n, ms * 100);
        }
    }
    // back-to-back empty kernels in a graph
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 100; ++i) k_empty<<<148, 256, 0, s>>>();
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("graph of 100 empty kernels: %.2f us per kernel\n", ms * 10);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
