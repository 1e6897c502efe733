// summary.cu -- per-frame result summaries for the sharded frame batches (the
// multi-GPU config-5 job gathers 32 B per frame over NCCL instead of the 153 MB frames).
//
// For frame b of a batch [B][V][3] (fp32, frame-major) the summary record is eight 32-bit words:
//   lo.xyz, hi.xyz  -- the bounding box (fp32 min / max per coordinate)
//   sum (uint64)    -- sum_i bits(x_i) * (2 i + 1) mod 2^64 over the 3V floats of the frame
// Min, max and a wrapping integer sum are exact and order-independent, so the record is
// deterministic whatever the block schedule.  Three launches: init, reduce, decode.
#include <algorithm>

#include "alsub.h"
#include "internal.h"

namespace alsub {
alsub_status set_error(alsub_status st, const char *msg);  // api.cu (thread-local last error)

__global__ void __launch_bounds__(kThreads) k_summary_init(SummaryRec *out, int32_t nb) {
    ALSUB_GRID_WAIT();
    const int32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    SummaryRec r;
    for (int c = 0; c < 3; ++c) {
        r.lo[c] = INT32_MAX;
        r.hi[c] = INT32_MIN;
    }
    r.sum = 0ull;
    out[b] = r;
}

// fold float i (coordinate c) into the running record
ALSUB_D void fold(int32_t (&lo)[3], int32_t (&hi)[3], unsigned long long &sum, int c, int64_t i, float v) {
    lo[c] = min(lo[c], f2ord(v));
    hi[c] = max(hi[c], f2ord(v));
    sum += (unsigned long long)(uint32_t)__float_as_int(v) * (unsigned long long)(2 * i + 1);
}

// grid (blocks per frame, frames).  VEC: the frame starts 16-B aligned, so each step takes four
// vertices = 48 B as three float4 loads (float 12 q + k has coordinate k mod 3); the V mod 4
// tail vertices and the !VEC case take three scalar loads per vertex.
template <bool VEC>
__global__ void __launch_bounds__(kThreads) k_summary_reduce(const float *__restrict__ frames, int64_t nv,
                                                             SummaryRec *out) {
    ALSUB_GRID_WAIT();
    const float *x = frames + (int64_t)blockIdx.y * 3 * nv;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    // min / max in the ordered-int domain (a total order: -0 < +0, NaNs beyond the infinities)
    int32_t lo[3], hi[3];
    for (int c = 0; c < 3; ++c) {
        lo[c] = INT32_MAX;
        hi[c] = INT32_MIN;
    }
    unsigned long long sum = 0ull;
    int64_t v0 = 0;
    if constexpr (VEC) {
        const int64_t nq = nv / 4;
        const float4 *x4 = reinterpret_cast<const float4 *>(x);
        for (int64_t q = tid; q < nq; q += nth) {
            const float4 a = __ldg(x4 + 3 * q), b = __ldg(x4 + 3 * q + 1), d = __ldg(x4 + 3 * q + 2);
            const float e[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, d.x, d.y, d.z, d.w};
#pragma unroll
            for (int k = 0; k < 12; ++k) fold(lo, hi, sum, k % 3, 12 * q + k, e[k]);
        }
        v0 = 4 * nq;
    }
    for (int64_t v = v0 + tid; v < nv; v += nth) {
        const float e0 = __ldg(x + 3 * v), e1 = __ldg(x + 3 * v + 1), e2 = __ldg(x + 3 * v + 2);
        fold(lo, hi, sum, 0, 3 * v, e0);
        fold(lo, hi, sum, 1, 3 * v + 1, e1);
        fold(lo, hi, sum, 2, 3 * v + 2, e2);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        for (int c = 0; c < 3; ++c) {
            lo[c] = min(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
            hi[c] = max(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
        }
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
    }
    if ((threadIdx.x & 31) == 0) {
        SummaryRec *r = out + blockIdx.y;
        for (int c = 0; c < 3; ++c) {
            atomicMin(&r->lo[c], lo[c]);
            atomicMax(&r->hi[c], hi[c]);
        }
        atomicAdd(&r->sum, sum);
    }
}

__global__ void __launch_bounds__(kThreads) k_summary_decode(SummaryRec *out, int32_t nb) {
    ALSUB_GRID_WAIT();
    const int32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    SummaryRec &r = out[b];
    for (int c = 0; c < 3; ++c) {
        r.lo[c] = __float_as_int(ord2f(r.lo[c]));
        r.hi[c] = __float_as_int(ord2f(r.hi[c]));
    }
}

void summary_init(SummaryRec *rec, int32_t nb, cudaStream_t s, Launches &L) {
    if (nb > 0) launch(L, "summary_init", k_summary_init, dim3(grid_for(nb)), dim3(kThreads), 0, s, rec, nb);
}
void summary_decode(SummaryRec *rec, int32_t nb, cudaStream_t s, Launches &L) {
    if (nb > 0) launch(L, "summary_decode", k_summary_decode, dim3(grid_for(nb)), dim3(kThreads), 0, s, rec, nb);
}

}  // namespace alsub

using namespace alsub;

extern "C" alsub_status alsub_frame_summary(const float *frames, int32_t num_frames, int64_t num_verts, void *summary,
                                            void *stream) {
    if (num_frames < 0 || num_verts < 0) return set_error(ALSUB_E_ARG, "negative count");
    if (num_frames == 0) return ALSUB_OK;
    if (!summary || (num_verts > 0 && !frames)) return set_error(ALSUB_E_ARG, "null pointer");
    if (num_frames > 65535) return set_error(ALSUB_E_ARG, "num_frames > 65535 per call");
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, summary) != cudaSuccess || a.type != cudaMemoryTypeDevice ||
        (num_verts > 0 && (cudaPointerGetAttributes(&a, frames) != cudaSuccess || a.type != cudaMemoryTypeDevice))) {
        cudaGetLastError();
        return set_error(ALSUB_E_ARG, "frames and summary must be device pointers");
    }
    cudaStream_t s = (cudaStream_t)stream;
    Launches L;
    SummaryRec *out = reinterpret_cast<SummaryRec *>(summary);
    const unsigned g1 = (unsigned)ceil_div(num_frames, kThreads);
    launch(L, "summary_init", k_summary_init, dim3(g1), dim3(kThreads), 0, s, out, num_frames);
    if (num_verts > 0) {
        // about 8 resident blocks per SM across the whole batch, at least one block per frame
        const int64_t want = std::max<int64_t>(1, (8 * 148 + num_frames - 1) / num_frames);
        const unsigned gx = (unsigned)std::min<int64_t>(want, ceil_div(num_verts, kThreads));
        // float4 path when every frame starts 16-B aligned (base aligned and 12 V % 16 == 0)
        const bool vec = (reinterpret_cast<uintptr_t>(frames) & 15u) == 0 && (num_frames == 1 || num_verts % 4 == 0);
        if (vec)
            launch(L, "summary_reduce", k_summary_reduce<true>, dim3(gx, (unsigned)num_frames), dim3(kThreads), 0, s,
                   frames, num_verts, out);
        else
            launch(L, "summary_reduce", k_summary_reduce<false>, dim3(gx, (unsigned)num_frames), dim3(kThreads), 0, s,
                   frames, num_verts, out);
    }
    launch(L, "summary_decode", k_summary_decode, dim3(g1), dim3(kThreads), 0, s, out, num_frames);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(ALSUB_E_CUDA, cudaGetErrorString(e));
    return ALSUB_OK;
}
