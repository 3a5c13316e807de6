// Shared device helpers for the MFB kernels (sm_100a, FP64 throughout).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "mfb.h"

#define MFB_CHECK_LAUNCH()                                   \
    do {                                                     \
        cudaError_t _e = cudaGetLastError();                 \
        if (_e != cudaSuccess) return MFB_ERR_LAUNCH;        \
    } while (0)

static inline cudaStream_t mfb_stream(void *s) { return (cudaStream_t)s; }

// deterministic block-wide sum: fixed warp-shuffle tree then fixed order over warps
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) tot += red[w];
    return tot;
}

__device__ __forceinline__ double mfb_term(int kind, double c, const double *K, int k) {
    if (kind == MFB_TERM_INV_K) return c / K[k];
    if (kind == MFB_TERM_INV_SQRT_K) return c / sqrt(K[k]);
    return c;
}
