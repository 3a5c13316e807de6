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

// same, for a runtime block size (multiple of 32); red holds blockDim/32 doubles
__device__ __forceinline__ double block_sum_dyn(double v, double *red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double tot = 0.0;
    for (int w = 0; w < nw; ++w) tot += red[w];
    return tot;
}

// block sum with alternating halves of red (2 x blockDim/32): one barrier;
// the caller guarantees a barrier between a thread's last write of the
// summed data and the call, which the barrier inside provides for the next
// call's buffer reuse
__device__ __forceinline__ double block_sum_alt(double v, double *red2, int &buf) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    double *red = red2 + buf * 32;
    buf ^= 1;
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double t0 = 0.0, t1 = 0.0;
    int w = 0;
    for (; w + 2 <= nw; w += 2) { t0 += red[w]; t1 += red[w + 1]; }
    if (w < nw) t0 += red[w];
    return t0 + t1;
}

__device__ __forceinline__ double mfb_term(int kind, double c, const double *K, int k) {
    if (kind == MFB_TERM_INV_K) return c / K[k];
    if (kind == MFB_TERM_INV_SQRT_K) return c / sqrt(K[k]);
    return c;
}
