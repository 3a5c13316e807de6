// Micro-benchmark of the band panel factorization (factor_publish) on one
// CTA: python-free, build with
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DMFB_PROFILE \
//        -I include -I paper_1802_06263_b200/csrc tools/factor_bench.cu -o tools/factor_bench
#include "../paper_1802_06263_b200/csrc/mfb_band.cu"
#include <cstdio>
#include <vector>
#include <random>

template <int NT>
__global__ void fb_kernel(const double *AB0, double *AB, long long nab, int n, int kl, int ku,
                          int ldab, double *slot, unsigned int *ready, long long *out, int reps) {
    constexpr int NW = NT / 32, NB = BAND_NB;
    __shared__ double s_cand[2 * NW * NB], s_fin[4 * NB];
    __shared__ unsigned long long red_k[2 * NW];
    __shared__ int s_fail;
    long long tot = 0;
    for (int r = 0; r < reps; ++r) {
        for (long long t = threadIdx.x; t < nab; t += NT) AB[t] = AB0[t];
        __syncthreads();
        long long t0 = clock64();
        factor_publish<NT, 1>(AB, n, kl, ku, ldab, 0, slot, slot + (kl + 16) * 16 + 32, ready,
                              s_cand, s_fin, red_k, &s_fail);
        __syncthreads();
        tot += clock64() - t0;
    }
    if (threadIdx.x == 0) { out[0] = tot / reps; out[1] = s_fail; }
}

int main(int argc, char **argv) {
    const int kl = argc > 1 ? atoi(argv[1]) : 152, ku = kl, n = 2 * kl + 64;
    const int ldab = 2 * kl + ku + 1;
    const long long nab = (long long)ldab * n;
    std::vector<double> h(nab);
    std::mt19937_64 g(7);
    std::uniform_real_distribution<double> U(-1, 1);
    for (auto &x : h) x = U(g);
    double *AB0, *AB, *slot;
    unsigned int *ready;
    long long *out;
    cudaMalloc(&AB0, nab * 8);
    cudaMalloc(&AB, nab * 8);
    cudaMalloc(&slot, (size_t)(kl + 16) * 16 * 8 + 1024);
    cudaMalloc(&ready, 4);
    cudaMallocManaged(&out, 16);
    cudaMemcpy(AB0, h.data(), nab * 8, cudaMemcpyHostToDevice);
    const int reps = argc > 2 ? atoi(argv[2]) : 20;
    fb_kernel<512><<<1, 512>>>(AB0, AB, nab, n, kl, ku, ldab, slot, ready, out, reps);
    cudaDeviceSynchronize();
    unsigned long long prof[16] = {0};
#ifdef MFB_PROFILE
    cudaMemcpyFromSymbol(prof, g_bprof, sizeof(prof));
#endif
    printf("finalize: bar %.0f unscale %.0f slot %.0f moves %.0f sync %.0f\n", prof[1] / (double)reps,
           prof[2] / (double)reps, prof[3] / (double)reps, prof[4] / (double)reps, prof[14] / (double)reps);
    printf("kl %d nr %d: factor %lld cycles/call (fail %lld); per call: load %.0f columns %.0f finalize+publish %.0f fence %.0f  err=%s\n",
           kl, kl + 16, out[0], out[1], prof[12] / (double)reps, prof[13] / (double)reps, prof[14] / (double)reps,
           prof[15] / (double)reps, cudaGetErrorString(cudaGetLastError()));
#ifdef MFB_FTS
    long long ts[128];
    cudaMemcpyFromSymbol(ts, g_fts, sizeof(ts));
    for (int c = 0; c < 16; ++c) {
        printf("col %2d:", c);
        for (int k = 1; k < 6; ++k) printf(" %5lld", ts[c * 8 + k] - ts[c * 8 + k - 1]);
        if (c < 15) printf("  -> next %5lld", ts[(c + 1) * 8] - ts[c * 8 + 5]);
        printf("\n");
    }
    long long t2[16 * 16 * 8];
    cudaMemcpyFromSymbol(t2, g_fts2, sizeof(t2));
    long long base = t2[0];
    for (int w = 0; w < 6; ++w) {
        printf("warp %d col 3..5 marks (rel):", w);
        for (int c = 3; c < 6; ++c) {
            printf(" |");
            for (int k = 0; k < 6; ++k) printf(" %6lld", t2[(w * 16 + c) * 8 + k] - base);
        }
        printf("\n");
    }
#endif
    return 0;
}
