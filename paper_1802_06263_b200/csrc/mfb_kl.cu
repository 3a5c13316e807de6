// KL permeability kernel: all local realizations of one KL region at once.
//
// K[l, c] = exp(mean[c] + sum_j Phi[c, j] xi[l, j])   (reference
// random_field.py:232-243: evaluate_log = mean + modes @ xi, then np.exp).
// Phi and xi are tiny (n_term <= ~10); each thread owns one (l, c) output,
// reads its Phi row (cached in L1, shared by all l) and the l-th xi row from
// shared memory, and writes K coalesced along c. Write-bound: 8 B per output.
#include "mfb_common.cuh"

namespace {
constexpr int KL_MAX_TERM = 64;

__global__ void kl_realize_kernel(const double *__restrict__ phi,
                                  const double *__restrict__ mean, int n_cells,
                                  int n_term, const double *__restrict__ xi,
                                  int n_loc, double *__restrict__ K, long long ld) {
    __shared__ double s_xi[KL_MAX_TERM];
    const int l = blockIdx.y;
    if (threadIdx.x < n_term) s_xi[threadIdx.x] = xi[(long long)l * n_term + threadIdx.x];
    __syncthreads();
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n_cells;
         c += gridDim.x * blockDim.x) {
        const double *row = phi + (long long)c * n_term;
        double dot = 0.0;
        for (int j = 0; j < n_term; ++j) dot = fma(row[j], s_xi[j], dot);
        K[(long long)l * ld + c] = exp(mean[c] + dot);
    }
}
// Every KL table of a sweep in one launch: blockIdx.z = table, blockIdx.y =
// row (row 0 of a table is its mean-field row, written to dst0), grid-stride
// over the cells.
__global__ void kl_batched_kernel(const MfbKlTable *__restrict__ tabs, double *__restrict__ K) {
    __shared__ double s_xi[KL_MAX_TERM];
    const MfbKlTable T = tabs[blockIdx.z];
    const int l = blockIdx.y;
    if (l > T.n_rows) return;
    if (threadIdx.x < T.n_term) s_xi[threadIdx.x] = T.xi[(long long)l * T.n_term + threadIdx.x];
    __syncthreads();
    double *out = l == 0 ? K + T.dst0 : K + T.dst + (long long)(l - 1) * T.ld;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < T.n_cells;
         c += gridDim.x * blockDim.x) {
        const double *row = T.phi + (long long)c * T.n_term;
        double dot = 0.0;
        for (int j = 0; j < T.n_term; ++j) dot = fma(row[j], s_xi[j], dot);
        out[c] = exp(T.mean[c] + dot);
    }
}
}  // namespace

extern "C" int mfb_kl_realize_ld(const double *phi, const double *mean, int n_cells,
                                 int n_term, const double *xi, int n_loc, double *K,
                                 long long ld, void *stream) {
    if (n_cells < 0 || n_loc < 0 || n_term < 0 || n_term > KL_MAX_TERM || ld < n_cells)
        return MFB_ERR_ARG;
    if (n_cells == 0 || n_loc == 0) return MFB_OK;
    const int nt = 256;
    int bx = (n_cells + nt - 1) / nt;
    if (bx > 64) bx = 64;
    dim3 grid(bx, n_loc);
    kl_realize_kernel<<<grid, nt, 0, mfb_stream(stream)>>>(phi, mean, n_cells, n_term,
                                                          xi, n_loc, K, ld);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}

extern "C" int mfb_kl_realize(const double *phi, const double *mean, int n_cells,
                              int n_term, const double *xi, int n_loc, double *K,
                              void *stream) {
    return mfb_kl_realize_ld(phi, mean, n_cells, n_term, xi, n_loc, K, n_cells, stream);
}

extern "C" int mfb_kl_realize_batched(int n_tables, const MfbKlTable *tables, int max_rows,
                                      int max_cells, double *K, void *stream) {
    if (n_tables < 0 || max_rows < 0 || max_cells < 0) return MFB_ERR_ARG;
    if (n_tables == 0) return MFB_OK;
    const int nt = 256;
    int bx = (max_cells + nt - 1) / nt;
    if (bx > 64) bx = 64;
    if (bx < 1) bx = 1;
    dim3 grid(bx, max_rows + 1, n_tables);
    kl_batched_kernel<<<grid, nt, 0, mfb_stream(stream)>>>(tables, K);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}
