// The reference's secondary seams on the device (seams.py): one interface
// operator application S p from stored flux-basis blocks (basis_apply,
// reference interface.py:238-247). The batched sweeps apply S inside their
// CG kernels; this is the single-vector form a caller of the seam uses.
#include "mfb_common.cuh"

namespace {

// rows[dof_ptr[i] + r] = sum_c B_i[r][c] p[dof_map[dof_ptr[i] + c]]: one CTA
// per subdomain, one thread per block row (columns in block order)
__global__ void basis_rows_kernel(const int *__restrict__ ndof, const int *__restrict__ dof_ptr,
                                  const int *__restrict__ dof_map,
                                  const long long *__restrict__ blk_base,
                                  const double *__restrict__ blocks, const double *__restrict__ p,
                                  double *__restrict__ rows) {
    const int i = blockIdx.x, nd = ndof[i], o = dof_ptr[i];
    const double *Bt = blocks + blk_base[i];          // column-major: Bt[c * nd + r]
    for (int r = threadIdx.x; r < nd; r += blockDim.x) {
        double acc = 0.0;
        for (int c = 0; c < nd; ++c) acc += Bt[(long long)c * nd + r] * p[dof_map[o + c]];
        rows[o + r] = acc;
    }
}

// out[d] = 0 + row of the lower subdomain + row of the upper one (basis_apply
// scatters the subdomains in ascending sid order into a zero vector)
__global__ void basis_scatter_kernel(int n_lambda, const int4 *__restrict__ sides,
                                     const int *__restrict__ dof_ptr,
                                     const double *__restrict__ rows, double *__restrict__ out) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= n_lambda) return;
    const int4 s = sides[d];
    double v = 0.0 + rows[dof_ptr[s.x] + s.y];
    if (s.z >= 0) v = v + rows[dof_ptr[s.z] + s.w];
    out[d] = v;
}

}  // namespace

extern "C" int mfb_basis_apply(int n_lambda, int n_sub, const int *ndof, const int *dof_ptr,
                               const int *dof_map, const int *sides, const long long *blk_base,
                               const double *blocks, const double *p, double *rows, double *out,
                               void *stream) {
    if (n_lambda < 0 || n_sub < 0) return MFB_ERR_ARG;
    if (n_lambda == 0 || n_sub == 0) return MFB_OK;
    cudaStream_t st = mfb_stream(stream);
    basis_rows_kernel<<<n_sub, 64, 0, st>>>(ndof, dof_ptr, dof_map, blk_base, blocks, p, rows);
    MFB_CHECK_LAUNCH();
    basis_scatter_kernel<<<(n_lambda + 255) / 256, 256, 0, st>>>(
        n_lambda, reinterpret_cast<const int4 *>(sides), dof_ptr, rows, out);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}
