// Batched interface CG: every collocation point of the S3 sweep at once.
//
// One CTA owns one collocation point k and runs the reference's plain CG
// (interface.py:107-139) to completion with all four vectors (x, r, p, Sp)
// resident in shared memory. The right-hand side is gathered from the
// precomputed per-(subdomain, local realization) bar jumps (the reference's
// compute_rhs, interface.py:166-177 + mortar.jump) and S p is applied from
// the flux-basis pool exactly as basis_apply does (interface.py:238-247):
// Sp[dofs_i] += B_{i, loc_i(k)} p[dofs_i]. Each mortar dof receives exactly
// two contributions (its two sides), accumulated with shared-memory atomics
// into a zeroed vector: 0 + a + b is order independent in IEEE arithmetic,
// so the result is deterministic. Dot products use a fixed reduction tree.
// Stopping test ||r|| <= tol ||g|| after the update, breakdown on p.Sp <= 0,
// x0 = 0 and the zero-rhs early exit follow the reference line by line.
#include "mfb_common.cuh"

namespace {

constexpr int CG_NT = 256;

__global__ void __launch_bounds__(CG_NT)
cg_kernel(int n_lambda, int n_sub, const int *__restrict__ ndof,
          const int *__restrict__ dof_ptr, const int *__restrict__ dof_map,
          const int *__restrict__ region, const long long *__restrict__ blk_base,
          const long long *__restrict__ h_base, const int *__restrict__ local_idx,
          int n_real, const double *__restrict__ blocks, const double *__restrict__ hbar,
          int k0, double tol, int max_iter, double *__restrict__ lam_out,
          int *__restrict__ iters_out, int *__restrict__ status_out,
          double *__restrict__ res_hist, int hist_cap, double *__restrict__ g_out) {
    extern __shared__ double sm[];
    __shared__ double red[CG_NT / 32];
    double *x = sm;
    double *r = x + n_lambda;
    double *p = r + n_lambda;
    double *Sp = p + n_lambda;
    const int pt = blockIdx.x;
    const int k = k0 + pt;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

    // ---- rhs g = sum_i scatter(h_{i, loc_i(k)}) --------------------------
    for (int d = tid; d < n_lambda; d += CG_NT) { x[d] = 0.0; r[d] = 0.0; }
    __syncthreads();
    for (int i = wid; i < n_sub; i += CG_NT / 32) {
        const int nd = ndof[i];
        const int loc = region[i] < 0 ? 0 : local_idx[(long long)region[i] * n_real + k];
        const double *h = hbar + h_base[i] + (long long)loc * nd;
        const int *dm = dof_map + dof_ptr[i];
        for (int a = lane; a < nd; a += 32) atomicAdd(&r[dm[a]], h[a]);
    }
    __syncthreads();
    double *lam = lam_out + (long long)pt * n_lambda;
    if (g_out)
        for (int d = tid; d < n_lambda; d += CG_NT) g_out[(long long)pt * n_lambda + d] = r[d];
    double part = 0.0;
    for (int d = tid; d < n_lambda; d += CG_NT) {
        p[d] = r[d];
        part += r[d] * r[d];
    }
    double rr = block_sum<CG_NT>(part, red);
    const double gnorm = sqrt(rr);
    if (gnorm == 0.0) {
        for (int d = tid; d < n_lambda; d += CG_NT) lam[d] = 0.0;
        if (tid == 0) { iters_out[pt] = 0; status_out[pt] = MFB_CG_ZERO_RHS; }
        return;
    }
    double *hist = res_hist + (long long)pt * hist_cap;
    int status = MFB_CG_MAX_ITER, it_done = max_iter;
    for (int it = 1; it <= max_iter; ++it) {
        // ---- Sp = sum_i scatter(B_i p_i) ----------------------------------
        for (int d = tid; d < n_lambda; d += CG_NT) Sp[d] = 0.0;
        __syncthreads();
        for (int i = wid; i < n_sub; i += CG_NT / 32) {
            const int nd = ndof[i];
            const int loc = region[i] < 0 ? 0 : local_idx[(long long)region[i] * n_real + k];
            const double *B = blocks + blk_base[i] + (long long)loc * nd * nd;
            const int *dm = dof_map + dof_ptr[i];
            for (int a = lane; a < nd; a += 32) {
                double acc = 0.0;
                for (int c = 0; c < nd; ++c) acc = fma(B[(long long)c * nd + a], p[dm[c]], acc);
                atomicAdd(&Sp[dm[a]], acc);
            }
        }
        __syncthreads();
        part = 0.0;
        for (int d = tid; d < n_lambda; d += CG_NT) part += p[d] * Sp[d];
        const double pSp = block_sum<CG_NT>(part, red);
        if (!(pSp > 0.0)) {
            status = MFB_CG_NOT_SPD;
            it_done = it;
            break;
        }
        const double a = rr / pSp;
        part = 0.0;
        for (int d = tid; d < n_lambda; d += CG_NT) {
            x[d] += a * p[d];
            const double rd = r[d] - a * Sp[d];
            r[d] = rd;
            part += rd * rd;
        }
        const double rr_new = block_sum<CG_NT>(part, red);
        const double rn = sqrt(rr_new);
        if (tid == 0 && it <= hist_cap) hist[it - 1] = rn / gnorm;
        if (rn <= tol * gnorm) {
            status = MFB_CG_CONVERGED;
            it_done = it;
            break;
        }
        const double beta = rr_new / rr;
        for (int d = tid; d < n_lambda; d += CG_NT) p[d] = r[d] + beta * p[d];
        rr = rr_new;
        __syncthreads();
    }
    for (int d = tid; d < n_lambda; d += CG_NT) lam[d] = x[d];
    if (tid == 0) { iters_out[pt] = it_done; status_out[pt] = status; }
}

}  // namespace

extern "C" int mfb_cg_batched(int n_lambda, int n_sub, const int *ndof, const int *dof_ptr,
                              const int *dof_map, const int *region,
                              const long long *blk_base, const long long *h_base,
                              const int *local_idx, int n_real, const double *blocks,
                              const double *hbar, int k0, int n_pts, double tol,
                              int max_iter, double *lam, int *iters, int *status,
                              double *res_hist, int hist_cap, double *g, void *stream) {
    if (n_pts <= 0) return n_pts == 0 ? MFB_OK : MFB_ERR_ARG;
    size_t smem = (size_t)4 * n_lambda * sizeof(double);
    if (smem > 227 * 1024) return MFB_ERR_SMEM;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(cg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return MFB_ERR_SMEM;
    cg_kernel<<<n_pts, CG_NT, smem, mfb_stream(stream)>>>(
        n_lambda, n_sub, ndof, dof_ptr, dof_map, region, blk_base, h_base, local_idx, n_real,
        blocks, hbar, k0, tol, max_iter, lam, iters, status, res_hist, hist_cap, g);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}
