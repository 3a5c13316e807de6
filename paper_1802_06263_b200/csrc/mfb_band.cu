// Batched subdomain solves for the flux basis (generic path).
//
// One CTA owns one (subdomain, local realization) system and does, without
// leaving the kernel:
//   1. assembly of the interior matrix from the subdomain's parametrised
//      entry list and this realization's K (reference darcy.py:114-137,
//      stokes.py:220-274 -- the matrix the reference hands to SuperLU);
//   2. banded LU with partial pivoting (LAPACK gbtf2 semantics, U grows to
//      kl+ku superdiagonals) while the same row operations are applied to
//      all right-hand sides: the border columns E, the N_dof mortar columns
//      Q (reference: one star solve per mortar dof, interface.py:218-235)
//      and the bar column (interface.py:166-177);
//   3. back substitution for every column;
//   4. the dense border (Stokes rigid-body pinning, stokes.py:276-298):
//      Schur complement Sigma = G - E^T K_II^-1 E, solved by Gaussian
//      elimination with partial pivoting, then the interior correction.
// The band lives in global memory (L2-resident per CTA); the pivot row,
// multipliers and the pivot rhs row are staged in shared memory so that
// every update element costs one global read-modify-write.
#include "mfb_common.cuh"

namespace {

constexpr int MAX_NB = 8;
constexpr int MAX_NCY = 160;

__device__ __forceinline__ long long bidx(int i, int k, int kl, int ku, int ldab) {
    return (long long)k * ldab + (kl + ku + i - k);
}

template <int NT>
__global__ void __launch_bounds__(NT)
band_solve_kernel(const MfbPattern *__restrict__ pats, const int *__restrict__ sys_pat,
                  const double *__restrict__ Kbuf, const long long *__restrict__ sys_koff,
                  double *__restrict__ work, const long long *__restrict__ sys_woff,
                  double *__restrict__ Xout, const long long *__restrict__ sys_xoff,
                  int *__restrict__ info) {
    extern __shared__ double smem[];
    __shared__ double red_v[NT / 32];
    __shared__ int red_i[NT / 32];
    __shared__ int s_piv;
    __shared__ double s_pivval;
    __shared__ double s_bord[MAX_NB * MAX_NCY];
    __shared__ double s_z[MAX_NB * MAX_NCY];
    __shared__ int s_flag;

    const int s = blockIdx.x;
    const MfbPattern P = pats[sys_pat[s]];
    const double *K = Kbuf + sys_koff[s];
    const int n = P.n, kl = P.kl, ku = P.ku, ldab = P.ldab, nb = P.nb;
    const int nrhs = P.ndof + 1;
    const int ncy = nb + nrhs;
    double *AB = work + sys_woff[s];
    double *Y = AB + (long long)ldab * n;
    double *s_l = smem;                 // kl multipliers
    double *s_u = s_l + kl + 1;         // kl+ku+1 pivot-row entries
    double *s_y = s_u + kl + ku + 2;    // ncy pivot rhs row
    const int tid = threadIdx.x;

    // ---- 1. assembly ---------------------------------------------------
    const long long nab = (long long)ldab * n, ny = (long long)n * ncy;
    for (long long t = tid; t < nab + ny; t += NT) AB[t] = 0.0;
    __syncthreads();
    for (int e = tid; e < P.n_entries; e += NT) {
        double v = 0.0;
        for (int t = P.e_tptr[e]; t < P.e_tptr[e + 1]; ++t)
            v += mfb_term(P.t_kind[t], P.t_c[t], K, P.t_k[t]);
        AB[bidx(P.e_row[e], P.e_col[e], kl, ku, ldab)] = v;
    }
    for (long long t = tid; t < (long long)n * nb; t += NT)
        Y[(t / nb) * ncy + (t % nb)] = P.E[t];
    for (int d = 0; d < P.ndof; ++d)
        for (int q = P.q_ptr[d] + tid; q < P.q_ptr[d + 1]; q += NT) {
            int r = P.q_row[q];
            if (r < n) Y[(long long)r * ncy + nb + d] = P.q_val[q];
        }
    for (int i = tid; i < n; i += NT) Y[(long long)i * ncy + nb + P.ndof] = P.bar_const[i];
    __syncthreads();
    for (int b = tid; b < P.n_bar_rows; b += NT) {
        int r = P.b_row[b];
        if (r >= n) continue;
        double v = 0.0;
        for (int t = P.b_tptr[b]; t < P.b_tptr[b + 1]; ++t)
            v += mfb_term(P.bt_kind[t], P.bt_c[t], K, P.bt_k[t]);
        Y[(long long)r * ncy + nb + P.ndof] += v;
    }
    __syncthreads();

    // ---- 2. banded LU with partial pivoting + forward elimination --------
    for (int j = 0; j < n; ++j) {
        const int iend = min(n - 1, j + kl);
        const int kend = min(n - 1, j + kl + ku);
        double best = -1.0;
        int bi = j;
        for (int i = j + tid; i <= iend; i += NT) {
            double a = fabs(AB[bidx(i, j, kl, ku, ldab)]);
            if (a > best) { best = a; bi = i; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            double ov = __shfl_down_sync(0xffffffffu, best, o);
            int oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
        }
        if ((tid & 31) == 0) { red_v[tid >> 5] = best; red_i[tid >> 5] = bi; }
        __syncthreads();
        if (tid == 0) {
            double bv = red_v[0];
            int bx = red_i[0];
            for (int w = 1; w < NT / 32; ++w)
                if (red_v[w] > bv || (red_v[w] == bv && red_i[w] < bx)) { bv = red_v[w]; bx = red_i[w]; }
            s_piv = bx;
            s_pivval = AB[bidx(bx, j, kl, ku, ldab)];
        }
        __syncthreads();
        const int p = s_piv;
        const double piv = s_pivval;
        if (piv == 0.0) {
            if (tid == 0) info[s] = j + 1;
            return;
        }
        // swap rows j <-> p over columns j..kend, stage pivot row and multipliers
        for (int k = j + tid; k <= kend; k += NT) {
            long long aj = bidx(j, k, kl, ku, ldab), ap = bidx(p, k, kl, ku, ldab);
            double vj = AB[aj], vp = AB[ap];
            if (p != j) { AB[aj] = vp; AB[ap] = vj; }
            s_u[k - j] = vp;
        }
        for (int c = tid; c < ncy; c += NT) {
            long long yj = (long long)j * ncy + c, yp = (long long)p * ncy + c;
            double vj = Y[yj], vp = Y[yp];
            if (p != j) { Y[yj] = vp; Y[yp] = vj; }
            s_y[c] = vp;
        }
        __syncthreads();
        // column j after the swap: row p holds the old row-j value
        for (int i = j + 1 + tid; i <= iend; i += NT)
            s_l[i - j - 1] = AB[bidx(i, j, kl, ku, ldab)] / piv;
        __syncthreads();
        const int nr = iend - j, nc = kend - j;
        for (int t = tid; t < nr * nc; t += NT) {
            const int ii = t % nr, kk = t / nr;
            const int i = j + 1 + ii, k = j + 1 + kk;
            AB[bidx(i, k, kl, ku, ldab)] -= s_l[ii] * s_u[kk + 1];
        }
        for (int t = tid; t < nr * ncy; t += NT) {
            const int ii = t / ncy, c = t % ncy;
            Y[(long long)(j + 1 + ii) * ncy + c] -= s_l[ii] * s_y[c];
        }
        __syncthreads();
    }

    // ---- 3. back substitution with U (kl+ku superdiagonals) -------------
    for (int j = n - 1; j >= 0; --j) {
        const double ujj = AB[bidx(j, j, kl, ku, ldab)];
        for (int c = tid; c < ncy; c += NT) {
            double y = Y[(long long)j * ncy + c] / ujj;
            Y[(long long)j * ncy + c] = y;
            s_y[c] = y;
        }
        __syncthreads();
        const int i0 = max(0, j - kl - ku);
        const int nr = j - i0;
        for (int t = tid; t < nr * ncy; t += NT) {
            const int ii = t / ncy, c = t % ncy;
            const int i = i0 + ii;
            Y[(long long)i * ncy + c] -= AB[bidx(i, j, kl, ku, ldab)] * s_y[c];
        }
        __syncthreads();
    }

    // ---- 4. border ------------------------------------------------------
    double *X = Xout + sys_xoff[s];
    if (nb > 0) {
        const int lane = tid & 31, wid = tid >> 5;
        for (int pr = wid; pr < nb * ncy; pr += NT / 32) {
            const int a = pr / ncy, col = pr % ncy;
            double acc = 0.0;
            for (int i = lane; i < n; i += 32)
                acc += P.E[(long long)i * nb + a] * Y[(long long)i * ncy + col];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
            if (lane == 0) s_bord[pr] = acc;
        }
        __syncthreads();
        if (tid == 0) {
            // Sigma (nb x nb) in s_bord[a*ncy + b], rhs (nb x nrhs) in s_z
            for (int a = 0; a < nb; ++a) {
                for (int b = 0; b < nb; ++b)
                    s_bord[a * ncy + b] = P.G[a * nb + b] - s_bord[a * ncy + b];
                for (int c = 0; c < nrhs; ++c) s_z[a * nrhs + c] = -s_bord[a * ncy + nb + c];
                s_z[a * nrhs + P.ndof] += P.bar_const[n + a];
            }
            for (int d = 0; d < P.ndof; ++d)
                for (int q = P.q_ptr[d]; q < P.q_ptr[d + 1]; ++q)
                    if (P.q_row[q] >= n) s_z[(P.q_row[q] - n) * nrhs + d] += P.q_val[q];
            for (int b = 0; b < P.n_bar_rows; ++b) {
                int r = P.b_row[b];
                if (r < n) continue;
                double v = 0.0;
                for (int t = P.b_tptr[b]; t < P.b_tptr[b + 1]; ++t)
                    v += mfb_term(P.bt_kind[t], P.bt_c[t], K, P.bt_k[t]);
                s_z[(r - n) * nrhs + P.ndof] += v;
            }
            // Gaussian elimination with partial pivoting on Sigma
            int ok = 1;
            for (int c = 0; c < nb && ok; ++c) {
                int pr = c;
                for (int r = c + 1; r < nb; ++r)
                    if (fabs(s_bord[r * ncy + c]) > fabs(s_bord[pr * ncy + c])) pr = r;
                if (s_bord[pr * ncy + c] == 0.0) { ok = 0; break; }
                if (pr != c) {
                    for (int b = 0; b < nb; ++b) {
                        double t0 = s_bord[c * ncy + b];
                        s_bord[c * ncy + b] = s_bord[pr * ncy + b];
                        s_bord[pr * ncy + b] = t0;
                    }
                    for (int b = 0; b < nrhs; ++b) {
                        double t0 = s_z[c * nrhs + b];
                        s_z[c * nrhs + b] = s_z[pr * nrhs + b];
                        s_z[pr * nrhs + b] = t0;
                    }
                }
                for (int r = c + 1; r < nb; ++r) {
                    double l = s_bord[r * ncy + c] / s_bord[c * ncy + c];
                    for (int b = c; b < nb; ++b) s_bord[r * ncy + b] -= l * s_bord[c * ncy + b];
                    for (int b = 0; b < nrhs; ++b) s_z[r * nrhs + b] -= l * s_z[c * nrhs + b];
                }
            }
            if (ok) {
                for (int c = nb - 1; c >= 0; --c)
                    for (int b = 0; b < nrhs; ++b) {
                        double v = s_z[c * nrhs + b];
                        for (int r = c + 1; r < nb; ++r) v -= s_bord[c * ncy + r] * s_z[r * nrhs + b];
                        s_z[c * nrhs + b] = v / s_bord[c * ncy + c];
                    }
            }
            s_flag = ok;
        }
        __syncthreads();
        if (!s_flag) {
            if (tid == 0) info[s] = -1;
            return;
        }
        for (long long t = tid; t < (long long)n * nrhs; t += NT) {
            const int i = (int)(t / nrhs), c = (int)(t % nrhs);
            double v = Y[(long long)i * ncy + nb + c];
            for (int a = 0; a < nb; ++a) v -= Y[(long long)i * ncy + a] * s_z[a * nrhs + c];
            X[t] = v;
        }
        for (int t = tid; t < nb * nrhs; t += NT) X[(long long)n * nrhs + t] = s_z[t];
    } else {
        for (long long t = tid; t < (long long)n * nrhs; t += NT) X[t] = Y[t];
    }
    if (tid == 0) info[s] = 0;
}

template <int NT>
__global__ void __launch_bounds__(NT)
extract_kernel(const MfbPattern *__restrict__ pats, const int *__restrict__ sys_pat,
               const double *__restrict__ Xall, const long long *__restrict__ sys_xoff,
               double *blocks, const long long *sys_boff, double *hbar,
               const long long *sys_hoff, double *M, const long long *sys_moff,
               double *Fb, const long long *sys_fboff) {
    const int s = blockIdx.x;
    const MfbPattern P = pats[sys_pat[s]];
    const double *X = Xall + sys_xoff[s];
    const int nd = P.ndof, nrhs = nd + 1;
    if (blocks || hbar) {
        for (int t = threadIdx.x; t < nd * nrhs; t += NT) {
            const int r = t / nrhs, c = t % nrhs;
            double v = 0.0;
            for (int q = P.q_ptr[r]; q < P.q_ptr[r + 1]; ++q)
                v += P.q_val[q] * X[(long long)P.q_row[q] * nrhs + c];
            if (c < nd) {
                if (blocks) blocks[sys_boff[s] + (long long)c * nd + r] = v;
            } else if (hbar) {
                hbar[sys_hoff[s] + r] = v + P.h_lift[r];
            }
        }
    }
    if (M || Fb) {
        for (long long t = threadIdx.x; t < (long long)P.nfield * nrhs; t += NT) {
            const int f = (int)(t / nrhs), c = (int)(t % nrhs);
            double v = 0.0;
            for (int q = P.p_ptr[f]; q < P.p_ptr[f + 1]; ++q)
                v += P.p_val[q] * X[(long long)P.p_col[q] * nrhs + c];
            if (c < nd) {
                if (M) M[sys_moff[s] + (long long)f * nd + c] = v;
            } else if (Fb) {
                Fb[sys_fboff[s] + f] = v + P.f_lift[f];
            }
        }
    }
}

}  // namespace

extern "C" int mfb_systems_solve(const MfbPattern *pats, int n_sys, const int *sys_pat,
                                 const double *Kbuf, const long long *sys_koff,
                                 double *work, const long long *sys_woff, double *X,
                                 const long long *sys_xoff, int *info, int threads,
                                 int smem_doubles, void *stream) {
    if (n_sys <= 0) return n_sys == 0 ? MFB_OK : MFB_ERR_ARG;
    // dynamic smem: multipliers + pivot row + rhs row of the widest band
    const int nt = threads;
    size_t smem = (size_t)smem_doubles * sizeof(double);
    cudaStream_t st = mfb_stream(stream);
    switch (nt) {
        case 128:
            if (smem > 48 * 1024 && cudaFuncSetAttribute(band_solve_kernel<128>,
                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                return MFB_ERR_SMEM;
            band_solve_kernel<128><<<n_sys, 128, smem, st>>>(pats, sys_pat, Kbuf, sys_koff,
                                                             work, sys_woff, X, sys_xoff, info);
            break;
        case 256:
            if (smem > 48 * 1024 && cudaFuncSetAttribute(band_solve_kernel<256>,
                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                return MFB_ERR_SMEM;
            band_solve_kernel<256><<<n_sys, 256, smem, st>>>(pats, sys_pat, Kbuf, sys_koff,
                                                             work, sys_woff, X, sys_xoff, info);
            break;
        case 512:
            if (smem > 48 * 1024 && cudaFuncSetAttribute(band_solve_kernel<512>,
                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                return MFB_ERR_SMEM;
            band_solve_kernel<512><<<n_sys, 512, smem, st>>>(pats, sys_pat, Kbuf, sys_koff,
                                                             work, sys_woff, X, sys_xoff, info);
            break;
        case 1024:
            if (smem > 48 * 1024 && cudaFuncSetAttribute(band_solve_kernel<1024>,
                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                return MFB_ERR_SMEM;
            band_solve_kernel<1024><<<n_sys, 1024, smem, st>>>(pats, sys_pat, Kbuf, sys_koff,
                                                               work, sys_woff, X, sys_xoff, info);
            break;
        default:
            return MFB_ERR_ARG;
    }
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}

extern "C" int mfb_systems_extract(const MfbPattern *pats, int n_sys, const int *sys_pat,
                                   const double *X, const long long *sys_xoff,
                                   double *blocks, const long long *sys_boff,
                                   double *hbar, const long long *sys_hoff, double *M,
                                   const long long *sys_moff, double *Fb,
                                   const long long *sys_fboff, void *stream) {
    if (n_sys <= 0) return n_sys == 0 ? MFB_OK : MFB_ERR_ARG;
    extract_kernel<256><<<n_sys, 256, 0, mfb_stream(stream)>>>(
        pats, sys_pat, X, sys_xoff, blocks, sys_boff, hbar, sys_hoff, M, sys_moff, Fb,
        sys_fboff);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}
