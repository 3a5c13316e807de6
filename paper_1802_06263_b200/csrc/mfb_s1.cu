// Solves with stored banded factors: the star solve of Method S1 (the
// reference's matrix-free interface operator, interface.py:180-194).
//
// The multipliers come from the per-panel copies the factorization keeps
// (rows by final position within the panel; the band itself cannot hold
// the multipliers of rows a later swap of the same panel moved more than kl
// below their column).
//
// For each item (system s, coefficient vector v of its N_dof mortar dofs):
//   x = S_s^-1 (Q_s v)            (star_data -> solve_star, problem.py:114-130,
//                                  darcy.py:195-207 / stokes.py:363-385)
//   r = Q_s^T x                   (side_functionals, problem.py:132-148)
// with the factors mfb_systems_solve left in the system's work buffer (LU of
// the band in gbtrf layout with per-panel pivot positions, the inverses of
// the diagonal U blocks) and, for Stokes systems with a rigid-body kernel,
// the same projection the factorization's own solves use (section 1b / 4 of
// mfb_band.cu): mu = (CC^T)^-1 C r, K_II x~ = (r - C^T mu)_I, x~_J = 0,
// x = x~ - C^T (CC^T)^-1 C x~. Q carries the reference's signs so that
// B = Q^T S^-1 Q is the flux basis (the same Q as the factorization's rhs).
//
// One CTA per item: the forward sweep applies each panel's recorded swaps,
// its unit lower L11 (one warp, 16 dependent steps) and its L21 block; the
// backward sweep subtracts the U block right of each diagonal block and
// applies the stored inverse of the diagonal block. Both are chains of n/16
// steps per item -- latency bound; the many items of an S1 iteration (every
// subdomain of every point in flight) run concurrently.
#include "mfb_common.cuh"

namespace {

constexpr int S1_NT = 128;
constexpr int S1_NB = 16;
constexpr int S1_MAX_NB = 8;
constexpr int S1_SLOTS = 17;     // BAND_GROUP_MAX + 1 publication slots (mfb_band.cu)

__device__ __forceinline__ long long bidx1(int i, int k, int kl, int ku, int ldab) {
    return (long long)k * ldab + (kl + ku + i - k);
}

__device__ __forceinline__ double block_sum128(double v, double *red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    return (red[0] + red[1]) + (red[2] + red[3]);
}

__global__ void __launch_bounds__(S1_NT)
band_apply_kernel(const MfbPattern *__restrict__ pats, const int *__restrict__ item_sys,
                  const int *__restrict__ sys_pat, const double *__restrict__ work,
                  const long long *__restrict__ sys_woff, const double *__restrict__ V,
                  long long ldv, double *__restrict__ Xout, long long ldx,
                  double *__restrict__ Rout, long long ldr, const int *__restrict__ item_live,
                  const int *__restrict__ item_list) {
    extern __shared__ double b[];                // n + nb
    __shared__ double red[4];
    __shared__ double s_part[8 * S1_NB];
    __shared__ double s_mu[S1_MAX_NB], s_cr[S1_MAX_NB];
    const int item = item_list ? item_list[blockIdx.x] : blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (item_live && !item_live[item]) return;        // its CG point has finished
    const int s = item_sys[item];
    const MfbPattern P = pats[sys_pat[s]];
    const int n = P.n, kl = P.kl, ku = P.ku, ldab = P.ldab, nb = P.nb, nd = P.ndof;
    // the work layout of mfb_systems_solve (band_solve_kernel)
    const double *AB = work + sys_woff[s];
    const long long ny = (long long)n * (nd + 1);
    const double *Y = AB + (long long)ldab * n;
    const double *slots = Y + ny + (((long long)ldab * n + ny) & 1);
    const long long SLOT = (long long)(kl + S1_NB) * S1_NB + 48;
    const double *udinv = slots + S1_SLOTS * SLOT;
    const double *u11inv =
        udinv + n + ((reinterpret_cast<uintptr_t>(udinv + n) & 15) ? 1 : 0);
    const int nblk = (n + S1_NB - 1) / S1_NB;
    const int *piv = reinterpret_cast<const int *>(u11inv + (long long)S1_NB * S1_NB * nblk);
    const double *Lpan = reinterpret_cast<const double *>(piv) + ((n + 1) / 2 + 1);
    const double *v = V + (long long)item * ldv;

    // ---- b = Q v (Q in CSC; a column's rows are distinct) ------------------
    for (int i = tid; i < n + nb; i += S1_NT) b[i] = 0.0;
    __syncthreads();
    for (int a = 0; a < nd; ++a) {
        const double va = v[a];
        for (int q = P.q_ptr[a] + tid; q < P.q_ptr[a + 1]; q += S1_NT)
            b[P.q_row[q]] += P.q_val[q] * va;
        __syncthreads();
    }
    // ---- rigid-body kernel: b_I -= C_I^T (CC^T)^-1 C b -------------------
    if (nb > 0) {
        for (int a = 0; a < nb; ++a) {
            double acc = 0.0;
            for (int i = tid; i < n; i += S1_NT) acc += P.E[(long long)i * nb + a] * b[i];
            acc = block_sum128(acc, red);
            if (tid == 0) s_cr[a] = acc;
        }
        __syncthreads();
        if (tid == 0) {
            double cr[S1_MAX_NB];
            for (int a = 0; a < nb; ++a) {
                double t = s_cr[a];
                for (int c = 0; c < nb; ++c) t += P.G[a * nb + c] * b[n + c];
                cr[a] = t;
            }
            for (int a = 0; a < nb; ++a) {
                double t = 0.0;
                for (int c = 0; c < nb; ++c) t += P.G[(nb + a) * nb + c] * cr[c];
                s_mu[a] = t;
            }
        }
        __syncthreads();
        for (int i = tid; i < n; i += S1_NT) {
            double t = b[i];
            for (int a = 0; a < nb; ++a) t -= P.E[(long long)i * nb + a] * s_mu[a];
            b[i] = t;
        }
        __syncthreads();
    }
    // ---- forward: per panel, its swaps, L11 (unit lower), then L21 ----------
    for (int k = 0; k < nblk; ++k) {
        const int j0 = k * S1_NB, pnb = min(S1_NB, n - j0);
        const int nr = min(n, j0 + pnb + kl) - j0;
        if (wid == 0) {         // the panel's pivots loaded at once, swapped in order
            const int pv = lane < pnb ? piv[j0 + lane] : lane;
            for (int c = 0; c < pnb; ++c) {
                const int p = __shfl_sync(0xffffffffu, pv, c);
                if (lane == 0 && p != c) {
                    const double t = b[j0 + c];
                    b[j0 + c] = b[j0 + p];
                    b[j0 + p] = t;
                }
            }
        }
        __syncthreads();
        const double *Lk = Lpan + (long long)k * (kl + S1_NB) * S1_NB;   // [row pos][c]
        if (wid == 0) {
            const int r = lane;
            double br = r < pnb ? b[j0 + r] : 0.0;
            double lr[S1_NB];
#pragma unroll
            for (int c = 0; c < S1_NB; ++c) lr[c] = (r < pnb && c < r) ? Lk[r * S1_NB + c] : 0.0;
#pragma unroll
            for (int c = 0; c < S1_NB - 1; ++c) {
                const double bc = __shfl_sync(0xffffffffu, br, c);
                if (r > c) br = fma(-lr[c], bc, br);
            }
            if (r < pnb) b[j0 + r] = br;
        }
        __syncthreads();
        // L21: a half-warp per row (16 lanes = the panel's 16 columns), so
        // every load instruction reads whole 128-byte rows -- no reliance on
        // L1 hits between the 16 column loads of a row; four row pairs per
        // warp in flight, then 16-lane shuffle sums
        {
            const int c = lane & 15, half = lane >> 4;
            const double bc = c < pnb ? b[j0 + c] : 0.0;
            constexpr int NW = S1_NT / 32, STEP = 2 * NW;
            for (int base = S1_NB + 2 * wid + half; base - half < nr; base += 4 * STEP) {
                double v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = base + u * STEP;
                    v[u] = (i < nr && c < pnb) ? Lk[(long long)i * S1_NB + c] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    double t = v[u] * bc;
                    t += __shfl_xor_sync(0xffffffffu, t, 8);
                    t += __shfl_xor_sync(0xffffffffu, t, 4);
                    t += __shfl_xor_sync(0xffffffffu, t, 2);
                    t += __shfl_xor_sync(0xffffffffu, t, 1);
                    const int i = base + u * STEP;
                    if (c == 0 && i < nr) b[j0 + i] -= t;
                }
            }
        }
        __syncthreads();
    }
    // ---- backward: b_blk -= U(blk, right) x, x_blk = U11^-1 b_blk -----------
    for (int k = nblk - 1; k >= 0; --k) {
        const int j0 = k * S1_NB, pnb = min(S1_NB, n - j0);
        const int c0 = j0 + pnb, c1 = min(n, j0 + S1_NB + kl + ku);
        const int r = tid & (S1_NB - 1), part = tid >> 4;       // 8 parts
        double acc = 0.0;
        if (r < pnb) {
            // columns of row j0+r inside the band: col - (j0+r) <= kl+ku;
            // four independent chains keep four loads in flight
            const int lim = min(c1, j0 + r + kl + ku + 1);
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            int col = c0 + part;
            for (; col + 24 < lim; col += 32) {
                a0 = fma(AB[bidx1(j0 + r, col, kl, ku, ldab)], b[col], a0);
                a1 = fma(AB[bidx1(j0 + r, col + 8, kl, ku, ldab)], b[col + 8], a1);
                a2 = fma(AB[bidx1(j0 + r, col + 16, kl, ku, ldab)], b[col + 16], a2);
                a3 = fma(AB[bidx1(j0 + r, col + 24, kl, ku, ldab)], b[col + 24], a3);
            }
            for (; col < lim; col += 8) a0 = fma(AB[bidx1(j0 + r, col, kl, ku, ldab)], b[col], a0);
            acc = (a0 + a1) + (a2 + a3);
        }
        s_part[part * S1_NB + r] = acc;
        __syncthreads();
        if (tid < S1_NB) {
            double t = 0.0;
            for (int q = 0; q < 8; ++q) t += s_part[q * S1_NB + tid];
            s_part[tid] = tid < pnb ? b[j0 + tid] - t : 0.0;   // part 0 row reused: y
        }
        __syncthreads();
        if (tid < S1_NB) {
            const double *ui = u11inv + (long long)k * S1_NB * S1_NB + tid * S1_NB;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
            for (int c = 0; c < S1_NB; c += 4) {
                a0 = fma(ui[c], s_part[c], a0);
                a1 = fma(ui[c + 1], s_part[c + 1], a1);
                a2 = fma(ui[c + 2], s_part[c + 2], a2);
                a3 = fma(ui[c + 3], s_part[c + 3], a3);
            }
            if (tid < pnb) b[j0 + tid] = (a0 + a1) + (a2 + a3);
        }
        __syncthreads();
    }
    // ---- rigid-body kernel: x = x~ - C^T (CC^T)^-1 C x~, x~_J = 0 -----------
    if (nb > 0) {
        for (int a = 0; a < nb; ++a) {
            double acc = 0.0;
            for (int i = tid; i < n; i += S1_NT) acc += P.E[(long long)i * nb + a] * b[i];
            acc = block_sum128(acc, red);
            if (tid == 0) s_cr[a] = acc;
        }
        __syncthreads();
        if (tid < nb) {
            double t = 0.0;
            for (int c = 0; c < nb; ++c) t += P.G[(nb + tid) * nb + c] * s_cr[c];
            s_mu[tid] = t;                                     // alpha
        }
        __syncthreads();
        for (int i = tid; i < n; i += S1_NT) {
            double t = b[i];
            for (int a = 0; a < nb; ++a) t -= P.E[(long long)i * nb + a] * s_mu[a];
            b[i] = t;
        }
        if (tid < nb) {
            double t = 0.0;
            for (int a = 0; a < nb; ++a) t -= P.G[a * nb + tid] * s_mu[a];
            b[n + tid] = t;
        }
        __syncthreads();
    }
    // ---- outputs: x and the readout Q^T x --------------------------------
    if (Xout)
        for (int i = tid; i < n + nb; i += S1_NT) Xout[(long long)item * ldx + i] = b[i];
    if (Rout) {
        for (int a = wid; a < nd; a += S1_NT / 32) {
            double acc = 0.0;
            for (int q = P.q_ptr[a] + lane; q < P.q_ptr[a + 1]; q += 32)
                acc = fma(P.q_val[q], b[P.q_row[q]], acc);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) Rout[(long long)item * ldr + a] = acc;
        }
    }
}

// ---------------------------------------------------------------------------
// Method S1's interface CG (cg_solve, interface.py:107-139, with
// direct_apply's matrix-free operator): every collocation point of the sweep
// iterates in lock step, one CTA per point. Iteration = one apply launch
// (the star solves of every live (point, subdomain) item) + one step launch
// (the CG update of every running point). sides[4d..4d+3] = (i, a_i, j, a_j):
// mortar dof d is local dof a_i of subdomain i and a_j of j (j < 0: one
// side). Item of (point pt, subdomain s) = pt * n_sub + s.
// scal[2pt] = r.r of the current residual, scal[2pt+1] = ||g||.
constexpr int S1_CG_NT = 256;
constexpr int S1_RUNNING = 4;

__device__ __forceinline__ void s1_write_items(const double *__restrict__ src, int n_lambda,
                                               const int *__restrict__ sides, int pt, int n_sub,
                                               double *__restrict__ V, long long ldv) {
    const long long base = (long long)pt * n_sub;
    for (int d = threadIdx.x; d < n_lambda; d += S1_CG_NT) {
        const int4 sd = reinterpret_cast<const int4 *>(sides)[d];
        const double v = src[d];
        V[(base + sd.x) * ldv + sd.y] = v;
        if (sd.z >= 0) V[(base + sd.z) * ldv + sd.w] = v;
    }
}

__device__ __forceinline__ void s1_finish(int pt, int n_sub, int *item_live, int *n_running) {
    for (int s = threadIdx.x; s < n_sub; s += S1_CG_NT) item_live[(long long)pt * n_sub + s] = 0;
    if (threadIdx.x == 0) atomicSub(n_running, 1);
}

__global__ void __launch_bounds__(S1_CG_NT)
s1_cg_begin_kernel(int n_lambda, int n_sub, const int *__restrict__ sides,
                   const double *__restrict__ hbar, const long long *__restrict__ item_hoff,
                   double *__restrict__ x, double *__restrict__ r, double *__restrict__ p,
                   double *__restrict__ scal, int *__restrict__ iters, int *__restrict__ status,
                   double *__restrict__ V, long long ldv, int *__restrict__ item_live,
                   int *__restrict__ n_running, double *__restrict__ g_out) {
    __shared__ double red[S1_CG_NT / 32];
    const int pt = blockIdx.x;
    const long long o = (long long)pt * n_lambda, base = (long long)pt * n_sub;
    // g = jump of the bar solutions (compute_rhs, interface.py:166-177)
    double part = 0.0;
    for (int d = threadIdx.x; d < n_lambda; d += S1_CG_NT) {
        const int4 sd = reinterpret_cast<const int4 *>(sides)[d];
        double g = hbar[item_hoff[base + sd.x] + sd.y];
        if (sd.z >= 0) g += hbar[item_hoff[base + sd.z] + sd.w];
        r[o + d] = g;
        p[o + d] = g;
        x[o + d] = 0.0;
        if (g_out) g_out[o + d] = g;
        part += g * g;
    }
    const double rr = block_sum<S1_CG_NT>(part, red);
    const double gnorm = sqrt(rr);
    if (threadIdx.x == 0) {
        scal[2 * pt] = rr;
        scal[2 * pt + 1] = gnorm;
        iters[pt] = 0;
        status[pt] = gnorm == 0.0 ? MFB_CG_ZERO_RHS : S1_RUNNING;
        if (gnorm != 0.0) atomicAdd(n_running, 1);
    }
    for (int s = threadIdx.x; s < n_sub; s += S1_CG_NT) item_live[base + s] = gnorm != 0.0;
    // the first apply's input: p = g (x = 0 for a zero right-hand side)
    s1_write_items(p + o, n_lambda, sides, pt, n_sub, V, ldv);
}

__global__ void __launch_bounds__(S1_CG_NT)
s1_cg_step_kernel(int n_lambda, int n_sub, const int *__restrict__ sides,
                  const double *__restrict__ R, long long ldr, double tol, int max_iter,
                  double *__restrict__ x, double *__restrict__ r, double *__restrict__ p,
                  double *__restrict__ scal, int *__restrict__ iters, int *__restrict__ status,
                  double *__restrict__ res_hist, int hist_cap, double *__restrict__ V,
                  long long ldv, int *__restrict__ item_live, int *__restrict__ n_running) {
    extern __shared__ double Sp[];                 // n_lambda
    __shared__ double red[S1_CG_NT / 32];
    const int pt = blockIdx.x, tid = threadIdx.x;
    if (status[pt] != S1_RUNNING) return;
    const long long o = (long long)pt * n_lambda, base = (long long)pt * n_sub;
    double *xp = x + o, *rp = r + o, *pp = p + o;
    const int it = iters[pt] + 1;
    const double rr = scal[2 * pt], gnorm = scal[2 * pt + 1];
    // Sp = -jump(side functionals of the star solves): each dof adds its
    // two sides' readouts
    double part = 0.0;
    for (int d = tid; d < n_lambda; d += S1_CG_NT) {
        const int4 sd = reinterpret_cast<const int4 *>(sides)[d];
        double v = R[(base + sd.x) * ldr + sd.y];
        if (sd.z >= 0) v += R[(base + sd.z) * ldr + sd.w];
        Sp[d] = v;
        part += pp[d] * v;
    }
    const double pSp = block_sum<S1_CG_NT>(part, red);
    if (!(pSp > 0.0)) {
        if (tid == 0) { status[pt] = MFB_CG_NOT_SPD; iters[pt] = it; }
        s1_write_items(xp, n_lambda, sides, pt, n_sub, V, ldv);
        s1_finish(pt, n_sub, item_live, n_running);
        return;
    }
    const double a = rr / pSp;
    part = 0.0;
    for (int d = tid; d < n_lambda; d += S1_CG_NT) {
        xp[d] += a * pp[d];
        const double rd = rp[d] - a * Sp[d];
        rp[d] = rd;
        part += rd * rd;
    }
    const double rr_new = block_sum<S1_CG_NT>(part, red);
    const double rn = sqrt(rr_new);
    if (tid == 0 && it - 1 < hist_cap) res_hist[(long long)pt * hist_cap + it - 1] = rn / gnorm;
    const bool conv = rn <= tol * gnorm;
    if (conv || it >= max_iter) {
        if (tid == 0) { status[pt] = conv ? MFB_CG_CONVERGED : MFB_CG_MAX_ITER; iters[pt] = it; }
        __syncthreads();                               // x complete before the item copy
        s1_write_items(xp, n_lambda, sides, pt, n_sub, V, ldv);   // the recovery's input
        s1_finish(pt, n_sub, item_live, n_running);
        return;
    }
    const double beta = rr_new / rr;
    for (int d = tid; d < n_lambda; d += S1_CG_NT) pp[d] = rp[d] + beta * pp[d];
    if (tid == 0) { scal[2 * pt] = rr_new; iters[pt] = it; }
    __syncthreads();
    s1_write_items(pp, n_lambda, sides, pt, n_sub, V, ldv);
}

// fields of (point, subdomain) item t: F[item_foff[t] + f] =
// Fb_sys[f] - (P x)_f -- recover_fields + postprocess (interface.py:250-260,
// problem.py:150-158): the bar fields plus the star solution's. Q carries
// the readout's sign (B = Q^T S^-1 Q = -restrict(...), interface.py:230),
// so x = S^-1 Q v is minus the reference's star solution.
__global__ void __launch_bounds__(128)
s1_fields_kernel(const MfbPattern *__restrict__ pats, const int *__restrict__ item_sys,
                 const int *__restrict__ sys_pat, const double *__restrict__ X, long long ldx,
                 const double *__restrict__ Fb, const long long *__restrict__ sys_fboff,
                 double *__restrict__ F, const long long *__restrict__ item_foff) {
    const int t = blockIdx.x, s = item_sys[t];
    const MfbPattern P = pats[sys_pat[s]];
    const double *xt = X + (long long)t * ldx;
    for (int f = threadIdx.x; f < P.nfield; f += blockDim.x) {
        double v = 0.0;
        for (int q = P.p_ptr[f]; q < P.p_ptr[f + 1]; ++q) v += P.p_val[q] * xt[P.p_col[q]];
        F[item_foff[t] + f] = Fb[sys_fboff[s] + f] - v;
    }
}

}  // namespace

extern "C" int mfb_systems_apply(const MfbPattern *pats, int n_items, const int *item_sys,
                                 const int *sys_pat, const double *work,
                                 const long long *sys_woff, const double *V, long long ldv,
                                 double *X, long long ldx, double *R, long long ldr,
                                 int max_n, const int *item_live, const int *item_list,
                                 void *stream) {
    if (n_items < 0 || max_n < 0) return MFB_ERR_ARG;
    if (n_items == 0) return MFB_OK;
    const size_t smem = (size_t)(max_n + S1_MAX_NB) * sizeof(double);
    if (smem > 200 * 1024) return MFB_ERR_SMEM;
    if (cudaFuncSetAttribute(band_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return MFB_ERR_SMEM;
    band_apply_kernel<<<n_items, S1_NT, smem, mfb_stream(stream)>>>(
        pats, item_sys, sys_pat, work, sys_woff, V, ldv, X, ldx, R, ldr, item_live, item_list);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}

extern "C" int mfb_s1_cg_begin(int n_lambda, int n_pts, int n_sub, const int *sides,
                               const double *hbar, const long long *item_hoff, double *x,
                               double *r, double *p, double *scal, int *iters, int *status,
                               double *V, long long ldv, int *item_live, int *n_running,
                               double *g_out, void *stream) {
    if (n_lambda <= 0 || n_pts < 0 || n_sub <= 0) return MFB_ERR_ARG;
    if (n_pts == 0) return MFB_OK;
    cudaStream_t st = mfb_stream(stream);
    if (cudaMemsetAsync(n_running, 0, sizeof(int), st) != cudaSuccess) return MFB_ERR_LAUNCH;
    s1_cg_begin_kernel<<<n_pts, S1_CG_NT, 0, st>>>(n_lambda, n_sub, sides, hbar, item_hoff, x,
                                                   r, p, scal, iters, status, V, ldv,
                                                   item_live, n_running, g_out);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}

extern "C" int mfb_s1_cg_step(int n_lambda, int n_pts, int n_sub, const int *sides,
                              const double *R, long long ldr, double tol, int max_iter,
                              double *x, double *r, double *p, double *scal, int *iters,
                              int *status, double *res_hist, int hist_cap, double *V,
                              long long ldv, int *item_live, int *n_running, void *stream) {
    if (n_lambda <= 0 || n_pts < 0 || n_sub <= 0 || hist_cap < 1) return MFB_ERR_ARG;
    if (n_pts == 0) return MFB_OK;
    const size_t smem = (size_t)n_lambda * sizeof(double);
    if (smem > 200 * 1024) return MFB_ERR_SMEM;
    if (cudaFuncSetAttribute(s1_cg_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return MFB_ERR_SMEM;
    s1_cg_step_kernel<<<n_pts, S1_CG_NT, smem, mfb_stream(stream)>>>(
        n_lambda, n_sub, sides, R, ldr, tol, max_iter, x, r, p, scal, iters, status, res_hist,
        hist_cap, V, ldv, item_live, n_running);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}

extern "C" int mfb_s1_fields(const MfbPattern *pats, int n_items, const int *item_sys,
                             const int *sys_pat, const double *X, long long ldx,
                             const double *Fb, const long long *sys_fboff, double *F,
                             const long long *item_foff, void *stream) {
    if (n_items < 0) return MFB_ERR_ARG;
    if (n_items == 0) return MFB_OK;
    s1_fields_kernel<<<n_items, 128, 0, mfb_stream(stream)>>>(pats, item_sys, sys_pat, X, ldx,
                                                             Fb, sys_fboff, F, item_foff);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}
