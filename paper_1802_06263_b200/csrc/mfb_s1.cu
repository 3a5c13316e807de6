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
                  double *__restrict__ Rout, long long ldr) {
    extern __shared__ double b[];                // n + nb
    __shared__ double red[4];
    __shared__ double s_part[8 * S1_NB];
    __shared__ double s_mu[S1_MAX_NB], s_cr[S1_MAX_NB];
    const int item = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
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
#if defined(S1_STOP) && S1_STOP == 1
    return;
#endif
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
        if (tid == 0) {
            for (int c = 0; c < pnb; ++c) {
                const int p = piv[j0 + c];
                if (p != c) {
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
        for (int i = S1_NB + tid; i < nr; i += S1_NT) {
            const double *li = Lk + (long long)i * S1_NB;
            double a0 = 0.0, a1 = 0.0;
            for (int c = 0; c < pnb; c += 2) {
                a0 = fma(li[c], b[j0 + c], a0);
                if (c + 1 < pnb) a1 = fma(li[c + 1], b[j0 + c + 1], a1);
            }
            b[j0 + i] -= a0 + a1;
        }
        __syncthreads();
    }
#if defined(S1_STOP) && S1_STOP == 2
    return;
#endif
    // ---- backward: b_blk -= U(blk, right) x, x_blk = U11^-1 b_blk -----------
    for (int k = nblk - 1; k >= 0; --k) {
        const int j0 = k * S1_NB, pnb = min(S1_NB, n - j0);
        const int c0 = j0 + pnb, c1 = min(n, j0 + S1_NB + kl + ku);
        const int r = tid & (S1_NB - 1), part = tid >> 4;       // 8 parts
        double acc = 0.0;
        if (r < pnb)
            for (int col = c0 + part; col < c1; col += 8)
                if (col - (j0 + r) <= kl + ku)
                    acc = fma(AB[bidx1(j0 + r, col, kl, ku, ldab)], b[col], acc);
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
#if defined(S1_STOP) && S1_STOP == 3
    return;
#endif
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

}  // namespace

extern "C" int mfb_systems_apply(const MfbPattern *pats, int n_items, const int *item_sys,
                                 const int *sys_pat, const double *work,
                                 const long long *sys_woff, const double *V, long long ldv,
                                 double *X, long long ldx, double *R, long long ldr,
                                 int max_n, void *stream) {
    if (n_items < 0 || max_n < 0) return MFB_ERR_ARG;
    if (n_items == 0) return MFB_OK;
    const size_t smem = (size_t)(max_n + S1_MAX_NB) * sizeof(double);
    if (smem > 200 * 1024) return MFB_ERR_SMEM;
    if (cudaFuncSetAttribute(band_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return MFB_ERR_SMEM;
    band_apply_kernel<<<n_items, S1_NT, smem, mfb_stream(stream)>>>(
        pats, item_sys, sys_pat, work, sys_woff, V, ldv, X, ldx, R, ldr);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}
