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

#ifdef MFB_PROFILE
__device__ unsigned long long g_bprof[16];
#define BPROF(i)                                                                  \
    do {                                                                          \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                \
            long long _c = clock64();                                             \
            if ((i) > 0) atomicAdd(&g_bprof[(i)], (unsigned long long)(_c - s_bt0)); \
            s_bt0 = _c;                                                           \
        }                                                                         \
    } while (0)
#else
#define BPROF(i) do {} while (0)
#endif

namespace {

constexpr int MAX_NB = 8;
constexpr int MAX_NCY = 160;
constexpr int BAND_NB = 16;

__device__ __forceinline__ long long bidx(int i, int k, int kl, int ku, int ldab) {
    return (long long)k * ldab + (kl + ku + i - k);
}

__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int NT>
__global__ void __launch_bounds__(NT)
band_solve_kernel(const MfbPattern *__restrict__ pats, const int *__restrict__ sys_pat,
                  const double *__restrict__ Kbuf, const long long *__restrict__ sys_koff,
                  double *__restrict__ work, const long long *__restrict__ sys_woff,
                  double *__restrict__ Xout, const long long *__restrict__ sys_xoff,
                  int *__restrict__ info) {
    constexpr int NB = BAND_NB;
    constexpr int PST = NB + 1;          // odd stride: lane-varying rows hit distinct banks
    constexpr int NW = NT / 32;
    extern __shared__ double smem[];
    __shared__ double red_v[NW];
    __shared__ int red_i[NW];
    __shared__ int s_ipiv[NB];
    __shared__ int s_low[NB];
    __shared__ int s_nlow;
    __shared__ double s_u11[NB * NB];
    __shared__ double s_linv[NB * NB];
    __shared__ double s_bord[MAX_NB * MAX_NCY];
    __shared__ double s_z[MAX_NB * MAX_NCY];
    __shared__ int s_flag;
#ifdef MFB_PROFILE
    __shared__ long long s_bt0;
#endif

    const int s = blockIdx.x;
    const MfbPattern P = pats[sys_pat[s]];
    const double *K = Kbuf + sys_koff[s];
    const int n = P.n, kl = P.kl, ku = P.ku, ldab = P.ldab, nb = P.nb;
    const int nrhs = P.ndof + 1;
    const int ncy = nb + nrhs;
    const int UST = kl + ku + 8;
    double *AB = work + sys_woff[s];
    double *Y = AB + (long long)ldab * n;
    double *Pnl = smem;                          // (kl + NB) x PST   panel L | U11
    double *U12s = Pnl + (kl + NB) * PST;        // NB x UST          U12 of the panel
    double *Tmp = U12s + NB * UST;               // NB x UST          staged A12
    double *Ytop = Tmp + NB * UST;               // NB x ncy          rhs rows of the panel
    int *s_perm = reinterpret_cast<int *>(Ytop + NB * ncy);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

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

    if (tid == 0) s_flag = 0;
    __syncthreads();
    // ---- 2. blocked banded LU with partial pivoting (gbtrf) --------------
    for (int j0 = 0; j0 < n; j0 += NB) {
        BPROF(0);
        const int pnb = min(NB, n - j0);
        const int r1 = min(n, j0 + pnb + kl);
        const int nr = r1 - j0;
        const int c0 = j0 + pnb;
        const int c1 = min(n, j0 + pnb + kl + ku);
        const int nc = max(0, c1 - c0);
        // panel columns j0..j0+pnb of rows j0..r1 (zero beyond the band / pnb)
        for (int t = tid; t < nr * NB; t += NT) {
            const int i = t % nr, c = t / nr;
            const int r = j0 + i, col = j0 + c;
            Pnl[i * PST + c] = (c < pnb && r - col <= kl && col - r <= kl + ku)
                                   ? AB[bidx(r, col, kl, ku, ldab)] : 0.0;
        }
        __syncthreads();
        BPROF(1);
        if (tid < 128) {
            // panel LU with partial pivoting on 4 warps (named barrier 2); the
            // pivot candidate of column c+1 is found while column c is applied
            const int pw = tid >> 5;
            double best = -1.0;
            int bi = 0;
            for (int i = tid; i < nr; i += 128) {
                const double a = fabs(Pnl[i * PST]);
                if (a > best) { best = a; bi = i; }
            }
            for (int c = 0; c < pnb; ++c) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const double ov = __shfl_down_sync(0xffffffffu, best, o);
                    const int oi = __shfl_down_sync(0xffffffffu, bi, o);
                    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
                }
                if (lane == 0) { red_v[pw] = best; red_i[pw] = bi; }
                asm volatile("bar.sync 2, 128;" ::: "memory");
                double bv = red_v[0];
                int p = red_i[0];
#pragma unroll
                for (int w = 1; w < 4; ++w)
                    if (red_v[w] > bv || (red_v[w] == bv && red_i[w] < p)) { bv = red_v[w]; p = red_i[w]; }
                if (!(bv > 0.0)) {
                    if (tid == 0) { info[s] = j0 + c + 1; s_flag = -1; }
                    break;
                }
                if (tid == 0) s_ipiv[c] = p;
                if (p != c && tid < NB) {
                    const double t0 = Pnl[c * PST + tid];
                    Pnl[c * PST + tid] = Pnl[p * PST + tid];
                    Pnl[p * PST + tid] = t0;
                }
                asm volatile("bar.sync 2, 128;" ::: "memory");
                const double inv = 1.0 / Pnl[c * PST + c];
                best = -1.0;
                bi = c + 1;
                for (int i = c + 1 + tid; i < nr; i += 128) {
                    const double l = Pnl[i * PST + c] * inv;
                    Pnl[i * PST + c] = l;
                    for (int cc = c + 1; cc < pnb; ++cc) Pnl[i * PST + cc] -= l * Pnl[c * PST + cc];
                    if (c + 1 < pnb) {
                        const double a = fabs(Pnl[i * PST + c + 1]);
                        if (a > best) { best = a; bi = i; }
                    }
                }
            }
        }
        __syncthreads();
        BPROF(2);
        if (s_flag < 0) return;
        // net row permutation of the panel's swaps
        if (tid == 0) {
            for (int i = 0; i < nr; ++i) s_perm[i] = i;
            int nl = 0;
            for (int q = 0; q < pnb; ++q) {
                const int p = s_ipiv[q];
                const int t0 = s_perm[q];
                s_perm[q] = s_perm[p];
                s_perm[p] = t0;
                if (p >= pnb) {
                    bool seen = false;
                    for (int z = 0; z < nl; ++z) seen |= (s_low[z] == p);
                    if (!seen) s_low[nl++] = p;
                }
            }
            s_nlow = nl;
        }
        __syncthreads();
        BPROF(3);
        for (int t = tid; t < nr * pnb; t += NT) {
            const int i = t % nr, c = t / nr;
            const int r = j0 + i, col = j0 + c;
            if (r - col <= kl && col - r <= kl + ku) AB[bidx(r, col, kl, ku, ldab)] = Pnl[i * PST + c];
        }
        // phase A: stage the permuted top rows of every trailing column (Tmp)
        // and the moved lower rows (U12s used as staging); all reads first
        const int nlow = s_nlow;
        const int ncpad = (nc + 7) & ~7;
        for (int t = tid; t < NB * ncpad; t += NT) {
            const int q = t / ncpad, cc = t % ncpad, col = c0 + cc;
            const int src = j0 + (q < pnb ? s_perm[q] : 0);
            const bool vt = q < pnb && cc < nc && col - src <= kl + ku && src - col <= kl;
            const int srl = j0 + (q < nlow ? s_perm[s_low[q]] : 0);
            const bool vl = q < nlow && cc < nc && col - srl <= kl + ku && srl - col <= kl;
            const double x = __ldcg(AB + (vt ? bidx(src, col, kl, ku, ldab) : 0));
            const double y = __ldcg(AB + (vl ? bidx(srl, col, kl, ku, ldab) : 0));
            Tmp[q * UST + cc] = vt ? x : 0.0;
            U12s[q * UST + cc] = vl ? y : 0.0;
        }
        if (tid < NB) {
            // column tid of L11^-1 (unit lower triangular)
            double x[NB];
#pragma unroll
            for (int q = 0; q < NB; ++q) {
                double v = (q == tid) ? 1.0 : 0.0;
#pragma unroll
                for (int qq = 0; qq < q; ++qq) v -= (q < pnb ? Pnl[q * PST + qq] : 0.0) * x[qq];
                x[q] = v;
            }
#pragma unroll
            for (int q = 0; q < NB; ++q) s_linv[q * NB + tid] = x[q];
        }
        __syncthreads();
        for (int t = tid; t < nlow * nc; t += NT) {
            const int z = t / nc, cc = t % nc, col = c0 + cc;
            const int row = j0 + s_low[z];
            if (row - col <= kl) AB[bidx(row, col, kl, ku, ldab)] = U12s[z * UST + cc];
        }
        __syncthreads();
        // U12 = L11^-1 A12 on DMMA; written to the band (top rows) and to U12s
        {
            const int g = lane >> 2, q4 = lane & 3;
            const int tcn = ncpad >> 3;
            for (int t = wid; t < 2 * tcn; t += NW) {
                const int ti = t & 1, tj = t >> 1;
                double d0 = 0.0, d1 = 0.0;
#pragma unroll
                for (int k0 = 0; k0 < NB; k0 += 4) {
                    const double a = s_linv[(ti * 8 + g) * NB + k0 + q4];
                    const double b = Tmp[(k0 + q4) * UST + tj * 8 + g];
                    dmma884(d0, d1, a, b);
                }
                const int q = ti * 8 + g, cc = tj * 8 + 2 * q4;
                U12s[q * UST + cc] = q < pnb ? d0 : 0.0;
                U12s[q * UST + cc + 1] = q < pnb ? d1 : 0.0;
                const int row = j0 + q;
                if (q < pnb && cc < nc && c0 + cc - row <= kl + ku)
                    AB[bidx(row, c0 + cc, kl, ku, ldab)] = d0;
                if (q < pnb && cc + 1 < nc && c0 + cc + 1 - row <= kl + ku)
                    AB[bidx(row, c0 + cc + 1, kl, ku, ldab)] = d1;
            }
        }
        // phase A': right-hand sides -- permute + forward substitution (thread per column)
        for (int cy = tid; cy < ncy; cy += NT) {
            double u[NB], low[NB];
#pragma unroll
            for (int q = 0; q < NB; ++q)
                u[q] = q < pnb ? Y[(long long)(j0 + s_perm[q]) * ncy + cy] : 0.0;
#pragma unroll
            for (int z = 0; z < NB; ++z)
                low[z] = z < nlow ? Y[(long long)(j0 + s_perm[s_low[z]]) * ncy + cy] : 0.0;
#pragma unroll
            for (int z = 0; z < NB; ++z)
                if (z < nlow) Y[(long long)(j0 + s_low[z]) * ncy + cy] = low[z];
#pragma unroll
            for (int q = 1; q < NB; ++q) {
                double v = u[q];
#pragma unroll
                for (int qq = 0; qq < q; ++qq) v -= Pnl[q * PST + qq] * u[qq];
                u[q] = v;
            }
#pragma unroll
            for (int q = 0; q < NB; ++q) {
                if (q < pnb) Y[(long long)(j0 + q) * ncy + cy] = u[q];
                Ytop[q * ncy + cy] = q < pnb ? u[q] : 0.0;
            }
        }
        __syncthreads();
        // phase B: A22 -= L21 U12 on FP64 tensor cores (DMMA 8x8x4 tiles).
        // A warp owns a column tile: its U12 fragments stay in registers while
        // it walks down the row tiles, four tiles in flight at a time.
        {
            const int mrows = nr - pnb;
            const int tr = (mrows + 7) >> 3, tcn = ncpad >> 3;
            const int g = lane >> 2, q4 = lane & 3;
            for (int tj = wid; tj < tcn; tj += NW) {
                double bf[NB / 4];
#pragma unroll
                for (int kk = 0; kk < NB / 4; ++kk) bf[kk] = U12s[(4 * kk + q4) * UST + tj * 8 + g];
                const int ca = c0 + tj * 8 + 2 * q4, cb = ca + 1;
                // band column pointers: element (row, col) = colp[row]
                double *pa = AB + (long long)ca * ldab + (kl + ku - ca);
                double *pb = pa + (ldab - 1);
                const int lima = ca < c1 ? min(r1, ca + kl + 1) : 0;
                const int limb = cb < c1 ? min(r1, cb + kl + 1) : 0;
                const int rbase = j0 + pnb + g;
                for (int tg = 0; tg < tr; tg += 4) {
                    double d0[4], d1[4];
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const int row = rbase + (tg + h) * 8;
                        d0[h] = row < lima ? pa[row] : 0.0;
                        d1[h] = row < limb ? pb[row] : 0.0;
                    }
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const int prow = pnb + (tg + h) * 8 + g;
                        const bool ra = prow < nr;
#pragma unroll
                        for (int kk = 0; kk < NB / 4; ++kk) {
                            const double a = ra ? -Pnl[prow * PST + 4 * kk + q4] : 0.0;
                            dmma884(d0[h], d1[h], a, bf[kk]);
                        }
                    }
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const int row = rbase + (tg + h) * 8;
                        if (row < lima) pa[row] = d0[h];
                        if (row < limb) pb[row] = d1[h];
                    }
                }
            }
        }
        // phase B': rhs rows below the panel, Y -= L21 Ytop (DMMA tiles; a warp
        // owns a row tile and keeps its L21 fragments in registers)
        {
            const int mrows = nr - pnb;
            const int tr = (mrows + 7) >> 3, tcy = (ncy + 7) >> 3;
            const int g = lane >> 2, q4 = lane & 3;
            for (int ti = wid; ti < tr; ti += NW) {
                const int prow = pnb + ti * 8 + g;
                const bool ra = prow < nr;
                double af[NB / 4];
#pragma unroll
                for (int kk = 0; kk < NB / 4; ++kk) af[kk] = ra ? -Pnl[prow * PST + 4 * kk + q4] : 0.0;
                const long long row = j0 + prow;
                for (int tc = 0; tc < tcy; ++tc) {
                    const int ca = tc * 8 + 2 * q4, cb = ca + 1;
                    double d0 = (ra && ca < ncy) ? Y[row * ncy + ca] : 0.0;
                    double d1 = (ra && cb < ncy) ? Y[row * ncy + cb] : 0.0;
#pragma unroll
                    for (int kk = 0; kk < NB / 4; ++kk) {
                        const int cc = tc * 8 + g;
                        const double b = cc < ncy ? Ytop[(4 * kk + q4) * ncy + cc] : 0.0;
                        dmma884(d0, d1, af[kk], b);
                    }
                    if (ra && ca < ncy) Y[row * ncy + ca] = d0;
                    if (ra && cb < ncy) Y[row * ncy + cb] = d1;
                }
            }
        }
        __syncthreads();
        BPROF(5);
    }

    // ---- 3. blocked column-oriented back substitution with U ---------------
    const int last = ((n - 1) / NB) * NB;
    for (int j0 = last; j0 >= 0; j0 -= NB) {
        const int pnb = min(NB, n - j0);
        for (int t = tid; t < NB * NB; t += NT) {
            const int r = t / NB, c = t % NB;
            s_u11[t] = (r < pnb && c < pnb && c >= r) ? AB[bidx(j0 + r, j0 + c, kl, ku, ldab)] : 0.0;
        }
        __syncthreads();
        for (int cy = tid; cy < ncy; cy += NT) {
            double x[NB];
#pragma unroll
            for (int r = NB - 1; r >= 0; --r) {
                if (r >= pnb) { x[r] = 0.0; continue; }
                double v = Y[(long long)(j0 + r) * ncy + cy];
#pragma unroll
                for (int rr = r + 1; rr < NB; ++rr) v -= s_u11[r * NB + rr] * x[rr];
                x[r] = v / s_u11[r * NB + r];
            }
#pragma unroll
            for (int r = 0; r < NB; ++r) {
                if (r < pnb) Y[(long long)(j0 + r) * ncy + cy] = x[r];
                Ytop[r * ncy + cy] = x[r];
            }
        }
        __syncthreads();
        // push the solved panel into the rows above: Y[i] -= U(i, panel) x_panel
        // (DMMA tiles; A = U block straight from the band, B = x from smem)
        {
            const int i0 = max(0, j0 - kl - ku);
            const int mrows = j0 - i0;
            const int tr = (mrows + 7) >> 3, tcy = (ncy + 7) >> 3;
            const int g = lane >> 2, q4 = lane & 3;
            for (int ti = wid; ti < tr; ti += NW) {
                const int i = i0 + ti * 8 + g;
                const bool ri = i < j0;
                double af[NB / 4];
#pragma unroll
                for (int kk = 0; kk < NB / 4; ++kk) {
                    const int k = 4 * kk + q4;
                    af[kk] = (ri && k < pnb && (j0 + k) - i <= kl + ku)
                                 ? -AB[bidx(i, j0 + k, kl, ku, ldab)] : 0.0;
                }
                for (int tc = 0; tc < tcy; ++tc) {
                    const int ca = tc * 8 + 2 * q4, cb = ca + 1;
                    double d0 = (ri && ca < ncy) ? Y[(long long)i * ncy + ca] : 0.0;
                    double d1 = (ri && cb < ncy) ? Y[(long long)i * ncy + cb] : 0.0;
#pragma unroll
                    for (int kk = 0; kk < NB / 4; ++kk) {
                        const int cc = tc * 8 + g;
                        const double b = cc < ncy ? Ytop[(4 * kk + q4) * ncy + cc] : 0.0;
                        dmma884(d0, d1, af[kk], b);
                    }
                    if (ri && ca < ncy) Y[(long long)i * ncy + ca] = d0;
                    if (ri && cb < ncy) Y[(long long)i * ncy + cb] = d1;
                }
            }
        }
        __syncthreads();
    }
    BPROF(7);

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
    // dynamic smem: see Pattern.smem_doubles (discretization.py)
    const int nt = threads;
    size_t smem = (size_t)smem_doubles * sizeof(double);
    cudaStream_t st = mfb_stream(stream);
    switch (nt) {
        case 128:
            if (cudaFuncSetAttribute(band_solve_kernel<128>,
                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                return MFB_ERR_SMEM;
            band_solve_kernel<128><<<n_sys, 128, smem, st>>>(pats, sys_pat, Kbuf, sys_koff,
                                                             work, sys_woff, X, sys_xoff, info);
            break;
        case 256:
            if (cudaFuncSetAttribute(band_solve_kernel<256>,
                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                return MFB_ERR_SMEM;
            band_solve_kernel<256><<<n_sys, 256, smem, st>>>(pats, sys_pat, Kbuf, sys_koff,
                                                             work, sys_woff, X, sys_xoff, info);
            break;
        case 512:
            if (cudaFuncSetAttribute(band_solve_kernel<512>,
                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                return MFB_ERR_SMEM;
            band_solve_kernel<512><<<n_sys, 512, smem, st>>>(pats, sys_pat, Kbuf, sys_koff,
                                                             work, sys_woff, X, sys_xoff, info);
            break;
        case 1024:
            if (cudaFuncSetAttribute(band_solve_kernel<1024>,
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

extern "C" int mfb_debug_bprof(unsigned long long *out) {
#ifdef MFB_PROFILE
    return cudaMemcpyFromSymbol(out, g_bprof, sizeof(unsigned long long) * 16) == cudaSuccess ? 0 : 2;
#else
    (void)out;
    return 1;
#endif
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
