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
#ifdef MFB_NO_DMMA
    // debug: the same 8x8x4 product with scalar FMAs (fragment exchange by shuffles)
    const int lane = threadIdx.x & 31, g = lane >> 2, q4 = lane & 3;
    double s0 = d0, s1 = d1;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double ak = __shfl_sync(0xffffffffu, a, g * 4 + k);
        const double b0 = __shfl_sync(0xffffffffu, b, (2 * q4) * 4 + k);
        const double b1 = __shfl_sync(0xffffffffu, b, (2 * q4 + 1) * 4 + k);
        s0 = fma(ak, b0, s0);
        s1 = fma(ak, b1, s1);
    }
    d0 = s0;
    d1 = s1;
#else
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
#endif
}

// Barrier among the C CTAs that share one system (co-resident: cooperative
// launch). Writes before it are published at GPU scope; reads of data other
// CTAs wrote go through L2 (__ldcg) because L1 is not coherent.
__device__ __forceinline__ void group_sync(unsigned int *ctr, int C, unsigned int &target) {
    __syncthreads();
    if (C > 1) {
        if (threadIdx.x == 0) {
            target += C;
            __threadfence();
            atomicAdd(ctr, 1u);
            unsigned int v;
            while (true) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
                if (v >= target) break;
                __nanosleep(32);
            }
            __threadfence();
        }
        __syncthreads();
    }
}

template <int NT>
__global__ void __launch_bounds__(NT)
band_solve_kernel(const MfbPattern *__restrict__ pats, const int *__restrict__ sys_pat,
                  const double *__restrict__ Kbuf, const long long *__restrict__ sys_koff,
                  double *__restrict__ work, const long long *__restrict__ sys_woff,
                  double *__restrict__ Xout, const long long *__restrict__ sys_xoff,
                  int *__restrict__ info, int C, unsigned int *__restrict__ bar) {
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
    __shared__ int s_flag;
#ifdef MFB_PROFILE
    __shared__ long long s_bt0;
#endif

    // C CTAs cooperate on system s: rank owns the trailing-column tiles and
    // rhs-column tiles t with t % C == rank; the panel is factored redundantly
    const int s = blockIdx.x / C, rank = blockIdx.x % C;
    unsigned int bar_target = 0;
    unsigned int *ctr = bar + s;
    const MfbPattern P = pats[sys_pat[s]];
    const double *K = Kbuf + sys_koff[s];
    const int n = P.n, kl = P.kl, ku = P.ku, ldab = P.ldab, nb = P.nb;
    const int nrhs = P.ndof + 1;
    const int ncy = nrhs;              // rhs block: N_dof mortar columns + bar
    const int UST = kl + ku + 8;
    double *AB = work + sys_woff[s];
    double *Y = AB + (long long)ldab * n;
    double *Pnl = smem;                          // (kl + NB) x PST   panel L | U11
    double *U12s = Pnl + (kl + NB) * PST;        // NB x UST          U12 of the panel
    double *Tmp = U12s + NB * UST;               // NB x UST          staged A12
    const int TMPN = max(NB * UST, 3 * MAX_NB * MAX_NCY);   // also kernel-projection scratch
    double *Ytop = Tmp + TMPN;                   // NB x ncy          rhs rows of the panel
    int *s_perm = reinterpret_cast<int *>(Ytop + NB * ncy);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

    // ---- 1. assembly ---------------------------------------------------
    const long long nab = (long long)ldab * n, ny = (long long)n * ncy;
    const int gt = rank * NT + tid, GS = C * NT;
    for (long long t = gt; t < nab + ny; t += GS) AB[t] = 0.0;
    group_sync(ctr, C, bar_target);
    for (int e = gt; e < P.n_entries; e += GS) {
        double v = 0.0;
        for (int t = P.e_tptr[e]; t < P.e_tptr[e + 1]; ++t)
            v += mfb_term(P.t_kind[t], P.t_c[t], K, P.t_k[t]);
        AB[bidx(P.e_row[e], P.e_col[e], kl, ku, ldab)] = v;
    }
    for (int d = 0; d < P.ndof; ++d)
        for (int q = P.q_ptr[d] + gt; q < P.q_ptr[d + 1]; q += GS) {
            int r = P.q_row[q];
            if (r < n) Y[(long long)r * ncy + d] = P.q_val[q];
        }
    for (int i = gt; i < n; i += GS) Y[(long long)i * ncy + P.ndof] = P.bar_const[i];
    group_sync(ctr, C, bar_target);
    for (int b = gt; b < P.n_bar_rows; b += GS) {
        int r = P.b_row[b];
        if (r >= n) continue;
        double v = 0.0;
        for (int t = P.b_tptr[b]; t < P.b_tptr[b + 1]; ++t)
            v += mfb_term(P.bt_kind[t], P.bt_c[t], K, P.bt_k[t]);
        Y[(long long)r * ncy + P.ndof] += v;
    }
    group_sync(ctr, C, bar_target);
#define OWN(tile) (((tile) % C) == rank)

    // ---- 1b. rigid-body kernel (Stokes, nb > 0): make the rhs compatible --
    // The reference pins the kernel with Lagrange rows C (stokes.py:276-298):
    // K x + C^T mu = r, C x = 0. With the nb pinned dofs J removed, K_II is
    // regular; mu = (C C^T)^-1 C r, then K_II x~ = (r - C^T mu)_I, x~_J = 0,
    // and x = x~ - C^T (C C^T)^-1 C x~ (section 4). E = C_I^T, G = [C_J; (CC^T)^-1].
    const int lane0 = tid & 31, wid0 = tid >> 5;
    if (nb > 0) {
        double *s_cr = Tmp;                      // nb x nrhs  (C r, then mu)
        for (int pr = wid0; pr < nb * nrhs; pr += NT / 32) {
            const int a = pr / nrhs, c = pr % nrhs;
            if (!OWN(c >> 3)) continue;
            double acc = 0.0;
            for (int i = lane0; i < n; i += 32) acc += P.E[(long long)i * nb + a] * Y[(long long)i * ncy + c];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
            if (lane0 == 0) s_cr[pr] = acc;
        }
        __syncthreads();
        if (tid == 0) {
            // pinned rows of r: Q entries with row >= n, bar_const and bar terms
            double *rj = Tmp + MAX_NB * MAX_NCY;
            for (int t = 0; t < nb * nrhs; ++t) rj[t] = 0.0;
            for (int d = 0; d < P.ndof; ++d)
                for (int q = P.q_ptr[d]; q < P.q_ptr[d + 1]; ++q)
                    if (P.q_row[q] >= n) rj[(P.q_row[q] - n) * nrhs + d] += P.q_val[q];
            for (int b = 0; b < nb; ++b) rj[b * nrhs + P.ndof] += P.bar_const[n + b];
            for (int bb = 0; bb < P.n_bar_rows; ++bb) {
                const int r = P.b_row[bb];
                if (r < n) continue;
                double v = 0.0;
                for (int t = P.b_tptr[bb]; t < P.b_tptr[bb + 1]; ++t)
                    v += mfb_term(P.bt_kind[t], P.bt_c[t], K, P.bt_k[t]);
                rj[(r - n) * nrhs + P.ndof] += v;
            }
            double *cr = Tmp + 2 * MAX_NB * MAX_NCY;
            for (int a = 0; a < nb; ++a)
                for (int c = 0; c < nrhs; ++c) {
                    double v = s_cr[a * nrhs + c];
                    for (int b = 0; b < nb; ++b) v += P.G[a * nb + b] * rj[b * nrhs + c];
                    cr[a * nrhs + c] = v;
                }
            for (int a = 0; a < nb; ++a)
                for (int c = 0; c < nrhs; ++c) {
                    double v = 0.0;
                    for (int b = 0; b < nb; ++b) v += P.G[(nb + a) * nb + b] * cr[b * nrhs + c];
                    s_cr[a * nrhs + c] = v;              // mu
                }
        }
        __syncthreads();
        for (long long t = tid; t < (long long)n * nrhs; t += NT) {
            const int i = (int)(t / nrhs), c = (int)(t % nrhs);
            if (!OWN(c >> 3)) continue;
            double v = Y[(long long)i * ncy + c];
            for (int a = 0; a < nb; ++a) v -= P.E[(long long)i * nb + a] * s_cr[a * nrhs + c];
            Y[(long long)i * ncy + c] = v;
        }
    }
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
                                   ? __ldcg(AB + bidx(r, col, kl, ku, ldab)) : 0.0;
        }
        // every CTA must hold the panel before rank 0 writes its factors back
        group_sync(ctr, C, bar_target);
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
                    if (tid == 0) { if (rank == 0) info[s] = j0 + c + 1; s_flag = -1; }
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
        if (rank == 0)
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
            if (!OWN((c0 >> 3) + (cc >> 3))) continue;
            const int src = j0 + (q < pnb ? s_perm[q] : 0);
            const bool vt = q < pnb && cc < nc && col - src <= kl + ku && src - col <= kl;
            const int srl = j0 + (q < nlow ? s_perm[s_low[q]] : 0);
            const bool vl = q < nlow && cc < nc && col - srl <= kl + ku && srl - col <= kl;
            const double x = __ldcg(AB + (vt ? bidx(src, col, kl, ku, ldab) : 0));
            const double y = __ldcg(AB + (vl ? bidx(srl, col, kl, ku, ldab) : 0));
            Tmp[q * UST + cc] = vt ? x : 0.0;
            U12s[q * UST + cc] = vl ? y : 0.0;
        }
        __syncthreads();
        for (int t = tid; t < nlow * nc; t += NT) {
            const int z = t / nc, cc = t % nc, col = c0 + cc;
            if (!OWN((c0 >> 3) + (cc >> 3))) continue;
            const int row = j0 + s_low[z];
            if (row - col <= kl) AB[bidx(row, col, kl, ku, ldab)] = U12s[z * UST + cc];
        }
        __syncthreads();
        // U12 = L11^-1 A12 by forward substitution (thread per column, as gbtrf's
        // dtrsm): written to the band (top rows) and to U12s
        for (int cc = tid; cc < ncpad; cc += NT) {
            if (!OWN((c0 >> 3) + (cc >> 3))) continue;
            double u[NB];
#pragma unroll
            for (int q = 0; q < NB; ++q) u[q] = Tmp[q * UST + cc];
#pragma unroll
            for (int q = 1; q < NB; ++q) {
                double v = u[q];
#pragma unroll
                for (int qq = 0; qq < q; ++qq) v -= Pnl[q * PST + qq] * u[qq];
                u[q] = q < pnb ? v : 0.0;
            }
            const int col = c0 + cc;
#pragma unroll
            for (int q = 0; q < NB; ++q) {
                U12s[q * UST + cc] = q < pnb ? u[q] : 0.0;
                const int row = j0 + q;
                if (q < pnb && cc < nc && col - row <= kl + ku) AB[bidx(row, col, kl, ku, ldab)] = u[q];
            }
        }
        // phase A': right-hand sides -- permute + forward substitution (thread per column)
        for (int cy = tid; cy < ncy; cy += NT) {
            if (!OWN(cy >> 3)) continue;
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
            // absolute tile ownership: a column keeps its owner across panels,
            // so its (L1-cached) reads only ever see the owner's own writes
            const int tbase = c0 >> 3;
            const int tj0 = ((rank - tbase) % C + C) % C;
            for (int tj = tj0 + C * wid; tj < tcn; tj += C * NW) {
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
                for (int tc = rank; tc < tcy; tc += C) {
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
        group_sync(ctr, C, bar_target);
        BPROF(5);
    }

    // ---- 3. blocked column-oriented back substitution with U ---------------
    const int last = ((n - 1) / NB) * NB;
    for (int j0 = last; j0 >= 0; j0 -= NB) {
        const int pnb = min(NB, n - j0);
        for (int t = tid; t < NB * NB; t += NT) {
            const int r = t / NB, c = t % NB;
            s_u11[t] = (r < pnb && c < pnb && c >= r) ? __ldcg(AB + bidx(j0 + r, j0 + c, kl, ku, ldab)) : 0.0;
        }
        __syncthreads();
        for (int cy = tid; cy < ncy; cy += NT) {
            if (!OWN(cy >> 3)) continue;
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
                                 ? -__ldcg(AB + bidx(i, j0 + k, kl, ku, ldab)) : 0.0;
                }
                for (int tc = rank; tc < tcy; tc += C) {
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

    // ---- 4. project out the rigid-body kernel (nb > 0) --------------------
    double *X = Xout + sys_xoff[s];
    if (nb > 0) {
        double *s_cx = Tmp;                      // nb x nrhs: C x~, then alpha
        for (int pr = wid0; pr < nb * nrhs; pr += NT / 32) {
            const int a = pr / nrhs, c = pr % nrhs;
            if (!OWN(c >> 3)) continue;
            double acc = 0.0;
            for (int i = lane0; i < n; i += 32) acc += P.E[(long long)i * nb + a] * Y[(long long)i * ncy + c];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
            if (lane0 == 0) s_cx[MAX_NB * MAX_NCY + pr] = acc;
        }
        __syncthreads();
        if (tid < nb * nrhs) {
            const int a = tid / nrhs, c = tid % nrhs;
            double v = 0.0;
            for (int b = 0; b < nb; ++b) v += P.G[(nb + a) * nb + b] * s_cx[MAX_NB * MAX_NCY + b * nrhs + c];
            s_cx[a * nrhs + c] = v;
        }
        __syncthreads();
        for (long long t = tid; t < (long long)n * nrhs; t += NT) {
            const int i = (int)(t / nrhs), c = (int)(t % nrhs);
            if (!OWN(c >> 3)) continue;
            double v = Y[(long long)i * ncy + c];
            for (int a = 0; a < nb; ++a) v -= P.E[(long long)i * nb + a] * s_cx[a * nrhs + c];
            X[t] = v;
        }
        for (int t = tid; t < nb * nrhs; t += NT) {
            const int b = t / nrhs, c = t % nrhs;
            if (!OWN(c >> 3)) continue;
            double v = 0.0;
            for (int a = 0; a < nb; ++a) v -= P.G[a * nb + b] * s_cx[a * nrhs + c];
            X[(long long)n * nrhs + t] = v;
        }
    } else {
        for (long long t = tid; t < (long long)n * nrhs; t += NT)
            if (OWN((int)(t % nrhs) >> 3)) X[t] = Y[t];
    }
    if (tid == 0 && rank == 0) info[s] = 0;
#undef OWN
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

template <int NT>
static int launch_band(int n_sys, int C, size_t smem, cudaStream_t st, const MfbPattern *pats,
                       const int *sys_pat, const double *Kbuf, const long long *sys_koff,
                       double *work, const long long *sys_woff, double *X,
                       const long long *sys_xoff, int *info, unsigned int *bar) {
    if (cudaFuncSetAttribute(band_solve_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return MFB_ERR_SMEM;
    if (C == 1) {
        band_solve_kernel<NT><<<n_sys, NT, smem, st>>>(pats, sys_pat, Kbuf, sys_koff, work,
                                                       sys_woff, X, sys_xoff, info, C, bar);
    } else {
        // the C CTAs of a system wait on one another: cooperative launch
        // guarantees they are co-resident
        if (cudaMemsetAsync(bar, 0, sizeof(unsigned int) * n_sys, st) != cudaSuccess)
            return MFB_ERR_LAUNCH;
        void *args[] = {(void *)&pats, (void *)&sys_pat, (void *)&Kbuf, (void *)&sys_koff,
                        (void *)&work, (void *)&sys_woff, (void *)&X, (void *)&sys_xoff,
                        (void *)&info, (void *)&C, (void *)&bar};
        if (cudaLaunchCooperativeKernel((const void *)band_solve_kernel<NT>, dim3(n_sys * C),
                                        dim3(NT), args, smem, st) != cudaSuccess)
            return MFB_ERR_LAUNCH;
    }
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}

extern "C" int mfb_systems_solve(const MfbPattern *pats, int n_sys, const int *sys_pat,
                                 const double *Kbuf, const long long *sys_koff,
                                 double *work, const long long *sys_woff, double *X,
                                 const long long *sys_xoff, int *info, int threads,
                                 int smem_doubles, int group, unsigned int *bar, void *stream) {
    if (n_sys <= 0) return n_sys == 0 ? MFB_OK : MFB_ERR_ARG;
    if (group < 1 || (group > 1 && bar == nullptr)) return MFB_ERR_ARG;
    const size_t smem = (size_t)smem_doubles * sizeof(double);
    cudaStream_t st = mfb_stream(stream);
    switch (threads) {
        case 128: return launch_band<128>(n_sys, group, smem, st, pats, sys_pat, Kbuf, sys_koff,
                                          work, sys_woff, X, sys_xoff, info, bar);
        case 256: return launch_band<256>(n_sys, group, smem, st, pats, sys_pat, Kbuf, sys_koff,
                                          work, sys_woff, X, sys_xoff, info, bar);
        case 512: return launch_band<512>(n_sys, group, smem, st, pats, sys_pat, Kbuf, sys_koff,
                                          work, sys_woff, X, sys_xoff, info, bar);
        default: return MFB_ERR_ARG;
    }
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
