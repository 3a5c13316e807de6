// Darcy flux basis by static condensation of the hybridised SPD system.
//
// Reference: the Darcy subdomain operator is the mixed RT0/P0 saddle matrix
// factored with SuperLU (darcy.py:67-147); the flux basis costs one
// backsolve per mortar dof (interface.py:218-235). Here the same discrete
// problem is solved in its hybridised form (paper_1802_06263_b200/hybrid.py):
// one SPD unknown per non-Dirichlet edge, every cell contributing K_T Hhat.
// The flux-basis block B and the bar jump h are the Schur complement left
// after eliminating all unknown edges from the bordered matrix
//     [ H_II  V ]      V = [H_IG G | v_b],   Z = initial border block,
//     [ V^T   Z ]
// so one CTA per (subdomain, local realization) runs a band Cholesky over a
// sliding window held entirely in shared memory -- rows enter the window as
// they are assembled from K, leave it once eliminated -- and never touches
// global memory for the factor. Per panel of BP pivots, one warp factors the
// panel (Cholesky + forward substitution of the border rows) while the other
// warps assemble the rows entering the window; then all warps apply the
// rank-BP trailing update to the window, the border panel and the Schur
// block on FP64 tensor cores (mma.sync m8n8k4 f64 -> SASS DMMA).
// Field mode additionally stores the panels so that mfb_darcy_backsolve can
// form X = H_II^-1 V and mfb_darcy_recover the cell fields.
#include "mfb_common.cuh"

#ifdef MFB_PROFILE
__device__ unsigned long long g_prof[16];
#define PROF_MARK(i)                                                              \
    do {                                                                          \
        if (blockIdx.x == 0 && (threadIdx.x == 0 || threadIdx.x == 32)) {         \
            long long _c = clock64();                                             \
            int _slot = (i) + (threadIdx.x == 32 ? 8 : 0);                        \
            if ((i) > 0) atomicAdd(&g_prof[_slot], (unsigned long long)(_c - s_t0[threadIdx.x >> 5])); \
            s_t0[threadIdx.x >> 5] = _c;                                          \
        }                                                                         \
    } while (0)
#else
#define PROF_MARK(i) do {} while (0)
#endif

namespace {

constexpr int HYB_NT = 256;
constexpr int HYB_NW = HYB_NT / 32;

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ int cpad(int nd) { return (nd + 1 + 7) & ~7; }

__device__ __forceinline__ double gcoef(const MfbHybPattern &P, int gi, int d) {
    for (int t = P.gam_ptr[gi]; t < P.gam_ptr[gi + 1]; ++t)
        if (P.gam_d[t] == d) return P.gam_c[t];
    return 0.0;
}

__device__ __forceinline__ double term_sum(const int *tptr, const int *cell,
                                           const double *coef, int e, const double *K) {
    double v = 0.0;
    for (int t = tptr[e]; t < tptr[e + 1]; ++t) {
        const int c = cell[t];
        v += c >= 0 ? coef[t] * K[c] : coef[t];
    }
    return v;
}

// scatter the term-table entries of rows [r0, r1) into the window (slots must
// be zero); each entry has a unique destination, so threads never collide
__device__ void assemble_entries(const MfbHybPattern &P, const double *K, int r0, int r1,
                                 int t0, int nt, double *W, double *Pb, int m, int ws, int Cp) {
    const int w = P.w;
    const int e0 = P.asm_ptr[r0], e1 = P.asm_ptr[r1];
    for (int e = e0 + t0; e < e1; e += nt) {
        const int r = P.asm_row[e], d = P.asm_dest[e];
        const double v = term_sum(P.asm_tptr, P.asm_cell, P.asm_coef, e, K);
        if (d <= w) W[(r % m) * ws + d] = v;
        else Pb[(r % m) * Cp + (d - w - 1)] = v;
    }
}

template <int BP>
__global__ void __launch_bounds__(HYB_NT, 2)
condense_kernel(const MfbHybPattern *__restrict__ pats, const int *__restrict__ sys_pat,
                const double *__restrict__ Kbuf, const long long *__restrict__ sys_koff,
                double *__restrict__ blocks, const long long *__restrict__ sys_boff,
                double *__restrict__ hbar, const long long *__restrict__ sys_hoff,
                double *__restrict__ Lstore, const long long *__restrict__ sys_loff,
                int *__restrict__ info) {
    constexpr int LS = BP + 4;
    extern __shared__ double sm[];
    __shared__ int s_bad;
    __shared__ double s_inv[8];
    __shared__ double s_linv[64], s_l11[64];
#ifdef MFB_PROFILE
    __shared__ long long s_t0[8];
#endif
    const int s = blockIdx.x;
    const MfbHybPattern &P = pats[sys_pat[s]];
    const double *K = Kbuf + sys_koff[s];
    const int n = P.n, w = P.w, ws = P.ws, nd = P.ndof;
    const int Cp = cpad(nd), m = w + BP;
    double *W = sm;                 // m x ws      window rows, lower band
    double *Pb = W + m * ws;        // m x Cp      border columns of the window rows
    double *S = Pb + m * Cp;        // Cp x Cp     Schur block
    double *Lb = S + Cp * Cp;       // m x LS      current panel (L11 | L21)
    double *Yb = Lb + m * LS;       // BP x CY     L11^-1 (border rows of the panel); rows 4 doubles
    const int CY = Cp + 4;          // apart from a multiple of 8: conflict-free MMA B operands
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int g = lane >> 2, q4 = lane & 3;
    if (tid == 0) {
        s_bad = 0;
        // the system's K (read a few cells per panel, first touch from DRAM)
        // brought into L2 up front by one bulk prefetch
        const unsigned bytes = (unsigned)(P.n_cells * 8) & ~15u;
        if (bytes)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(K), "r"(bytes)
                         : "memory");
    }
    for (int t = tid; t < Cp * Cp; t += HYB_NT) S[t] = 0.0;
    // initial border block Z and the first window rows (term tables, thread per entry)
    for (int t = tid; t < m * ws; t += HYB_NT) W[t] = 0.0;
    for (int t = tid; t < m * Cp; t += HYB_NT) Pb[t] = 0.0;
    __syncthreads();
    for (int e = tid; e < P.z_n; e += HYB_NT) {
        const int d1 = P.z_dest[e] / (nd + 1), d2 = P.z_dest[e] % (nd + 1);
        S[d1 * Cp + d2] = term_sum(P.z_tptr, P.z_cell, P.z_coef, e, K);
    }
    assemble_entries(P, K, 0, min(n, m), tid, HYB_NT, W, Pb, m, ws, Cp);

    __syncthreads();

    const int n_pan = (n + BP - 1) / BP;
    const long long pstride = (long long)m * LS + (long long)BP * Cp;
    for (int pi = 0; pi < n_pan; ++pi) {
        PROF_MARK(0);
        const int k = pi * BP;
        const int nb = min(BP, n - k);
        const int rend = min(n, k + BP + w);
        const int nrow = rend - k;
        const int kslot = k % m;                  // window slot of row k
        for (int t = tid; t < nrow * BP; t += HYB_NT) {
            const int i = t / BP, p = t % BP;
            int sl = kslot + i;
            if (sl >= m) sl -= m;
            double v = 0.0;
            if (p < nb && i >= p && i - p <= w) v = W[sl * ws + (p - i + w)];
            Lb[i * LS + p] = v;
        }
        for (int t = tid; t < BP * Cp; t += HYB_NT) {
            const int p = t / Cp, c = t - p * Cp;
            int sl = kslot + p;
            if (sl >= m) sl -= m;
            Yb[p * CY + c] = p < nb ? Pb[sl * Cp + c] : 0.0;
        }
        __syncthreads();
        PROF_MARK(1);
        if (wid == 0) {
            // 8x8 diagonal block: Cholesky on warp 0, lane (i, c) = (lane / 4,
            // lane % 4) holding a[i][c] and a[i][c + 4] (missing pivots of a
            // short last panel are identity rows). Right-looking: step p
            // scales column p and subtracts L(i,p) L(j,p) from every (i, j) of
            // the lower triangle with j > p -- per entry the same sequence of
            // fused multiply-adds, in the same order, as a serial left-looking
            // loop over q < j, so the factor does not depend on the form.
            {
                const int i = lane >> 2, c = lane & 3;
                double A0 = (i < nb && c < nb) ? Lb[i * LS + c] : (i == c ? 1.0 : 0.0);
                double A1 = (i < nb && c + 4 < nb) ? Lb[i * LS + c + 4] : (i == c + 4 ? 1.0 : 0.0);
                bool ok = true;
                double dinv = 0.0;               // 1 / L(i,i), kept by the diagonal's lane
#pragma unroll
                for (int p = 0; p < 8; ++p) {
                    const double v = __shfl_sync(0xffffffffu, p < 4 ? A0 : A1, p * 4 + (p & 3));
                    ok = ok && (v > 0.0);
                    const double d = sqrt(v);
                    const double inv = 1.0 / d;
                    if (c == (p & 3)) {
                        double &col = p < 4 ? A0 : A1;
                        if (i > p) col = col * inv;
                        else if (i == p) { col = d; dinv = inv; }
                    }
                    const double lip = __shfl_sync(0xffffffffu, p < 4 ? A0 : A1,
                                                   (lane & ~3) | (p & 3));
                    const double l0 = __shfl_sync(0xffffffffu, p < 4 ? A0 : A1, c * 4 + (p & 3));
                    const double l1 = __shfl_sync(0xffffffffu, p < 4 ? A0 : A1,
                                                  (c + 4) * 4 + (p & 3));
                    if (c > p && i >= c) A0 -= lip * l0;
                    if (c + 4 > p && i >= c + 4) A1 -= lip * l1;
                }
                if (!__all_sync(0xffffffffu, ok) && lane == 0) { s_bad = 1; info[s] = -(k + 1); }
                if (i < nb) {
                    Lb[i * LS + c] = (c <= i && c < nb) ? A0 : 0.0;
                    Lb[i * LS + c + 4] = (c + 4 <= i && c + 4 < nb) ? A1 : 0.0;
                }
                if (c == (i & 3)) {              // the diagonal's lane
                    s_inv[i] = dinv;
                    if (i < nb) Lb[i * LS + BP] = dinv;   // padding column: 1 / L(i,i)
                }
                // the factor (identity rows past a short panel) for the inverse below
                s_l11[i * 8 + c] = A0;
                s_l11[i * 8 + c + 4] = A1;
            }
            __syncwarp();
            // L11^-1 (lower triangular) for the panel solves on the tensor
            // cores: column j by lane j (forward substitution, the sums in the
            // order of a serial loop) -- off thread 0's chain
            if (lane < 8) {
                const int j = lane;
                double x[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    double v = 0.0;
                    if (i == j) {
                        v = s_inv[i];
                    } else if (i > j) {
#pragma unroll
                        for (int q = 0; q < i; ++q)
                            if (q >= j) v -= s_l11[i * 8 + q] * x[q];
                        v *= s_inv[i];
                    }
                    x[i] = v;
                    s_linv[i * 8 + j] = v;
                }
            }
        } else {
            // rows entering the window take the freed slots of this panel:
            // zero them, sync the assembly warps, scatter the term-table entries
            const int r0 = k + m, r1 = min(n, k + m + BP);
            const int at = tid - 32, an = HYB_NT - 32;
            // (the slots of rows k .. k + nr - 1: one or, when the window wraps,
            // two contiguous runs of rows in W and in Pb, zeroed as flat arrays)
            const int nr = r1 - r0;
            if (nr > 0) {
                const int n1 = min(nr, m - kslot), n2 = nr - n1;
                for (int t = at; t < n1 * ws; t += an) W[kslot * ws + t] = 0.0;
                for (int t = at; t < n2 * ws; t += an) W[t] = 0.0;
                for (int t = at; t < n1 * Cp; t += an) Pb[kslot * Cp + t] = 0.0;
                for (int t = at; t < n2 * Cp; t += an) Pb[t] = 0.0;
            }
            asm volatile("bar.sync 1, %0;" ::"r"(HYB_NT - 32));
            PROF_MARK(6);
            // the entries of the entering rows, flattened per panel at plan time
            // (hybrid.py panel_entries): record -> K, no table walk
            const int e0 = P.pe_ptr[pi], e1 = P.pe_ptr[pi + 1];
            const int4 *rec = reinterpret_cast<const int4 *>(P.pe_rec);
            const double2 *cf = reinterpret_cast<const double2 *>(P.pe_coef);
            for (int e = e0 + at; e < e1; e += an) {
                const int4 r = rec[e];
                const double2 c = cf[e];
                double v = 0.0;
                v += r.y >= 0 ? c.x * K[r.y] : c.x;
                if (r.w > 1) v += r.z >= 0 ? c.y * K[r.z] : c.y;
                W[r.x] = v;                           // W | Pb: one shared-memory region
            }
            PROF_MARK(7);
        }
        PROF_MARK(5);
        __syncthreads();
        PROF_MARK(2);
        if (s_bad) return;
        {
            // panel solves as products with L11^-1 on DMMA tiles (all warps):
            // L21 = A21 L11^-T (row tiles), Yb = L11^-1 Yb (column tiles); a
            // tile's operands are read before its results overwrite them
            const int R = nrow - nb;
            const int tr = (R + 7) >> 3, tc = Cp >> 3;
            const double li0 = s_linv[g * 8 + q4], li1 = s_linv[g * 8 + 4 + q4];
            for (int it = wid; it < tr + tc; it += HYB_NW) {
                double d0 = 0.0, d1 = 0.0;
                if (it < tr) {
                    const int ra = nb + it * 8 + g;
                    const double a0 = ra < nrow ? Lb[ra * LS + q4] : 0.0;
                    const double a1 = ra < nrow ? Lb[ra * LS + 4 + q4] : 0.0;
                    dmma(d0, d1, a0, li0);
                    dmma(d0, d1, a1, li1);
                    __syncwarp();
                    if (ra < nrow) {
                        Lb[ra * LS + 2 * q4] = d0;
                        Lb[ra * LS + 2 * q4 + 1] = d1;
                    }
                } else {
                    const int c = (it - tr) * 8;
                    const double b0 = Yb[q4 * CY + c + g], b1 = Yb[(4 + q4) * CY + c + g];
                    dmma(d0, d1, li0, b0);
                    dmma(d0, d1, li1, b1);
                    __syncwarp();
                    Yb[g * CY + c + 2 * q4] = d0;
                    Yb[g * CY + c + 2 * q4 + 1] = d1;
                }
            }
        }
        __syncthreads();
        PROF_MARK(3);
        if (Lstore) {
            double *dst = Lstore + sys_loff[s] + (long long)pi * pstride;
            for (int t = tid; t < nrow * LS; t += HYB_NT) dst[t] = Lb[t];
            for (int t = tid; t < BP * Cp; t += HYB_NT)
                dst[(long long)m * LS + t] = Yb[(t / Cp) * CY + t % Cp];
        }
        // trailing updates on DMMA: window (lower band), border panel, Schur
        // block. A warp owns whole row tiles (its A fragments stay in registers
        // across the row's window and border tiles); row tiles are dealt in
        // snake order so the triangular work is balanced across warps.
        const int R = nrow - nb;
        const int tr = (R + 7) >> 3, tc = Cp >> 3;
        int rbase = kslot + nb;
        if (rbase >= m) rbase -= m;
        for (int it = wid; it < tr + tc; it += HYB_NW) {
            if (it < tr) {
                const int ti = (it & 1) ? (tr - 1 - (it >> 1)) : (it >> 1);
                const int ii = ti * 8 + g;
                const int ra = nb + ii;
                const double a0 = ra < nrow ? -Lb[ra * LS + q4] : 0.0;
                const double a1 = ra < nrow ? -Lb[ra * LS + 4 + q4] : 0.0;
                int rr = rbase + ii;
                if (rr >= m) rr -= m;
                const bool rv = ii < R;
                double *rowW = W + (rv ? rr : 0) * ws + (w - ii);
                double *rowP = Pb + (rv ? rr : 0) * Cp;
                for (int tj = 0; tj <= ti; ++tj) {
                    const int rb = nb + tj * 8 + g;
                    const double b0 = rb < nrow ? Lb[rb * LS + q4] : 0.0;
                    const double b1 = rb < nrow ? Lb[rb * LS + 4 + q4] : 0.0;
                    const int ja = tj * 8 + 2 * q4;
                    const bool va = rv && ja <= ii, vb = rv && ja + 1 <= ii;
                    double d0 = va ? rowW[ja] : 0.0;
                    double d1 = vb ? rowW[ja + 1] : 0.0;
                    dmma(d0, d1, a0, b0);
                    dmma(d0, d1, a1, b1);
                    if (va) rowW[ja] = d0;
                    if (vb) rowW[ja + 1] = d1;
                }
                for (int tcol = 0; tcol < tc; ++tcol) {
                    const int ca = tcol * 8 + 2 * q4;
                    double d0 = rv ? rowP[ca] : 0.0;
                    double d1 = rv ? rowP[ca + 1] : 0.0;
                    dmma(d0, d1, a0, Yb[q4 * CY + tcol * 8 + g]);
                    dmma(d0, d1, a1, Yb[(4 + q4) * CY + tcol * 8 + g]);
                    if (rv) {
                        rowP[ca] = d0;
                        rowP[ca + 1] = d1;
                    }
                }
            } else {
                const int t1 = it - tr;
                const double a0 = -Yb[q4 * CY + t1 * 8 + g];
                const double a1 = -Yb[(4 + q4) * CY + t1 * 8 + g];
                double *rowS = S + (t1 * 8 + g) * Cp;
                for (int t2 = 0; t2 < tc; ++t2) {
                    const int ca = t2 * 8 + 2 * q4;
                    double d0 = rowS[ca], d1 = rowS[ca + 1];
                    dmma(d0, d1, a0, Yb[q4 * CY + t2 * 8 + g]);
                    dmma(d0, d1, a1, Yb[(4 + q4) * CY + t2 * 8 + g]);
                    rowS[ca] = d0;
                    rowS[ca + 1] = d1;
                }
            }
        }
        __syncthreads();
        PROF_MARK(4);
    }
    for (int t = tid; t < nd * nd; t += HYB_NT) {
        const int r = t % nd, c = t / nd;
        blocks[sys_boff[s] + t] = S[r * Cp + c];      // column-major: Bt[c*nd + r]
    }
    for (int r = tid; r < nd; r += HYB_NT) hbar[sys_hoff[s] + r] = S[r * Cp + nd];
    if (tid == 0) info[s] = 0;
}

template <int BP>
__global__ void __launch_bounds__(HYB_NT)
backsolve_kernel(const MfbHybPattern *__restrict__ pats, const int *__restrict__ sys_pat,
                 const double *__restrict__ Lstore, const long long *__restrict__ sys_loff,
                 double *__restrict__ X, const long long *__restrict__ sys_xoff) {
    constexpr int LS = BP + 4;
    extern __shared__ double sm[];
    const int s = blockIdx.x;
    const MfbHybPattern &P = pats[sys_pat[s]];
    const int n = P.n, w = P.w, nd = P.ndof;
    const int Cp = cpad(nd), m = w + BP;
    double *Xw = sm;                // m x Cp   solved rows (circular)
    double *Lp = Xw + m * Cp;       // m x LS   panel factor
    double *Tp = Lp + m * LS;       // BP x Cp  panel rhs
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int g = lane >> 2, q4 = lane & 3;
    const long long pstride = (long long)m * LS + (long long)BP * Cp;
    double *Xs = X + sys_xoff[s];
    const int n_pan = (n + BP - 1) / BP;
    for (int pi = n_pan - 1; pi >= 0; --pi) {
        const int k = pi * BP;
        const int nb = min(BP, n - k);
        const int rend = min(n, k + BP + w);
        const int nrow = rend - k, R = nrow - nb;
        const double *src = Lstore + sys_loff[s] + (long long)pi * pstride;
        for (int t = tid; t < nrow * LS; t += HYB_NT) Lp[t] = src[t];
        for (int t = tid; t < BP * Cp; t += HYB_NT) Tp[t] = src[(long long)m * LS + t];
        __syncthreads();
        // Tp -= L21^T X[k+nb .. rend)   (DMMA; a warp owns one 8x8 output tile)
        const int ti_n = BP / 8, tc = Cp >> 3;
        for (int t = wid; t < ti_n * tc; t += HYB_NW) {
            const int ti = t / tc, tj = t % tc;
            const int ca = tj * 8 + 2 * q4;
            double d0 = Tp[(ti * 8 + g) * Cp + ca];
            double d1 = Tp[(ti * 8 + g) * Cp + ca + 1];
            for (int k0 = 0; k0 < R; k0 += 4) {
                const int kk = k0 + q4;
                const double a = kk < R ? -Lp[(nb + kk) * LS + ti * 8 + g] : 0.0;
                const double b = kk < R ? Xw[((k + nb + kk) % m) * Cp + tj * 8 + g] : 0.0;
                dmma(d0, d1, a, b);
            }
            Tp[(ti * 8 + g) * Cp + ca] = d0;
            Tp[(ti * 8 + g) * Cp + ca + 1] = d1;
        }
        __syncthreads();
        // L11^T x = Tp (backward, one thread per column, column-oriented so the
        // dependency chain is two ops per row; 1/L(q,q) sits in column BP)
        for (int c = tid; c < Cp; c += HYB_NT) {
            double t[BP];
#pragma unroll
            for (int q = 0; q < BP; ++q) t[q] = q < nb ? Tp[q * Cp + c] : 0.0;
#pragma unroll
            for (int q = BP - 1; q >= 0; --q) {
                if (q >= nb) continue;
                const double v = t[q] * Lp[q * LS + BP];
                t[q] = v;
#pragma unroll
                for (int qq = 0; qq < q; ++qq) t[qq] -= Lp[q * LS + qq] * v;
            }
#pragma unroll
            for (int q = 0; q < BP; ++q) {
                if (q >= nb) continue;
                Tp[q * Cp + c] = t[q];
                Xw[((k + q) % m) * Cp + c] = t[q];
                Xs[(long long)(k + q) * Cp + c] = t[q];
            }
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(HYB_NT)
recover_kernel(const MfbHybPattern *__restrict__ pats, const int *__restrict__ sys_pat,
               const double *__restrict__ Kbuf, const long long *__restrict__ sys_koff,
               const double *__restrict__ X, const long long *__restrict__ sys_xoff,
               double *__restrict__ M, const long long *__restrict__ sys_moff,
               double *__restrict__ Fb, const long long *__restrict__ sys_fboff) {
    const int s = blockIdx.y;
    const MfbHybPattern &P = pats[sys_pat[s]];
    const double *K = Kbuf + sys_koff[s];
    const int nd = P.ndof, Cp = cpad(nd);
    const int ne = P.n_edges, nc = P.n_cells;
    const double *Xs = X + sys_xoff[s];
    double *Ms = M + sys_moff[s];
    double *Fs = Fb + sys_fboff[s];
    const double hx = P.hx, hy = P.hy, s2 = P.s2;
    const double B[4] = {hy, -hy, hx, -hx};
    for (int T = blockIdx.x * HYB_NT + threadIdx.x; T < nc; T += gridDim.x * HYB_NT) {
        const double kap = K[T] / (P.nu * hx * hy);
        int e[4], kind[4], id[4];
        for (int a = 0; a < 4; ++a) {
            e[a] = P.cell_edges[4 * T + a];
            kind[a] = P.edge_kind[e[a]];
            id[a] = P.edge_idx[e[a]];
        }
        for (int c = 0; c <= nd; ++c) {
            const bool bar = c == nd;
            double gv[4], f[4], bg = 0.0, bf = 0.0, b2mu = 0.0;
            for (int a = 0; a < 4; ++a) {
                double mu;
                if (kind[a] == 0) mu = bar ? Xs[(long long)id[a] * Cp + nd] : -Xs[(long long)id[a] * Cp + c];
                else if (kind[a] == 1) mu = bar ? 0.0 : gcoef(P, id[a], c);
                else mu = bar ? P.p_val[id[a]] : 0.0;
                f[a] = (bar && P.has_src) ? P.cell_f[4 * T + a] : 0.0;
                gv[a] = f[a] + B[a] * mu;
                bg += B[a] * gv[a];
                bf += B[a] * f[a];
                b2mu += B[a] * B[a] * mu;
            }
            const double q = (bar && P.has_src) ? P.cell_q[T] : 0.0;
            double u[4];
            u[0] = kap * (4.0 * gv[0] - 2.0 * gv[1] - 3.0 * B[0] * bg / s2) - B[0] * q / (2.0 * s2);
            u[1] = kap * (-2.0 * gv[0] + 4.0 * gv[1] - 3.0 * B[1] * bg / s2) - B[1] * q / (2.0 * s2);
            u[2] = kap * (4.0 * gv[2] - 2.0 * gv[3] - 3.0 * B[2] * bg / s2) - B[2] * q / (2.0 * s2);
            u[3] = kap * (-2.0 * gv[2] + 4.0 * gv[3] - 3.0 * B[3] * bg / s2) - B[3] * q / (2.0 * s2);
            const double p = (bf + b2mu) / (2.0 * s2) + (q != 0.0 ? q / (12.0 * kap * s2) : 0.0);
            const double cvx = 0.5 * (u[0] + u[1]), cvy = 0.5 * (u[2] + u[3]);
            const double sg = bar ? 1.0 : -1.0;
            auto put = [&](long long row, double v) {
                if (bar) Fs[row] = v;
                else Ms[row * nd + c] = sg * v;
            };
            for (int a = 0; a < 4; ++a)
                if (P.edge_cells[2 * e[a]] == T) put(e[a], P.edge_noflow[e[a]] ? 0.0 : u[a]);
            put(ne + T, p);
            put(ne + nc + 2 * T, cvx);
            put(ne + nc + 2 * T + 1, cvy);
            put(ne + 3 * nc + T, p);
        }
    }
}

}  // namespace

extern "C" int mfb_darcy_condense(const MfbHybPattern *pats, int n_sys, const int *sys_pat,
                                  const double *Kbuf, const long long *sys_koff, double *blocks,
                                  const long long *sys_boff, double *hbar,
                                  const long long *sys_hoff, double *Lstore,
                                  const long long *sys_loff, int *info, int panel,
                                  int smem_bytes, void *stream) {
    if (n_sys <= 0) return n_sys == 0 ? MFB_OK : MFB_ERR_ARG;
    if ((panel & 255) != 8) return MFB_ERR_ARG;
    if (cudaFuncSetAttribute(condense_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem_bytes) != cudaSuccess)
        return MFB_ERR_SMEM;
    condense_kernel<8><<<n_sys, HYB_NT, smem_bytes, mfb_stream(stream)>>>(
        pats, sys_pat, Kbuf, sys_koff, blocks, sys_boff, hbar, sys_hoff, Lstore, sys_loff, info);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}

extern "C" int mfb_debug_prof(unsigned long long *out) {
#ifdef MFB_PROFILE
    return cudaMemcpyFromSymbol(out, g_prof, sizeof(unsigned long long) * 16) == cudaSuccess ? 0 : 2;
#else
    (void)out;
    return 1;
#endif
}

extern "C" int mfb_darcy_backsolve(const MfbHybPattern *pats, int n_sys, const int *sys_pat,
                                   const double *Lstore, const long long *sys_loff, double *X,
                                   const long long *sys_xoff, int panel, int smem_bytes,
                                   void *stream) {
    if (n_sys <= 0) return n_sys == 0 ? MFB_OK : MFB_ERR_ARG;
    cudaStream_t st = mfb_stream(stream);
    if (panel == 16) {
        if (cudaFuncSetAttribute(backsolve_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_bytes) != cudaSuccess)
            return MFB_ERR_SMEM;
        backsolve_kernel<16><<<n_sys, HYB_NT, smem_bytes, st>>>(pats, sys_pat, Lstore, sys_loff,
                                                                X, sys_xoff);
    } else if (panel == 8) {
        if (cudaFuncSetAttribute(backsolve_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_bytes) != cudaSuccess)
            return MFB_ERR_SMEM;
        backsolve_kernel<8><<<n_sys, HYB_NT, smem_bytes, st>>>(pats, sys_pat, Lstore, sys_loff,
                                                               X, sys_xoff);
    } else {
        return MFB_ERR_ARG;
    }
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}

extern "C" int mfb_darcy_recover(const MfbHybPattern *pats, int n_sys, const int *sys_pat,
                                 const double *Kbuf, const long long *sys_koff, const double *X,
                                 const long long *sys_xoff, double *M, const long long *sys_moff,
                                 double *Fb, const long long *sys_fboff, void *stream) {
    if (n_sys <= 0) return n_sys == 0 ? MFB_OK : MFB_ERR_ARG;
    dim3 grid(4, n_sys);
    recover_kernel<<<grid, HYB_NT, 0, mfb_stream(stream)>>>(pats, sys_pat, Kbuf, sys_koff, X,
                                                            sys_xoff, M, sys_moff, Fb, sys_fboff);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}
