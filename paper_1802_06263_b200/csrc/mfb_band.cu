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
__device__ unsigned long long g_bprof[24];
__device__ unsigned long long g_tl[4][4096];     // system 0 timeline (globaltimer ns)
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TL(which, k)                                                              \
    do {                                                                          \
        if (s == 0 && threadIdx.x == 0 && (k) < 4096) g_tl[which][k] = gtime();   \
    } while (0)
#define BPROF(i)                                                                  \
    do {                                                                          \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                \
            long long _c = clock64();                                             \
            if ((i) > 0) atomicAdd(&g_bprof[(i)], (unsigned long long)(_c - s_bt0)); \
            s_bt0 = _c;                                                           \
        }                                                                         \
    } while (0)
#define FPROF(i)                                                                  \
    do {                                                                          \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                \
            long long _c = clock64();                                             \
            if ((i) > 0) atomicAdd(&g_bprof[(i)], (unsigned long long)(_c - f_t0)); \
            f_t0 = _c;                                                            \
        }                                                                         \
    } while (0)
#else
#define BPROF(i) do {} while (0)
#define FPROF(i) do {} while (0)
#define TL(which, k) do {} while (0)
#endif
#ifdef MFB_FTS
__device__ long long g_fts[16 * 8];
__device__ long long g_fts2[16 * 16 * 8];
#define FTS(c, k) do { if (threadIdx.x == 0) s_fts[(c) * 8 + (k)] = clock64(); \
    if ((threadIdx.x & 31) == 0) s_fts2[((threadIdx.x >> 5) * 16 + (c)) * 8 + (k)] = clock64(); } while (0)
#else
#define FTS(c, k) do {} while (0)
#endif

namespace {

constexpr int MAX_NB = 8;
constexpr int MAX_NCY = 160;
constexpr int BAND_NB = 16;
constexpr int BAND_GROUP_MAX = 16;   // CTAs per system; panel slots = group + 1 <= 17

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

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}

// one-dimensional TMA bulk copies completing on an mbarrier
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "MFB_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra MFB_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes,
                                         unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void st_release(unsigned int *p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Factor panel kp (columns kp*NB.., rows down to the band edge) with partial
// pivoting, held in registers: thread t owns panel rows t, t+NT, .. (RPT of
// them); only the warps holding rows take part (named barrier 1).
//
// FP64 ALU latency on sm_100 is ~90 cycles, so the column loop keeps
// divisions and data movement off its dependency chain:
//  * rows never move: each row carries its logical position `pos`; a pivot
//    step only exchanges the positions of the pivot row and of the row at
//    position c (getf2's swap), and rows are written out by position;
//  * elimination is division-free (scaled, Bareiss-like): with pivot P~ and
//    pivot row u~ of step c,  a~(i,j) <- sigma (a~(i,j) P~ - a~(i,c) u~(j)),
//    sigma = 2^-e(P~) exact, so all active rows share one scale S_c
//    (S_{c+1} = sigma S_c P~, 1 <= S < 2^NB) and the pivot choice is that of
//    the unscaled matrix; afterwards L(i,c) = a~(i,c)/P~_c, U(c,j) = a~(c,j)/S_c
//    with 2*NB reciprocals computed once;
//  * argmax key = |a| bits with the low mantissa bits replaced by
//    (1023 - pos, warp): one warp redux pair, one barrier, a tree max over
//    the warps' posted keys (ties within 2^-38 go to the first position, as
//    idamax's first index); each warp posts its candidate row.
// The factors go to the band (the owner's own columns), to the publication
// slot (L rows by position, row moves, fail) and 1/U(c,c) to udinv; then
// `ready` is released to kp+1. Returns 0, or j+1 for a zero pivot at band
// column j.
template <int NT, int RPT>
__device__ __noinline__ int factor_publish(double *__restrict__ AB, int n, int kl, int ku,
                                           int ldab, int kp, double *__restrict__ slot,
                                           double *__restrict__ udinv, unsigned int *ready,
                                           double *s_cand, double *s_fin,
                                           unsigned long long *red_k, int *s_fail,
                                           double *__restrict__ Lp = nullptr) {
    constexpr int NB = BAND_NB, NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int j0 = kp * NB, pnb = min(NB, n - j0);
    const int nr = min(n, j0 + pnb + kl) - j0;
    const int nwf = RPT == 1 ? (nr + 31) >> 5 : NW;
    int fail = 0;
    double a[RPT][NB];
    int pos[RPT];
    int *spiv = reinterpret_cast<int *>(slot + (long long)(kl + NB) * NB + 2 * NB);
#ifdef MFB_PROFILE
    long long f_t0 = 0;
#endif
    FPROF(0);
    if (wid < nwf) {
#pragma unroll
        for (int rr = 0; rr < RPT; ++rr) {
            const int i = tid + rr * NT, r = j0 + i;
            pos[rr] = i < nr ? i : 0x3ff;         // 0x3ff: no row
#pragma unroll
            for (int c = 0; c < NB; ++c) {
                const int col = j0 + c;
                a[rr][c] = (i < nr && c < pnb && r - col <= kl && col - r <= kl + ku)
                               ? __ldcg(AB + bidx(r, col, kl, ku, ldab)) : 0.0;
            }
        }
#ifdef MFB_FTS
        __shared__ long long s_fts[16 * 8];
        __shared__ long long s_fts2[16 * 16 * 8];
#endif
        FPROF(12);
        double S = 1.0;                          // running row scale (thread 0)
#pragma unroll
        for (int c = 0; c < NB; ++c) {
            if (c >= pnb) {
                if (tid == 0) spiv[c] = c;
                continue;
            }
            const int par = c & 1;
            FTS(c, 0);
            unsigned long long key = 0ull;
            int crow = -1;                       // which of my rows is my key's
#pragma unroll
            for (int rr = 0; rr < RPT; ++rr) {
                const unsigned long long k2 =
                    ((unsigned long long)__double_as_longlong(a[rr][c]) & 0x7FFFFFFFFFFFC000ull) |
                    ((unsigned long long)(1023 - pos[rr]) << 4) | (unsigned long long)wid;
                if (pos[rr] >= c && pos[rr] < nr && k2 > key) { key = k2; crow = rr; }
            }
            {   // warp max: redux on the high word, then on the low word among
                // the lanes holding the high maximum
                const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
                const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
                const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
                const unsigned long long wk = ((unsigned long long)mh << 32) | ml;
                if (key != wk) crow = -1;        // not the warp's candidate
                key = wk;
            }
            FTS(c, 1);
            double *cand = s_cand + (par * NW + wid) * NB;
#pragma unroll
            for (int rr = 0; rr < RPT; ++rr)
                if (crow == rr) {
#pragma unroll
                    for (int cc = 0; cc < NB; ++cc) cand[cc] = a[rr][cc];
                }
            if (lane == 0) red_k[par * NW + wid] = key;
            FTS(c, 2);
#ifndef FB_NOBAR
            asm volatile("bar.sync 1, %0;" ::"r"(nwf * 32) : "memory");
#endif
            // max over the warps' keys: lane w reads warp w's key, one redux pair
            unsigned long long kb;
            {
                const unsigned long long kl_ = lane < nwf ? red_k[par * NW + lane] : 0ull;
                const unsigned hi = (unsigned)(kl_ >> 32), lo = (unsigned)kl_;
                const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
                const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
                kb = ((unsigned long long)mh << 32) | ml;
            }
            FTS(c, 3);
            if ((kb & ~0x3FFFull) == 0ull) { fail = j0 + c + 1; break; }   // uniform over the warps
            const int p = 1023 - (int)((kb >> 4) & 1023ull);
            if (tid == 0) spiv[c] = p;
            const double *prow = s_cand + (par * NW + (int)(kb & 15ull)) * NB;
            const double P = prow[c];
            // P' = sigma P~ in [1, 2) and sigma = 2^-e, from the bits (exact)
            const long long pbits = __double_as_longlong(P);
            const int ef = (int)((pbits >> 52) & 0x7ff);
            const bool nrm = ef > 0 && ef < 0x7ff;
            const double Pp = nrm ? __longlong_as_double((pbits & (long long)0x800FFFFFFFFFFFFFull) |
                                                         0x3FF0000000000000ll) : P;
            const double sg = nrm ? __longlong_as_double((long long)(2046 - ef) << 52) : 1.0;
            FTS(c, 4);
            if (tid == 0) {                       // the scales, for the unscaling
                s_fin[c] = P;
                s_fin[NB + c] = S;
                S = sg * S * P;
            }
#pragma unroll
            for (int rr = 0; rr < RPT; ++rr) {
                const bool active = pos[rr] > c && pos[rr] != p && pos[rr] < nr;
                const bool rowc = pos[rr] == c && p != c;    // moves to position p, stays active
#ifdef FB_NOUPD
                if (false) {
#else
                if (active || rowc) {
#endif
                    const double t = sg * a[rr][c];
                    if (c + 1 < NB) a[rr][c + 1] = fma(-t, prow[c + 1], a[rr][c + 1] * Pp);
#pragma unroll
                    for (int cc = c + 2; cc < NB; ++cc) a[rr][cc] = fma(-t, prow[cc], a[rr][cc] * Pp);
                }
                pos[rr] = pos[rr] == p ? c : (rowc ? p : pos[rr]);
            }
            FTS(c, 5);
        }
#ifdef MFB_FTS
        if (tid == 0) for (int q = 0; q < 16 * 8; ++q) g_fts[q] = s_fts[q];
        if (lane == 0) for (int q = 0; q < 16 * 8; ++q) g_fts2[wid * 128 + q] = s_fts2[wid * 128 + q];
#endif
        FPROF(13);
        // publish by position: the scaled rows a~ (rows x NB, zero past pnb),
        // then P~_c, S_c, the pivot positions and the flag; consumers unscale
        // (L = a~ / P~_c, U row c = a~ / S_c) and derive the row moves
#pragma unroll
        for (int rr = 0; rr < RPT; ++rr) {
            const int i = pos[rr];
            if (i < nr) {
#pragma unroll
                for (int c = 0; c < NB; c += 2)
                    reinterpret_cast<double2 *>(slot + i * NB)[c >> 1] = make_double2(a[rr][c], a[rr][c + 1]);
            }
        }
        double *sd = slot + (long long)(kl + NB) * NB;
        if (tid == 0) {
            spiv[NB] = fail;
            *s_fail = fail;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(nwf * 32) : "memory");   // s_fin complete
        if (tid < 2 * NB) sd[tid] = s_fin[tid];
    }
    __syncthreads();
    FPROF(14);
    if (tid == 0) {
        __threadfence();
        st_release(ready, (unsigned int)(kp + 1));
    }
    FPROF(15);
    // off the chain: the unscaled band copy (read by the back substitution,
    // after the group barrier) and 1/U(c,c)
    if (wid < nwf && !fail) {
        if (tid < 2 * NB && (tid & (NB - 1)) < pnb) s_fin[2 * NB + tid] = 1.0 / s_fin[tid];
        asm volatile("bar.sync 1, %0;" ::"r"(nwf * 32) : "memory");
#pragma unroll
        for (int rr = 0; rr < RPT; ++rr) {
            const int i = pos[rr], r = j0 + i;
            if (i < nr) {
#pragma unroll
                for (int c = 0; c < NB; ++c) {
                    const int col = j0 + c;
                    const double v = (c < pnb && c < i) ? a[rr][c] * s_fin[2 * NB + c]
                                   : (i < pnb && c >= i) ? a[rr][c] * s_fin[3 * NB + i] : a[rr][c];
                    if (c < pnb && r - col <= kl && col - r <= kl + ku) AB[bidx(r, col, kl, ku, ldab)] = v;
                    // the whole multiplier panel (rows by final position within
                    // the panel can sit further than kl below their column:
                    // the band cannot hold those, later solves need them)
                    if (Lp && c < pnb && c < i) Lp[(long long)i * NB + c] = v;
                }
            }
        }
        if (tid < pnb) udinv[j0 + tid] = s_fin[NB + tid] * s_fin[2 * NB + tid];   // S_c / P~_c
    }
    return *s_fail;
}

template <int NT>
__global__ void __launch_bounds__(NT)
band_solve_kernel(const MfbPattern *__restrict__ pats, const int *__restrict__ sys_pat,
                  const double *__restrict__ Kbuf, const long long *__restrict__ sys_koff,
                  double *__restrict__ work, const long long *__restrict__ sys_woff,
                  double *__restrict__ Xout, const long long *__restrict__ sys_xoff,
                  int *__restrict__ info, int C, unsigned int *__restrict__ bar, int keep) {
    constexpr int NB = BAND_NB;
    constexpr int PST = NB + 1;          // odd stride: lane-varying rows hit distinct banks
    constexpr int NW = NT / 32;
    extern __shared__ double smem[];
    __shared__ int s_tsrc[NB], s_ldst[NB], s_lsrc[NB];
    __shared__ double s_cinv[2 * NB];
    __shared__ unsigned long long s_bsbar[2];
    __shared__ int s_ush[2][NB];
    __shared__ int s_nlow;
    __shared__ int s_flag;
    __shared__ double s_cand[2 * NW * NB], s_fin[4 * NB];
    __shared__ unsigned long long s_fred_k[2 * NW];
    __shared__ int s_ffail;
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
    const int UST = (kl + ku + 16) | 1;  // odd: the 16 staged rows hit distinct banks
    double *AB = work + sys_woff[s];
    double *Y = AB + (long long)ldab * n;
    double *Pnl = smem;                          // (kl + NB) x PST   panel L | U11
    double *U12s = Pnl + (kl + NB) * PST;        // NB x UST          U12 of the panel
    double *Tmp = U12s + NB * UST;               // NB x UST          staged A12
    const int TMPN = max(NB * UST, 3 * MAX_NB * MAX_NCY);   // also kernel-projection scratch
    double *Ytop = Tmp + TMPN;                   // NB x ncy          rhs rows of the panel
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (kl + NB > 2 * NT) {                   // panel rows exceed two per thread
        if (tid == 0 && rank == 0) info[s] = -2;
        return;
    }

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
    // ---- 2. banded LU with partial pivoting (gbtrf), look-ahead over the group
    // Column block b (NB columns) belongs to rank b % C, which applies every
    // panel's row swaps and updates to it. The owner of block k+1 updates that
    // block first when panel k arrives, factors panel k+1 and publishes it
    // (slot (k+1) % D + release of `ready`), and only then updates the rest of
    // its columns, so the panel chain does not wait for the trailing updates.
    // D = C + 1 slots suffice: a rank loads panel k before it can publish any
    // later panel, and the owners of panels k+1..k+C cover every rank.
    const int nblk = (n + NB - 1) / NB;
    const int D = C + 1, D_MAX = BAND_GROUP_MAX + 1;
    const long long SLOT = (long long)(kl + NB) * NB + 48;   // rows, P~ and S, 32 ints
    double *slots = Y + ny + ((ldab * (long long)n + ny) & 1);   // 16-byte aligned (double2 stores)
    double *udinv = slots + D_MAX * SLOT;          // 1 / U(j, j), written by the panel owners
    // inverses of the diagonal 16 x 16 U blocks (back substitution), 16-byte aligned
    double *u11inv = udinv + n + ((reinterpret_cast<uintptr_t>(udinv + n) & 15) ? 1 : 0);
    // the panels' pivot positions, kept for later solves with these factors
    // (mfb_systems_apply: Method S1's matrix-free star solves)
    int *piv = reinterpret_cast<int *>(u11inv + (long long)NB * NB * ((n + NB - 1) / NB));
    // the multiplier panels, (kl + NB) x NB each, rows by final position
    double *Lpan = reinterpret_cast<double *>(piv) + ((n + 1) / 2 + 1);
    unsigned int *ready = bar + gridDim.x / C + s;
    const int NTF = kl + NB <= NT ? 1 : 2;
    auto factor = [&](int kp) -> int {
        double *slot = slots + (kp % D) * SLOT;
        double *Lp = keep ? Lpan + (long long)kp * (kl + NB) * NB : nullptr;
        const int f = NTF == 1 ? factor_publish<NT, 1>(AB, n, kl, ku, ldab, kp, slot, udinv,
                                                       ready, s_cand, s_fin, s_fred_k, &s_ffail,
                                                       Lp)
                               : factor_publish<NT, 2>(AB, n, kl, ku, ldab, kp, slot, udinv,
                                                       ready, s_cand, s_fin, s_fred_k, &s_ffail,
                                                       Lp);
        if (keep && tid == 0) {  // written by this thread inside factor_publish
            const int *sp = reinterpret_cast<const int *>(slot + (long long)(kl + NB) * NB + 2 * NB);
            for (int c = 0; c < NB && kp * NB + c < n; ++c) piv[kp * NB + c] = sp[c];
        }
        return f;
    };
#define OWNB(b) (((b) % C) == rank)
    if (rank == 0) {
        const int f = factor(0);
        if (f) {
            if (tid == 0) info[s] = f;
            return;
        }
    }
    for (int k = 0; k < nblk; ++k) {
        BPROF(0);
        const int j0 = k * NB;
        const int pnb = min(NB, n - j0);
        const int r1 = min(n, j0 + pnb + kl);
        const int nr = r1 - j0;
        const int c0 = j0 + pnb;
        const int c1 = min(n, j0 + pnb + kl + ku);
        if (k + 1 < nblk && OWNB(k + 1)) TL(3, k);
        if (tid == 0)
            while (ld_acquire(ready) < (unsigned int)(k + 1)) {}
        __syncthreads();
        const double *slot = slots + (k % D) * SLOT;
        const double *sd = slot + (long long)(kl + NB) * NB;
        const int *si = reinterpret_cast<const int *>(sd + 2 * NB);
        for (int t0 = tid; t0 < nr * NB; t0 += 8 * NT) {     // eight loads in flight
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = t0 + u * NT < nr * NB ? __ldcg(slot + t0 + u * NT) : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int t = t0 + u * NT;
                if (t < nr * NB) Pnl[(t >> 4) * PST + (t & (NB - 1))] = v[u];
            }
        }
        if (wid == 0) {
            // reciprocal scales 1/P~_c (lanes 0..15) and 1/S_c (16..31)
            const double sv = __ldcg(sd + lane);
            s_cinv[lane] = (lane & (NB - 1)) < pnb ? 1.0 / sv : 0.0;
            // row moves of the panel's swaps: final top row q holds the row
            // found by undoing the swaps; each distinct pivot row below the
            // panel receives a top row (getf2 swap order)
            int pv[NB];
#pragma unroll
            for (int c = 0; c < NB; ++c) pv[c] = __ldcg(si + c);
            const int q = lane & (NB - 1);
            int x = q;
#pragma unroll
            for (int c = NB - 1; c >= 0; --c)
                if (c < pnb) x = (x == c) ? pv[c] : (x == pv[c] ? c : x);
            int pz = 0;
            bool lowv = false;
#pragma unroll
            for (int c = 0; c < NB; ++c)
                if (c == q) { pz = pv[c]; lowv = c < pnb && pv[c] >= pnb; }
#pragma unroll
            for (int c = 0; c < NB; ++c)
                if (c < q && pv[c] == pz) lowv = false;
            int y = pz;
#pragma unroll
            for (int c = NB - 1; c >= 0; --c)
                if (c < pnb) y = (y == c) ? pv[c] : (y == pv[c] ? c : y);
            const unsigned m = __ballot_sync(0xffffffffu, lane < NB && lowv);
            const int zp = __popc(m & ((1u << q) - 1u));
            if (lane < NB) {
                s_tsrc[lane] = x;
                if (lowv) {
                    s_ldst[zp] = pz;
                    s_lsrc[zp] = y;
                }
            }
            if (lane == 0) {
                s_nlow = __popc(m);
                s_flag = __ldcg(si + NB);
            }
        }
        __syncthreads();
        if (!s_flag)
            for (int t = tid; t < nr * NB; t += NT) {
                const int i = t >> 4, c = t & (NB - 1);
                if (c < pnb && c < i) Pnl[i * PST + c] *= s_cinv[c];
                else if (i < pnb && c >= i) Pnl[i * PST + c] *= s_cinv[NB + i];
            }
        __syncthreads();
        if (s_flag) return;                  // the panel's owner set info[s]
        BPROF(1);
        const int nlow = s_nlow;

        // swaps + U12 + trailing update of the owned blocks in [blo, bhi]
        auto update_blocks = [&](int blo, int bhi) {
            if (blo > bhi) return;
            const int bf0 = blo + ((rank - blo) % C + C) % C;
            if (bf0 > bhi) return;
            const int nob = (bhi - bf0) / C + 1;
            const int nel = nob * NB * NB;
            // stage the permuted top rows (Tmp) and the moved lower rows (U12s)
            for (int t = tid; t < nel; t += NT) {
                const int q = t & (NB - 1), c16 = (t >> 4) & (NB - 1), ob = t >> 8;
                const int col = (bf0 + ob * C) * NB + c16, cc = col - c0;
                const int src = j0 + (q < pnb ? s_tsrc[q] : 0);
                const bool vt = q < pnb && col < c1 && col - src <= kl + ku && src - col <= kl;
                const int srl = j0 + (q < nlow ? s_lsrc[q] : 0);
                const bool vl = q < nlow && col < c1 && col - srl <= kl + ku && srl - col <= kl;
                const double x = vt ? AB[bidx(src, col, kl, ku, ldab)] : 0.0;
                const double y = vl ? AB[bidx(srl, col, kl, ku, ldab)] : 0.0;
                Tmp[q * UST + cc] = x;
                U12s[q * UST + cc] = y;
            }
            __syncthreads();
            BPROF(8);
            for (int t = tid; t < nel; t += NT) {
                const int z = t & (NB - 1), c16 = (t >> 4) & (NB - 1), ob = t >> 8;
                if (z >= nlow) continue;
                const int col = (bf0 + ob * C) * NB + c16, cc = col - c0;
                const int row = j0 + s_ldst[z];
                if (col < c1 && row - col <= kl) AB[bidx(row, col, kl, ku, ldab)] = U12s[z * UST + cc];
            }
            __syncthreads();
            BPROF(9);
            // U12 = L11^-1 A12 by forward substitution (thread per column)
            for (int u = tid; u < nob * NB; u += NT) {
                const int col = (bf0 + (u >> 4) * C) * NB + (u & (NB - 1)), cc = col - c0;
                double uu[NB];
#pragma unroll
                for (int q = 0; q < NB; ++q) uu[q] = Tmp[q * UST + cc];
                // column-oriented (axpy) order: dependent chain NB deep, not NB^2/2
#pragma unroll
                for (int qq = 0; qq < NB - 1; ++qq)
#pragma unroll
                    for (int q = qq + 1; q < NB; ++q) uu[q] -= Pnl[q * PST + qq] * uu[qq];
#pragma unroll
                for (int q = 0; q < NB; ++q) uu[q] = q < pnb ? uu[q] : 0.0;
#pragma unroll
                for (int q = 0; q < NB; ++q) {
                    U12s[q * UST + cc] = q < pnb ? uu[q] : 0.0;
                    const int row = j0 + q;
                    if (q < pnb && col < c1 && col - row <= kl + ku) AB[bidx(row, col, kl, ku, ldab)] = uu[q];
                }
            }
            __syncthreads();
            BPROF(10);
            // A22 -= L21 U12 on FP64 tensor cores (DMMA 8x8x4); work item =
            // (8-column tile, group of four 8-row tiles), U12 fragments in registers
            const int mrows = nr - pnb;
            const int tr = (mrows + 7) >> 3, nrg = (tr + 3) >> 2, ntc = 2 * nob;
            const int g = lane >> 2, q4 = lane & 3;
            for (int it = wid; it < ntc * nrg; it += NW) {
                const int rg = it / ntc, ot = it - rg * ntc;
                const int col8 = (bf0 + (ot >> 1) * C) * NB + (ot & 1) * 8;
                const int cct = col8 - c0;
                double bf[NB / 4];
#pragma unroll
                for (int kk = 0; kk < NB / 4; ++kk) bf[kk] = U12s[(4 * kk + q4) * UST + cct + g];
                const int ca = col8 + 2 * q4, cb = ca + 1;
                double *pa = AB + (long long)ca * ldab + (kl + ku - ca);
                double *pb = pa + (ldab - 1);
                const int lima = ca < c1 ? min(r1, ca + kl + 1) : 0;
                const int limb = cb < c1 ? min(r1, cb + kl + 1) : 0;
                const int rbase = j0 + pnb + g;
                const int tg = rg * 4;
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
            __syncthreads();
            BPROF(11);
        };

        const int bend = c1 > c0 ? (c1 - 1) / NB : k;
        if (k + 1 < nblk && OWNB(k + 1)) {
            TL(0, k);
            update_blocks(k + 1, k + 1);
            TL(1, k);
            BPROF(2);
            const int f = factor(k + 1);
            TL(2, k);
            if (f) {
                if (tid == 0) info[s] = f;
                return;
            }
            BPROF(3);
            update_blocks(k + 2, bend);
        } else {
            update_blocks(k + 1, bend);
        }
        BPROF(4);
        // right-hand sides: permute + forward substitution (thread per column)
        for (int cy = tid; cy < ncy; cy += NT) {
            if (!OWN(cy >> 3)) continue;
            double u[NB], low[NB];
#pragma unroll
            for (int q = 0; q < NB; ++q)
                u[q] = q < pnb ? Y[(long long)(j0 + s_tsrc[q]) * ncy + cy] : 0.0;
#pragma unroll
            for (int z = 0; z < NB; ++z)
                low[z] = z < nlow ? Y[(long long)(j0 + s_lsrc[z]) * ncy + cy] : 0.0;
#pragma unroll
            for (int z = 0; z < NB; ++z)
                if (z < nlow) Y[(long long)(j0 + s_ldst[z]) * ncy + cy] = low[z];
#pragma unroll
            for (int qq = 0; qq < NB - 1; ++qq)
#pragma unroll
                for (int q = qq + 1; q < NB; ++q) u[q] -= Pnl[q * PST + qq] * u[qq];
#pragma unroll
            for (int q = 0; q < NB; ++q) {
                if (q < pnb) Y[(long long)(j0 + q) * ncy + cy] = u[q];
                Ytop[q * ncy + cy] = q < pnb ? u[q] : 0.0;
            }
        }
        __syncthreads();
        // rhs rows below the panel, Y -= L21 Ytop (DMMA tiles; a warp owns a
        // row tile and keeps its L21 fragments in registers)
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
        __syncthreads();
        BPROF(5);
    }
#undef OWNB
    // every rank's factors and rhs updates in place before the back substitution
    group_sync(ctr, C, bar_target);

    // ---- 2b. inverses of the diagonal U blocks, all blocks in parallel ------
    // The back substitution's per-panel triangular solve is a chain of 2 NB
    // dependent FP64 operations (~90 cycles each on sm_100); with U11^-1 it
    // becomes independent 16-term dot products. Column c of U11^-1 solves
    // U11 y = e_c (rows c..0), one thread per (block, column).
    {
        const int nblk2 = (n + NB - 1) / NB;
        for (int t = rank * NT + tid; t < nblk2 * NB; t += C * NT) {
            const int b = t / NB, c = t % NB, j0 = b * NB;
            const int pn = min(NB, n - j0);
            double y[NB];
#pragma unroll
            for (int r = 0; r < NB; ++r) y[r] = 0.0;
            if (c < pn) {
                y[c] = __ldcg(udinv + j0 + c);
#pragma unroll
                for (int r = NB - 1; r >= 0; --r) {
                    if (r >= c || r >= pn) continue;
                    double acc = 0.0;
#pragma unroll
                    for (int q = r + 1; q < NB; ++q)
                        if (q <= c) acc = fma(__ldcg(AB + bidx(j0 + r, j0 + q, kl, ku, ldab)), y[q], acc);
                    y[r] = -acc * __ldcg(udinv + j0 + r);
                }
            }
            double *dst = u11inv + (long long)b * NB * NB;
#pragma unroll
            for (int r = 0; r < NB; ++r) dst[r * NB + c] = y[r];
        }
    }
    group_sync(ctr, C, bar_target);


    // ---- 3. back substitution U x = y, per owned rhs tile of 8 columns -----
    // The tile's active rows live in a circular shared-memory window (the
    // panel being solved and the kl+ku rows above it that its solution
    // updates). The U block above each diagonal block is copied global ->
    // shared by TMA bulk copies (one per column, mbarrier completion) one
    // panel ahead into a double buffer, so the copy overlaps the previous
    // panel's solve and push; the push Y -= U x is DMMA from shared memory;
    // the next U11 and the rows entering the window are staged a panel ahead.
    {
        const int last = ((n - 1) / NB) * NB;
        const int WR = kl + ku + 2 * NB;             // window rows (circular)
        const int LDU = ((kl + ku + 8 + 7) & ~7) + 4;   // U block column stride
        double *Yw = smem;                           // WR x 8
        double *Ub2 = Yw + WR * 8;                   // 2 x NB x LDU (column k, row i - i0)
        double *Xs = Ub2 + 2 * NB * LDU;             // NB x 8 solved panel rows
        double *U11b = Xs + NB * 8;                  // 2 x NB x NB (diagonal: 1/U(r,r))
        const int tcy = (ncy + 7) >> 3;
        const int g = lane >> 2, q4 = lane & 3;
        if (tid == 0) {
            mbar_init(&s_bsbar[0], 1);
            mbar_init(&s_bsbar[1], 1);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        unsigned bsphase[2] = {0u, 0u};
        // U(i0..jj-1, jj..jj+pn-1) -> buffer b: a contiguous run of the band per
        // column, started one element early when odd (16-byte aligned ends)
        // issued by the 16 lanes of warp 0, one column each: lane 0 posts the
        // transaction count (warp sum of the column byte counts) before any
        // copy is issued
        auto issue_u = [&](int jj, int b) {
            if (tid >= 32) return;
            const int pn = min(NB, n - jj), ii0 = max(0, jj - kl - ku), mr = jj - ii0;
            const int k = tid;
            unsigned bytes = 0;
            const double *src = AB;
            if (k < NB) {
                const long long off = (long long)(jj + k) * ldab + (kl + ku + ii0 - (jj + k));
                const int sh = (int)(off & 1);
                s_ush[b][k] = sh;
                src = AB + off - sh;
                bytes = (k < pn && mr > 0) ? (unsigned)(((mr + sh + 1) & ~1) * 8) : 0u;
            }
            unsigned tot = bytes;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (tid == 0) mbar_arrive_expect_tx(&s_bsbar[b], tot);
            __syncwarp();
            if (bytes) bulk_g2s(Ub2 + (b * NB + k) * LDU, src, bytes, &s_bsbar[b]);
        };
        auto u11_load = [&](int jj, double *dst) {        // U11^-1 of the block at jj
            const double *src = u11inv + (long long)(jj / NB) * NB * NB;
            for (int t = tid; t < NB * NB; t += NT) dst[t] = __ldcg(src + t);
        };
        if (rank < tcy) __syncthreads();             // smem reuse after the LU loop
        for (int tc = rank; tc < tcy; tc += C) {
            const int cb0 = tc * 8;
            const int rlo = max(0, last - kl - ku);
            issue_u(last, 0);
            for (int t = tid; t < (n - rlo) * 8; t += NT) {
                const int r = rlo + (t >> 3), c = t & 7;
                Yw[(r % WR) * 8 + c] = cb0 + c < ncy ? Y[(long long)r * ncy + cb0 + c] : 0.0;
            }
            u11_load(last, U11b);
            __syncthreads();
            int buf = 0;
            for (int j0 = last; j0 >= 0; j0 -= NB) {
                BPROF(16);
                const int pnb = min(NB, n - j0);
                const int i0 = max(0, j0 - kl - ku);
                const int mrows = j0 - i0;
                const double *u11 = U11b + buf * NB * NB;
                const double *Ub = Ub2 + buf * NB * LDU;
                const int *ush = s_ush[buf];
                // the next panel's U block into the other buffer (its last
                // reader, the previous push, finished at the loop-end barrier)
                if (j0 > 0) issue_u(j0 - NB, buf ^ 1);
                BPROF(17);
                // rows entering the window for the next panel, and its U11
                if (j0 > 0) {
                    const int ni0 = max(0, j0 - NB - kl - ku), nbase = ni0 % WR;
                    for (int t = tid; t < (i0 - ni0) * 8; t += NT) {
                        const int r = ni0 + (t >> 3), c = t & 7;
                        int w = nbase + (t >> 3);
                        if (w >= WR) w -= WR;
                        Yw[w * 8 + c] = cb0 + c < ncy ? Y[(long long)r * ncy + cb0 + c] : 0.0;
                    }
                    u11_load(j0 - NB, U11b + (buf ^ 1) * NB * NB);
                }
                BPROF(18);
                // panel rows x = U11^-1 y: one thread per (row, column), a
                // 16-term dot product with four accumulators
                const int jbase = j0 % WR, ibase = i0 % WR;    // window slots of j0, i0
                if (tid < NB * 8) {
                    const int r = tid >> 3, c = tid & 7;
                    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
                    for (int q = 0; q < NB; q += 4) {
                        int w = jbase + q;
                        if (w >= WR) w -= WR;
                        int w1 = w + 1, w2 = w + 2, w3 = w + 3;
                        if (w1 >= WR) w1 -= WR;
                        if (w2 >= WR) w2 -= WR;
                        if (w3 >= WR) w3 -= WR;
                        a0 = fma(u11[r * NB + q], q < pnb ? Yw[w * 8 + c] : 0.0, a0);
                        a1 = fma(u11[r * NB + q + 1], q + 1 < pnb ? Yw[w1 * 8 + c] : 0.0, a1);
                        a2 = fma(u11[r * NB + q + 2], q + 2 < pnb ? Yw[w2 * 8 + c] : 0.0, a2);
                        a3 = fma(u11[r * NB + q + 3], q + 3 < pnb ? Yw[w3 * 8 + c] : 0.0, a3);
                    }
                    const double x = r < pnb ? (a0 + a1) + (a2 + a3) : 0.0;
                    Xs[r * 8 + c] = x;
                    if (r < pnb && cb0 + c < ncy) Y[(long long)(j0 + r) * ncy + cb0 + c] = x;
                }
                mbar_wait(&s_bsbar[buf], bsphase[buf]);
                bsphase[buf] ^= 1u;
                __syncthreads();
                BPROF(19);
                // push: Yw[i] -= U(i, panel) x_panel for i in [i0, j0) (DMMA)
                const int tr = (mrows + 7) >> 3;
                for (int ti = wid; ti < tr; ti += NW) {
                    const int il = ti * 8 + g, i = i0 + il;
                    const bool ri = il < mrows;
                    int w = ibase + (ri ? il : 0);
                    if (w >= WR) w -= WR;
                    double *yr = Yw + w * 8 + 2 * q4;
                    double d0 = ri ? yr[0] : 0.0, d1 = ri ? yr[1] : 0.0;
#pragma unroll
                    for (int kk = 0; kk < NB / 4; ++kk) {
                        const int k = 4 * kk + q4;
                        const double a = (ri && k < pnb && (j0 + k) - i <= kl + ku)
                                             ? -Ub[k * LDU + ush[k] + il] : 0.0;
                        dmma884(d0, d1, a, Xs[k * 8 + g]);
                    }
                    if (ri) {
                        yr[0] = d0;
                        yr[1] = d1;
                    }
                }
                __syncthreads();
                BPROF(20);
                buf ^= 1;
            }
        }
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
    const int t0 = blockIdx.y * NT + threadIdx.x, TS = gridDim.y * NT;   // CTAs split outputs
    if (blocks || hbar) {
        for (int t = t0; t < nd * nrhs; t += TS) {
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
        for (long long t = t0; t < (long long)P.nfield * nrhs; t += TS) {
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
                       const long long *sys_xoff, int *info, unsigned int *bar, int keep) {
    if (cudaFuncSetAttribute(band_solve_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return MFB_ERR_SMEM;
    // bar: n_sys group-barrier counters, then n_sys panel-ready counters
    if (cudaMemsetAsync(bar, 0, sizeof(unsigned int) * 2 * n_sys, st) != cudaSuccess)
        return MFB_ERR_LAUNCH;
    if (C == 1) {
        band_solve_kernel<NT><<<n_sys, NT, smem, st>>>(pats, sys_pat, Kbuf, sys_koff, work,
                                                       sys_woff, X, sys_xoff, info, C, bar,
                                                       keep);
    } else {
        // the C CTAs of a system wait on one another: cooperative launch
        // guarantees they are co-resident
        void *args[] = {(void *)&pats, (void *)&sys_pat, (void *)&Kbuf, (void *)&sys_koff,
                        (void *)&work, (void *)&sys_woff, (void *)&X, (void *)&sys_xoff,
                        (void *)&info, (void *)&C, (void *)&bar, (void *)&keep};
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
                                 int smem_doubles, int group, unsigned int *bar,
                                 int keep_factors, void *stream) {
    if (n_sys <= 0) return n_sys == 0 ? MFB_OK : MFB_ERR_ARG;
    if (group < 1 || group > BAND_GROUP_MAX || bar == nullptr) return MFB_ERR_ARG;
    const size_t smem = (size_t)smem_doubles * sizeof(double);
    cudaStream_t st = mfb_stream(stream);
    switch (threads) {
        case 256: return launch_band<256>(n_sys, group, smem, st, pats, sys_pat, Kbuf, sys_koff,
                                          work, sys_woff, X, sys_xoff, info, bar,
                                          keep_factors);
        case 384: return launch_band<384>(n_sys, group, smem, st, pats, sys_pat, Kbuf, sys_koff,
                                          work, sys_woff, X, sys_xoff, info, bar,
                                          keep_factors);
        default: return MFB_ERR_ARG;
    }
}

extern "C" int mfb_debug_timeline(unsigned long long *out) {
#ifdef MFB_PROFILE
    return cudaMemcpyFromSymbol(out, g_tl, sizeof(unsigned long long) * 4 * 4096) == cudaSuccess ? 0 : 2;
#else
    (void)out;
    return 1;
#endif
}

extern "C" int mfb_debug_bprof(unsigned long long *out) {
#ifdef MFB_PROFILE
    return cudaMemcpyFromSymbol(out, g_bprof, sizeof(unsigned long long) * 24) == cudaSuccess ? 0 : 2;
#else
    (void)out;
    return 1;
#endif
}

// B <- (B + B^T) / 2 for every system's basis block (one CTA per block)
__global__ void symmetrize_kernel(const MfbPattern *__restrict__ pats,
                                  const int *__restrict__ sys_pat, double *__restrict__ blocks,
                                  const long long *__restrict__ sys_boff) {
    const int s = blockIdx.x, nd = pats[sys_pat[s]].ndof;
    double *B = blocks + sys_boff[s];
    for (int e = threadIdx.x; e < nd * nd; e += blockDim.x) {
        const int r = e / nd, c = e - r * nd;
        if (r < c) {
            const double v = 0.5 * (B[r * nd + c] + B[c * nd + r]);
            B[r * nd + c] = v;
            B[c * nd + r] = v;
        }
    }
}

extern "C" int mfb_blocks_symmetrize(const MfbPattern *pats, int n_sys, const int *sys_pat,
                                     double *blocks, const long long *sys_boff, void *stream) {
    if (n_sys <= 0) return n_sys == 0 ? MFB_OK : MFB_ERR_ARG;
    symmetrize_kernel<<<n_sys, 256, 0, mfb_stream(stream)>>>(pats, sys_pat, blocks, sys_boff);
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
    // few systems (Stokes) get many CTAs each; many systems need no split
    const int split = n_sys >= 148 ? 1 : (n_sys >= 37 ? 4 : 32);
    extract_kernel<256><<<dim3(n_sys, split), 256, 0, mfb_stream(stream)>>>(
        pats, sys_pat, X, sys_xoff, blocks, sys_boff, hbar, sys_hoff, M, sys_moff, Fb,
        sys_fboff);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}
