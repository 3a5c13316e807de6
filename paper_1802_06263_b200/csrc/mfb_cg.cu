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
#include <stdint.h>

#ifdef MFB_PROFILE
__device__ unsigned long long g_cgprof[8];
#define CGP(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) { long long _c = clock64(); \
    if ((i) > 0) g_cgprof[(i)] += (unsigned long long)(_c - cg_t0); cg_t0 = _c; } } while (0)
#else
#define CGP(i) do {} while (0)
#endif

namespace {

constexpr int CG_NT_MAX = 1024;

// one row of a column-major nd x nd basis block against the gathered p:
// four independent accumulators, 32-bit strides
__device__ __forceinline__ double row_dot(const double *__restrict__ B, int meta,
                                          const int *__restrict__ sdm,
                                          const double *__restrict__ p) {
    const int nd = meta >> 20;
    const int *dm = sdm + (meta & 0xFFFFF);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int c = 0;
    for (; c + 4 <= nd; c += 4, B += 4 * nd) {
        a0 = fma(B[0], p[dm[c]], a0);
        a1 = fma(B[nd], p[dm[c + 1]], a1);
        a2 = fma(B[2 * nd], p[dm[c + 2]], a2);
        a3 = fma(B[3 * nd], p[dm[c + 3]], a3);
    }
    for (; c < nd; ++c, B += nd) a0 = fma(B[0], p[dm[c]], a0);
    return (a0 + a1) + (a2 + a3);
}

// same with p already gathered into the stacked row space (pr = p_rows + d0)
__device__ __forceinline__ double row_dot_r(const double *__restrict__ B, int nd,
                                            const double *__restrict__ pr) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int c = 0;
#pragma unroll 2
    for (; c + 4 <= nd; c += 4, B += 4 * nd) {
        a0 = fma(B[0], pr[c], a0);
        a1 = fma(B[nd], pr[c + 1], a1);
        a2 = fma(B[2 * nd], pr[c + 2], a2);
        a3 = fma(B[3 * nd], pr[c + 3], a3);
    }
    for (; c < nd; ++c, B += nd) a0 = fma(B[0], pr[c], a0);
    return (a0 + a1) + (a2 + a3);
}

// Row r of the stacked basis blocks (r in [0, dof_ptr[n_sub]) enumerates every
// (subdomain i, local mortar dof a)) is owned by thread r mod blockDim; its
// per-point metadata lives in shared memory: the block column base, the dof
// list offset, nd and the output dof. When `stage` > 0 the point's blocks
// (stage = sum_i nd_i^2 doubles) and the dof lists are copied to shared
// memory once, so every iteration's GEMV reads shared memory only; the row's
// dot product runs with four independent accumulators.
__global__ void __launch_bounds__(CG_NT_MAX)
cg_kernel(int n_lambda, int n_sub, const int *__restrict__ ndof,
          const int *__restrict__ dof_ptr, const int *__restrict__ dof_map,
          const int *__restrict__ region, const long long *__restrict__ blk_base,
          const long long *__restrict__ h_base, const int *__restrict__ local_idx,
          int n_real, const double *__restrict__ blocks, const double *__restrict__ hbar,
          int k0, double tol, int max_iter, double *__restrict__ lam_out,
          int *__restrict__ iters_out, int *__restrict__ status_out,
          double *__restrict__ res_hist, int hist_cap, double *__restrict__ g_out,
          long long stage, int use_prow) {
    extern __shared__ double sm[];
    __shared__ double red2[2 * (CG_NT_MAX / 32)];   // alternating reduction buffers
    int rbuf = 0;
    const int NT = blockDim.x;
    const int nrows = dof_ptr[n_sub];
    if (nrows > 2 * n_lambda) __trap();      // shared layout assumes two sides per dof
    double *x = sm;
    double *r = x + n_lambda;
    double *p = r + n_lambda;
    double *Sp = p + n_lambda;
    double *sB = Sp + n_lambda;                                       // staged blocks
    double *rowval = sB + stage;                                      // row results
    double *prow = rowval + nrows;                                    // p in row space
    int *rb = reinterpret_cast<int *>(prow + (use_prow ? nrows : 0)); // block base + a
    int *rmeta = rb + nrows;                                          // dof offset | nd << 20
    int *sdm = rmeta + nrows;                                         // dof lists (no prow)
    int *sbo = sdm + (use_prow ? 0 : nrows);                          // staged block offsets
    int *side0 = sbo + n_sub;                                         // rows of dof d
    int *side1 = side0 + n_lambda;
    const int pt = blockIdx.x;
    const int k = k0 + pt;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

    // ---- per-point row metadata and rhs g = sum_i scatter(h_{i, loc_i(k)}) --
    for (int d = tid; d < n_lambda; d += NT) { x[d] = 0.0; r[d] = 0.0; }
    if (stage > 0 && tid == 0) {
        int o = 0;
        for (int i = 0; i < n_sub; ++i) {
            sbo[i] = o;
            o += ndof[i] * ndof[i];
        }
    }
    if (!use_prow)
        for (int d = tid; d < nrows; d += NT) sdm[d] = dof_map[d];
    for (int d = tid; d < n_lambda; d += NT) { side0[d] = 0x7fffffff; side1[d] = -1; }
    __syncthreads();
    for (int row = tid; row < nrows; row += NT) {
        atomicMin(&side0[dof_map[row]], row);
        atomicMax(&side1[dof_map[row]], row);
    }
    for (int i = wid; i < n_sub; i += NT / 32) {
        const int nd = ndof[i], d0 = dof_ptr[i];
        const int loc = region[i] < 0 ? 0 : local_idx[(long long)region[i] * n_real + k];
        const long long bb = blk_base[i] + (long long)loc * nd * nd;
        if (stage > 0) {
            const double *src = blocks + bb;
            double *dst = sB + sbo[i];
            for (int e = lane; e < nd * nd; e += 32) dst[e] = src[e];
        }
        for (int a = lane; a < nd; a += 32) {
            rb[d0 + a] = (int)((stage > 0 ? sbo[i] : bb) + a);
            rmeta[d0 + a] = d0 | (nd << 20);
        }
    }
    __syncthreads();
    for (int i = wid; i < n_sub; i += NT / 32) {
        const int nd = ndof[i];
        const int loc = region[i] < 0 ? 0 : local_idx[(long long)region[i] * n_real + k];
        const double *h = hbar + h_base[i] + (long long)loc * nd;
        const int *dm = dof_map + dof_ptr[i];
        for (int a = lane; a < nd; a += 32) atomicAdd(&r[dm[a]], h[a]);
    }
    __syncthreads();
    double *lam = lam_out + (long long)pt * n_lambda;
    if (g_out)
        for (int d = tid; d < n_lambda; d += NT) g_out[(long long)pt * n_lambda + d] = r[d];
    double part = 0.0;
    for (int d = tid; d < n_lambda; d += NT) {
        p[d] = r[d];
        if (use_prow) {
            prow[side0[d]] = r[d];
            prow[side1[d]] = r[d];
        }
        part += r[d] * r[d];
    }
    __syncthreads();
    double rr = block_sum_alt(part, red2, rbuf);
    const double gnorm = sqrt(rr);
    if (gnorm == 0.0) {
        for (int d = tid; d < n_lambda; d += NT) lam[d] = 0.0;
        if (tid == 0) { iters_out[pt] = 0; status_out[pt] = MFB_CG_ZERO_RHS; }
        return;
    }
    double *hist = res_hist + (long long)pt * hist_cap;
    int status = MFB_CG_MAX_ITER, it_done = max_iter;
#ifdef MFB_PROFILE
    long long cg_t0 = 0;
#endif
    for (int it = 1; it <= max_iter; ++it) {
        CGP(0);
        // ---- Sp = sum_i scatter(B_i p_i): row results, then each dof adds
        // its two sides (0 + a + b of basis_apply, order free in IEEE) ------
        __syncthreads();                         // p of the previous iteration
        CGP(1);
        if (use_prow) {
            const double *Bs = stage > 0 ? sB : blocks;
            for (int row = tid; row < nrows; row += NT) {
                const int meta = rmeta[row];
                rowval[row] = row_dot_r(Bs + rb[row], meta >> 20, prow + (meta & 0xFFFFF));
            }
        } else if (stage > 0) {
            for (int row = tid; row < nrows; row += NT)
                rowval[row] = row_dot(sB + rb[row], rmeta[row], sdm, p);
        } else {
            for (int row = tid; row < nrows; row += NT)
                rowval[row] = row_dot(blocks + rb[row], rmeta[row], sdm, p);
        }
        __syncthreads();
        part = 0.0;
        for (int d = tid; d < n_lambda; d += NT) {
            const int s0 = side0[d], s1 = side1[d];
            const double v = s1 != s0 ? rowval[s0] + rowval[s1] : rowval[s0];
            Sp[d] = v;
            part += p[d] * v;
        }
        CGP(2);
        const double pSp = block_sum_alt(part, red2, rbuf);
        CGP(3);
        if (!(pSp > 0.0)) {
            status = MFB_CG_NOT_SPD;
            it_done = it;
            break;
        }
        const double a = rr / pSp;
        part = 0.0;
        for (int d = tid; d < n_lambda; d += NT) {
            const double rd = __dsub_rn(r[d], __dmul_rn(a, Sp[d]));
            r[d] = rd;
            part += rd * rd;
        }
        CGP(4);
        const double rr_new = block_sum_alt(part, red2, rbuf);
        CGP(5);
        for (int d = tid; d < n_lambda; d += NT) x[d] = __dadd_rn(x[d], __dmul_rn(a, p[d]));   // p still this iteration's
        const double rn = sqrt(rr_new);
        // rn now, rn / gnorm after the loop (keeps the division off the chain)
        if (tid == 0 && it <= hist_cap) hist[it - 1] = rn;
        if (rn <= tol * gnorm) {
            status = MFB_CG_CONVERGED;
            it_done = it;
            break;
        }
        const double beta = rr_new / rr;
        for (int d = tid; d < n_lambda; d += NT) {
            const double pd = __dadd_rn(r[d], __dmul_rn(beta, p[d]));
            p[d] = pd;
            if (use_prow) {
                prow[side0[d]] = pd;
                prow[side1[d]] = pd;
            }
        }
        rr = rr_new;
        CGP(6);
    }
    for (int d = tid; d < n_lambda; d += NT) lam[d] = x[d];
    if (tid == 0) { iters_out[pt] = it_done; status_out[pt] = status; }
    __syncthreads();                              // tid 0's rn entries
    const int nh = min(status == MFB_CG_NOT_SPD ? it_done - 1 : it_done, hist_cap);
    for (int j = tid; j < nh; j += NT) hist[j] = hist[j] / gnorm;
}



// Register rows, paired: thread 2d + side holds the block row of mortar dof
// d's lower (side 0) or upper (side 1) subdomain in registers, so S p[d] =
// row_lower + row_upper is one shuffle inside the warp (basis_apply's
// ascending-sid scatter from zero; an absent side is an all-zero row), and
// x, r, p of dof d live in the even thread's registers. Per iteration: one
// barrier for p, the GEMV from registers against p in row space (shared
// memory), and the two reductions -- three barriers in all.
template <int RN>
__global__ void __launch_bounds__(608)
cg_pair_kernel(int n_lambda, int n_sub, const int *__restrict__ ndof,
               const int *__restrict__ dof_ptr, const int *__restrict__ dof_map,
               const int *__restrict__ region, const long long *__restrict__ blk_base,
               const long long *__restrict__ h_base, const int *__restrict__ local_idx,
               int n_real, const double *__restrict__ blocks, const double *__restrict__ hbar,
               int k0, double tol, int max_iter, double *__restrict__ lam_out,
               int *__restrict__ iters_out, int *__restrict__ status_out,
               double *__restrict__ res_hist, int hist_cap, double *__restrict__ g_out) {
    extern __shared__ double sm[];
    __shared__ double red2[2 * (CG_NT_MAX / 32)];
    int rbuf = 0;
    const int NT = blockDim.x;
    const int nrows = dof_ptr[n_sub];
    double *r0 = sm;                                            // rhs assembly, n_lambda
    double *prow = r0 + n_lambda;                               // p in row space (+RN pad)
    long long *rb = reinterpret_cast<long long *>(prow + nrows + RN);   // block row base
    int *rmeta = reinterpret_cast<int *>(rb + nrows);           // dof offset | nd << 20
    int *side0 = rmeta + nrows;                                 // rows of dof d
    int *side1 = side0 + n_lambda;
    const int pt = blockIdx.x;
    const int k = k0 + pt;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

    for (int d = tid; d < n_lambda; d += NT) { r0[d] = 0.0; side0[d] = 0x7fffffff; side1[d] = -1; }
    if (tid < RN) prow[nrows + tid] = 0.0;
    __syncthreads();
    for (int row = tid; row < nrows; row += NT) {
        atomicMin(&side0[dof_map[row]], row);
        atomicMax(&side1[dof_map[row]], row);
    }
    for (int i = wid; i < n_sub; i += NT / 32) {
        const int nd = ndof[i], d0 = dof_ptr[i];
        const int loc = region[i] < 0 ? 0 : local_idx[(long long)region[i] * n_real + k];
        const long long bb = blk_base[i] + (long long)loc * nd * nd;
        for (int a = lane; a < nd; a += 32) {
            rb[d0 + a] = bb + a;
            rmeta[d0 + a] = d0 | (nd << 20);
        }
        const double *h = hbar + h_base[i] + (long long)loc * nd;
        const int *dm = dof_map + d0;
        // 0 + a + b: two contributions per dof, order free in IEEE
        for (int a = lane; a < nd; a += 32) atomicAdd(&r0[dm[a]], h[a]);
    }
    __syncthreads();
    const int d = tid >> 1, sd = tid & 1;
    const bool own = d < n_lambda;
    int row = -1;
    if (own) {
        const int s0 = side0[d], s1 = side1[d];
        row = sd == 0 ? s0 : (s1 != s0 ? s1 : -1);
    }
    double breg[RN];
    int rd0 = 0;
    {
        const int meta = row >= 0 ? rmeta[row] : 0;
        const int nd = row >= 0 ? (meta >> 20) : 0;
        rd0 = meta & 0xFFFFF;
        const double *Bp = blocks + (row >= 0 ? rb[row] : 0);
#pragma unroll
        for (int c = 0; c < RN; ++c) breg[c] = c < nd ? __ldg(Bp + (long long)c * nd) : 0.0;
    }
    const bool head = own && sd == 0;           // the dof's state lives here
    double x = 0.0, r = 0.0, pd = 0.0;
    const double g = own ? r0[d] : 0.0;
    if (head) {
        r = g;
        pd = g;
        if (g_out) g_out[(long long)pt * n_lambda + d] = g;
    }
    if (row >= 0) prow[row] = g;
    double rr = block_sum_alt(head ? g * g : 0.0, red2, rbuf);
    const double gnorm = sqrt(rr);
    double *lam = lam_out + (long long)pt * n_lambda;
    if (gnorm == 0.0) {
        if (head) lam[d] = 0.0;
        if (tid == 0) { iters_out[pt] = 0; status_out[pt] = MFB_CG_ZERO_RHS; }
        return;
    }
    double *hist = res_hist + (long long)pt * hist_cap;
    int status = MFB_CG_MAX_ITER, it_done = max_iter;
    for (int it = 1; it <= max_iter; ++it) {
        __syncthreads();                          // p (row space) of this iteration
        const double *pr = prow + rd0;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int c = 0; c < RN; c += 4) {
            a0 = fma(breg[c], pr[c], a0);
            a1 = fma(breg[c + 1], pr[c + 1], a1);
            a2 = fma(breg[c + 2], pr[c + 2], a2);
            a3 = fma(breg[c + 3], pr[c + 3], a3);
        }
        const double v = (a0 + a1) + (a2 + a3);
        const double vu = __shfl_down_sync(0xffffffffu, v, 1);
        const double sp = v + vu;                 // lower + upper (even threads)
        const double pSp = block_sum_alt(head ? pd * sp : 0.0, red2, rbuf);
        if (!(pSp > 0.0)) {
            status = MFB_CG_NOT_SPD;
            it_done = it;
            break;
        }
        const double a = rr / pSp;
        r = __dsub_rn(r, __dmul_rn(a, sp));
        const double rr_new = block_sum_alt(head ? r * r : 0.0, red2, rbuf);
        x = __dadd_rn(x, __dmul_rn(a, pd));
        const double rn = sqrt(rr_new);
        // rn now, rn / gnorm after the loop (keeps the division off the chain)
        if (tid == 0 && it <= hist_cap) hist[it - 1] = rn;
        if (rn <= tol * gnorm) {
            status = MFB_CG_CONVERGED;
            it_done = it;
            break;
        }
        const double beta = rr_new / rr;
        pd = __dadd_rn(r, __dmul_rn(beta, pd));
        const double pv = __shfl_sync(0xffffffffu, pd, lane & ~1);
        if (row >= 0) prow[row] = pv;
        rr = rr_new;
    }
    if (head) lam[d] = x;
    if (tid == 0) { iters_out[pt] = it_done; status_out[pt] = status; }
    __syncthreads();                              // tid 0's rn entries
    const int nh = min(status == MFB_CG_NOT_SPD ? it_done - 1 : it_done, hist_cap);
    for (int j = tid; j < nh; j += NT) hist[j] = hist[j] / gnorm;
}

}  // namespace

extern "C" int mfb_debug_cgprof(unsigned long long *out) {
#ifdef MFB_PROFILE
    return cudaMemcpyFromSymbol(out, g_cgprof, sizeof(unsigned long long) * 8) == cudaSuccess ? 0 : 2;
#else
    (void)out;
    return 1;
#endif
}

extern "C" int mfb_cg_batched(int n_lambda, int n_sub, const int *ndof, const int *dof_ptr,
                              const int *dof_map, const int *region,
                              const long long *blk_base, const long long *h_base,
                              const int *local_idx, int n_real, const double *blocks,
                              const double *hbar, int k0, int n_pts, double tol,
                              int max_iter, double *lam, int *iters, int *status,
                              double *res_hist, int hist_cap, double *g,
                              long long stage_doubles, int reg_ndof, void *stream) {
    if (n_pts <= 0) return n_pts == 0 ? MFB_OK : MFB_ERR_ARG;
    // every mortar dof has two sides: the stacked block rows number 2 n_lambda
    const int nrows = 2 * n_lambda;
    int nt = ((nrows + 31) / 32) * 32;
    if (nt > CG_NT_MAX) nt = CG_NT_MAX;
    if (nt < 64) nt = 64;
    // vectors, row results, row block offsets + metadata, stage offsets, sides
    size_t smem = (size_t)4 * n_lambda * 8 + (size_t)nrows * (8 + 4 + 4) + (size_t)n_sub * 4 +
                  (size_t)n_lambda * 8 + 64;
    // p gathered into row space (no index chase in the GEMV) when it fits,
    // else the dof lists; then the point's blocks when they fit too
    int use_prow = smem + (size_t)nrows * 8 <= 200 * 1024;
    smem += use_prow ? (size_t)nrows * 8 : (size_t)nrows * 4;
    long long stage = stage_doubles;
    // register rows (cg_pair_kernel): one block row per thread, the two
    // sides of a dof on adjacent lanes, at most 608 threads for the register
    // budget, max ndof <= 32 and a multiple of 4; nothing is staged
    const int rn = (reg_ndof <= 16 ? 16 : 32);
    const bool regs = use_prow && reg_ndof > 0 && reg_ndof <= 32 && nrows <= 608;
    if (stage < 0 || smem + (size_t)stage * sizeof(double) > 200 * 1024) stage = 0;
    smem += (size_t)stage * sizeof(double);
    if (smem > 227 * 1024) return MFB_ERR_SMEM;
    cudaStream_t st = mfb_stream(stream);
#define MFB_CG_LAUNCH()                                                                     \
    do {                                                                                    \
        if (cudaFuncSetAttribute(cg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                 (int)smem) != cudaSuccess)                                 \
            return MFB_ERR_SMEM;                                                            \
        cg_kernel<<<n_pts, nt, smem, st>>>(                                                 \
            n_lambda, n_sub, ndof, dof_ptr, dof_map, region, blk_base, h_base, local_idx,   \
            n_real, blocks, hbar, k0, tol, max_iter, lam, iters, status, res_hist, hist_cap, \
            g, stage, use_prow);                                                            \
    } while (0)
#define MFB_CG_PAIR(R)                                                                      \
    do {                                                                                    \
        const size_t sm2 = (size_t)n_lambda * 8 + (size_t)(nrows + R) * 8 +                \
                           (size_t)nrows * (8 + 4) + (size_t)n_lambda * 8 + 64;            \
        if (cudaFuncSetAttribute(cg_pair_kernel<R>,                                         \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,               \
                                 (int)sm2) != cudaSuccess)                                  \
            return MFB_ERR_SMEM;                                                            \
        cg_pair_kernel<R><<<n_pts, nt, sm2, st>>>(                                          \
            n_lambda, n_sub, ndof, dof_ptr, dof_map, region, blk_base, h_base, local_idx,   \
            n_real, blocks, hbar, k0, tol, max_iter, lam, iters, status, res_hist, hist_cap, \
            g);                                                                             \
    } while (0)
    if (!regs) MFB_CG_LAUNCH();
    else if (rn == 16) MFB_CG_PAIR(16);
    else MFB_CG_PAIR(32);
#undef MFB_CG_LAUNCH
#undef MFB_CG_PAIR
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}
