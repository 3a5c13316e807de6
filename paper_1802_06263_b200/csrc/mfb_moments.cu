// Moments of the S3 sweep (reference moments.py:10-58, interface.py:250-268).
//
// Field keys: the reference reconstructs every point's fields by a star solve
// and streams s += w f, q += w f f. Here the fields of point k on subdomain
// i are affine in lambda: f_k = Fb_l - M_l lam_k|_i with l = loc_i(k), so
// the sweep only needs, per group (i, l), shifted sufficient statistics of
// lambda (W, s, C around the first member lam*), then
//   mean = sum_l (W_l f*_l + t_l),  f* = Fb - M lam*,  t = -M s
//   var  = sum_l [W_l (f*_l - m)^2 + 2 (f*_l - m) t_l + q_l] + m^2 (1 - W)
// with q = diag(M C M^T). This equals sum w f^2 - m^2 (what the reference
// computes) algebraically, including sweeps whose weights do not sum to 1.
// The "lambda" key is streamed in realization order with the reference's
// exact operation order (no FMA), so identical lambdas give identical bits.
#include "mfb_common.cuh"

namespace {

constexpr int GS_NT = 256;
constexpr int GS_TILE = 16;

__global__ void __launch_bounds__(GS_NT)
group_stats_kernel(const int *__restrict__ grp_sid, const int *__restrict__ grp_ptr,
                   const int *__restrict__ grp_members, const int *__restrict__ ndof,
                   const int *__restrict__ dof_ptr, const int *__restrict__ dof_map,
                   int n_lambda, const double *__restrict__ lam,
                   const double *__restrict__ weights, const long long *__restrict__ grp_voff,
                   const long long *__restrict__ grp_coff, double *__restrict__ W,
                   double *__restrict__ lamstar, double *__restrict__ s_out,
                   double *__restrict__ C_out) {
    extern __shared__ double sm[];
    const int g = blockIdx.x;
    const int sid = grp_sid[g];
    const int nd = ndof[sid];
    const int *dm = dof_map + dof_ptr[sid];
    const int m0 = grp_ptr[g], m1 = grp_ptr[g + 1];
    double *ls = sm;                     // lam* (nd)
    double *dt = ls + nd;                // GS_TILE x nd deviations
    double *wt = dt + GS_TILE * nd;      // GS_TILE weights
    const int tid = threadIdx.x;
    if (m1 == m0) {
        for (int a = tid; a < nd; a += GS_NT) {
            lamstar[grp_voff[g] + a] = 0.0;
            s_out[grp_voff[g] + a] = 0.0;
        }
        for (int e = tid; e < nd * nd; e += GS_NT) C_out[grp_coff[g] + e] = 0.0;
        if (tid == 0) W[g] = 0.0;
        return;
    }
    const int k_first = grp_members[m0];
    for (int a = tid; a < nd; a += GS_NT) ls[a] = lam[(long long)k_first * n_lambda + dm[a]];
    // each thread owns a fixed set of C entries and s entries: fixed order sums
    const int nce = nd * nd;
    const int per = (nce + GS_NT - 1) / GS_NT;   // <= 16 for nd <= 64
    double cacc[16];
    for (int q = 0; q < 16; ++q) cacc[q] = 0.0;
    double sacc = 0.0, wacc = 0.0;
    __syncthreads();
    for (int base = m0; base < m1; base += GS_TILE) {
        const int cnt = min(GS_TILE, m1 - base);
        for (int e = tid; e < cnt * nd; e += GS_NT) {
            const int mm = e / nd, a = e % nd;
            const int k = grp_members[base + mm];
            dt[mm * nd + a] = lam[(long long)k * n_lambda + dm[a]] - ls[a];
        }
        if (tid < cnt) wt[tid] = weights[grp_members[base + tid]];
        __syncthreads();
        for (int mm = 0; mm < cnt; ++mm) {
            const double w = wt[mm];
            const double *d = dt + mm * nd;
            for (int q = 0; q < per; ++q) {
                const int e = tid + q * GS_NT;
                if (e < nce) cacc[q] += (w * d[e / nd]) * d[e % nd];
            }
            if (tid < nd) sacc += w * d[tid];
            if (tid == 0) wacc += w;
        }
        __syncthreads();
    }
    for (int q = 0; q < per; ++q) {
        const int e = tid + q * GS_NT;
        if (e < nce) C_out[grp_coff[g] + e] = cacc[q];
    }
    if (tid < nd) {
        s_out[grp_voff[g] + tid] = sacc;
        lamstar[grp_voff[g] + tid] = ls[tid];
    }
    if (tid == 0) W[g] = wacc;
}

__global__ void __launch_bounds__(GS_NT)
group_fields_kernel(const int *__restrict__ grp_sid, const int *__restrict__ ndof,
                    const int *__restrict__ nfield, const double *__restrict__ M,
                    const long long *__restrict__ grp_moff, const double *__restrict__ Fb,
                    const long long *__restrict__ grp_fboff,
                    const long long *__restrict__ grp_voff,
                    const long long *__restrict__ grp_coff,
                    const double *__restrict__ lamstar, const double *__restrict__ s,
                    const double *__restrict__ C, double *__restrict__ fstar,
                    double *__restrict__ t, double *__restrict__ q) {
    extern __shared__ double sm[];
    const int g = blockIdx.y;
    const int sid = grp_sid[g];
    const int nd = ndof[sid], nf = nfield[sid];
    double *Cs = sm;
    double *ls = Cs + nd * nd;
    double *ss = ls + nd;
    for (int e = threadIdx.x; e < nd * nd; e += GS_NT) Cs[e] = C[grp_coff[g] + e];
    for (int a = threadIdx.x; a < nd; a += GS_NT) {
        ls[a] = lamstar[grp_voff[g] + a];
        ss[a] = s[grp_voff[g] + a];
    }
    __syncthreads();
    const double *Mg = M + grp_moff[g];
    constexpr int NDR = 32;                  // rows up to 32 dofs live in registers
    for (int f = blockIdx.x * GS_NT + threadIdx.x; f < nf; f += gridDim.x * GS_NT) {
        const double *row = Mg + (long long)f * nd;
        double ml = 0.0, ms = 0.0, qq = 0.0;
        if (nd <= NDR) {
            double m[NDR];
#pragma unroll
            for (int b = 0; b < NDR; ++b) m[b] = b < nd ? row[b] : 0.0;
#pragma unroll
            for (int a = 0; a < NDR; ++a) {
                if (a >= nd) break;
                ml += m[a] * ls[a];
                ms += m[a] * ss[a];
                double cm = 0.0;
#pragma unroll
                for (int b = 0; b < NDR; ++b)
                    if (b < nd) cm += Cs[a * nd + b] * m[b];
                qq += m[a] * cm;
            }
        } else {
            for (int a = 0; a < nd; ++a) {
                const double ma = row[a];
                ml += ma * ls[a];
                ms += ma * ss[a];
                double cm = 0.0;
                for (int b = 0; b < nd; ++b) cm += Cs[a * nd + b] * row[b];
                qq += ma * cm;
            }
        }
        const long long o = grp_fboff[g] + f;
        fstar[o] = Fb[o] - ml;
        t[o] = -ms;
        q[o] = qq;
    }
}

__global__ void moments_reduce_kernel(int n_sub, const int *__restrict__ gptr,
                                      const int *__restrict__ nfield,
                                      const long long *__restrict__ grp_fboff,
                                      const double *__restrict__ W,
                                      const double *__restrict__ fstar,
                                      const double *__restrict__ t,
                                      const double *__restrict__ q, double wtot,
                                      const long long *__restrict__ sid_out_off,
                                      double *__restrict__ mean, double *__restrict__ var) {
    const int sid = blockIdx.y;
    const int nf = nfield[sid];
    const int g0 = gptr[sid], g1 = gptr[sid + 1];
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nf; f += gridDim.x * blockDim.x) {
        double m = 0.0;
        for (int g = g0; g < g1; ++g) {
            const long long o = grp_fboff[g] + f;
            m += W[g] * fstar[o] + t[o];
        }
        double v = 0.0;
        for (int g = g0; g < g1; ++g) {
            const long long o = grp_fboff[g] + f;
            const double dfs = fstar[o] - m;
            v += W[g] * dfs * dfs + 2.0 * dfs * t[o] + q[o];
        }
        v += m * m * (1.0 - wtot);
        mean[sid_out_off[sid] + f] = m;
        var[sid_out_off[sid] + f] = v;
    }
}

__global__ void lambda_moments_kernel(int n_lambda, int n_real, const double *__restrict__ lam,
                                      const double *__restrict__ w, double *__restrict__ mean,
                                      double *__restrict__ var, double *__restrict__ sumsq) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= n_lambda) return;
    double s = 0.0, q = 0.0;
    for (int k = 0; k < n_real; ++k) {
        const double v = lam[(long long)k * n_lambda + d];
        const double wv = __dmul_rn(w[k], v);
        s = __dadd_rn(s, wv);
        q = __dadd_rn(q, __dmul_rn(wv, v));
    }
    mean[d] = s;
    var[d] = __dsub_rn(q, __dmul_rn(s, s));
    sumsq[d] = q;
}

}  // namespace

extern "C" int mfb_group_stats(int n_groups, const int *grp_sid, const int *grp_ptr,
                               const int *grp_members, const int *ndof, const int *dof_ptr,
                               const int *dof_map, int n_lambda, const double *lam,
                               const double *weights, const long long *grp_voff,
                               const long long *grp_coff, double *W, double *lamstar,
                               double *s, double *C, void *stream) {
    if (n_groups <= 0) return n_groups == 0 ? MFB_OK : MFB_ERR_ARG;
    const int max_nd = 64;
    size_t smem = (size_t)(max_nd + GS_TILE * max_nd + GS_TILE) * sizeof(double);
    group_stats_kernel<<<n_groups, GS_NT, smem, mfb_stream(stream)>>>(
        grp_sid, grp_ptr, grp_members, ndof, dof_ptr, dof_map, n_lambda, lam, weights,
        grp_voff, grp_coff, W, lamstar, s, C);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}

extern "C" int mfb_group_fields(int n_groups, const int *grp_sid, const int *ndof,
                                const int *nfield, const double *M, const long long *grp_moff,
                                const double *Fb, const long long *grp_fboff,
                                const long long *grp_voff, const long long *grp_coff,
                                const double *lamstar, const double *s, const double *C,
                                double *fstar, double *t, double *q, void *stream) {
    if (n_groups <= 0) return n_groups == 0 ? MFB_OK : MFB_ERR_ARG;
    const int max_nd = 64;
    size_t smem = (size_t)(max_nd * max_nd + 2 * max_nd) * sizeof(double);
    if (cudaFuncSetAttribute(group_fields_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return MFB_ERR_SMEM;
    dim3 grid(8, n_groups);
    group_fields_kernel<<<grid, GS_NT, smem, mfb_stream(stream)>>>(
        grp_sid, ndof, nfield, M, grp_moff, Fb, grp_fboff, grp_voff, grp_coff, lamstar, s, C,
        fstar, t, q);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}

extern "C" int mfb_moments_reduce(int n_sub, const int *gptr, const int *nfield,
                                  const long long *grp_fboff, const double *W,
                                  const double *fstar, const double *t, const double *q,
                                  double wtot, const long long *sid_out_off, double *mean,
                                  double *var, void *stream) {
    if (n_sub <= 0) return n_sub == 0 ? MFB_OK : MFB_ERR_ARG;
    dim3 grid(16, n_sub);
    moments_reduce_kernel<<<grid, 256, 0, mfb_stream(stream)>>>(
        n_sub, gptr, nfield, grp_fboff, W, fstar, t, q, wtot, sid_out_off, mean, var);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}

extern "C" int mfb_lambda_moments(int n_lambda, int n_real, const double *lam,
                                  const double *weights, double *mean, double *var,
                                  double *sumsq, void *stream) {
    if (n_lambda <= 0 || n_real < 0) return MFB_ERR_ARG;
    lambda_moments_kernel<<<(n_lambda + 127) / 128, 128, 0, mfb_stream(stream)>>>(
        n_lambda, n_real, lam, weights, mean, var, sumsq);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}

#ifndef MFB_SOURCE_HASH
#define MFB_SOURCE_HASH "unknown"
#endif
// "mfb-b200 <version> (sm_100a) src <hash>": <hash> = _build.source_hash() of
// the csrc/include tree this library was compiled from (checked at load time)
extern "C" const char *mfb_version(void) {
    return "mfb-b200 0.2.0 (sm_100a) src " MFB_SOURCE_HASH;
}

extern "C" const char *mfb_strerror(int code) {
    switch (code) {
        case MFB_OK: return "ok";
        case MFB_ERR_ARG: return "invalid argument";
        case MFB_ERR_LAUNCH: return "kernel launch failed";
        case MFB_ERR_SMEM: return "shared-memory request exceeds the device limit";
        default: return "unknown error";
    }
}

// ---- self test: FP64 tensor-core fragment layout used by the band kernel ----
namespace {
__global__ void selftest_dmma_kernel(double *err) {
    const int lane = threadIdx.x;
    const int g = lane >> 2, q4 = lane & 3;
    // A[i][k] = 1 + i + 0.5 k, B[k][j] = 2 - 0.25 j + k, C[i][j] = i - j
    const double a = 1.0 + g + 0.5 * q4;
    const double b = 2.0 - 0.25 * g + q4;
    double d0 = g - 2 * q4, d1 = g - (2 * q4 + 1);
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
    double e = 0.0;
    for (int h = 0; h < 2; ++h) {
        const int i = g, j = 2 * q4 + h;
        double ref = i - j;
        for (int k = 0; k < 4; ++k) ref += (1.0 + i + 0.5 * k) * (2.0 - 0.25 * j + k);
        e = fmax(e, fabs((h ? d1 : d0) - ref));
    }
    for (int o = 16; o > 0; o >>= 1) e = fmax(e, __shfl_down_sync(0xffffffffu, e, o));
    if (lane == 0) *err = e;
}
}  // namespace

extern "C" int mfb_selftest_dmma(double *err, void *stream) {
    selftest_dmma_kernel<<<1, 32, 0, mfb_stream(stream)>>>(err);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}
