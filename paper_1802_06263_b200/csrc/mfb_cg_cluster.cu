// Batched interface CG for large interfaces on thread-block clusters.
//
// cfg4 (n_lambda = 2,720, 128 subdomains, 2.2 MB of blocks per point, 54,273
// points): NP collocation points (the slots) are solved in lockstep by one
// cluster of C CTAs. The subdomains are split into C geometric parts
// (cgcluster.py); CTA c applies only its part's flux-basis blocks and keeps
// the CG vectors of the mortar dofs it owns ON CHIP:
//
//   p   shared memory, owned rows + halo rows (the columns of the part's
//       blocks owned by another part, refreshed by their owner over DSMEM);
//   S p shared memory, owned rows (+ a cut buffer: upper-side rows of the
//       interfaces the partition cuts, stored by the other part over DSMEM);
//   r   registers (a fixed set of (row, slot pair) elements per thread);
//   x   global scratch (read-modify-write once per iteration).
//
// Per iteration: S p on the FP64 tensor cores (mma.m8n8k4, the NP slots are
// NP/8 N-tiles, so every block fragment read from L2 feeds NP/8 MMAs), then
// the reference's recurrences (interface.py:107-139) elementwise on the
// owned rows, with the two dot products reduced per CTA and all-gathered
// across the cluster through DSMEM (every CTA sums the C partials in rank
// order, so every CTA holds the same alpha, beta and verdicts and the slot
// state machine is replicated, not communicated). Four cluster barriers per
// iteration. Slots are refilled from a global work counter (rank 0 draws
// and mails the point ids), so long-running points do not hold the others.
//
// Per point the arithmetic is independent of the other slots and of the
// cluster it runs in: block rows accumulate in the packed fragment order
// with two chains (even/odd fragments, summed), S p = lower row + upper row
// (basis_apply's order, interface.py:238-247, one addition whichever part
// computed each side), dot products by a fixed thread/warp/rank tree.
//
// Residual histories are written into a segmented pool (segments of `seg`
// entries drawn from a counter as a point's iterations cross a multiple of
// seg), so device memory scales with the iterations actually run, not with
// n_points x max_iter.
#include <cooperative_groups.h>
#include <stdint.h>

#include "mfb_common.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int KT = 256;          // threads per CTA
constexpr int KW = KT / 32;
constexpr int KMAXC = 8;         // cluster size (portable maximum)
constexpr int HDR = 16;
constexpr int RSLOT = 5;         // A-fragment ring slots per warp (TMA bulk copies)
constexpr int SLOT_D = 256;      // doubles per slot: 8 fragments of 32

struct ClArgs {
    int n_lambda, n_regions, n_real, k0, n_pts, max_iter, C;
    int used_max, own_max, cut_max, cm_max, unit_max, strip_max;   // shared-memory layout of every rank
    int r_smem, x_smem, s_glob;               // r / x in shared memory (else rs / xs); S p in global (ss)
    double tol;
    const int *hdr, *tab, *local_idx, *ndof, *region;
    const int4 *sides;
    const long long *h_base;
    const double *hbar, *packed;
    double *lam, *g, *xs, *rs, *ss, *hist;
    int *iters, *status, *next, *seg_tab, *seg_next;
    int seg, max_segs;
    long long seg_cap;
    int dbg;
};
static int g_cl_dbg = 0;
__device__ long long g_cl_prof[1024 * 8];
__device__ int g_trace_on;
__device__ int g_cl_dbg_nofence;
__device__ int g_trace_n;

__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// element (row u, slot s) of a [rows][NP] shared array; with NP = 16 the two
// 64-byte halves of odd rows are swapped so the 4 rows of an MMA B fragment
// (consecutive columns) spread over all 32 banks
template <int NP>
__device__ __forceinline__ int pel(int u, int s) {
    return NP == 16 ? u * 16 + (s ^ ((u & 1) << 3)) : u * NP + s;
}

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ double lds_f64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
// column maps are written once before the first cluster barrier: a pure load
__device__ __forceinline__ int lds_s32(unsigned a) {
    int v;
    asm("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

// ---- mbarrier + TMA bulk copy (global -> this CTA's shared memory) -------
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void bulk_load(unsigned dst, const void *src, unsigned bytes,
                                          unsigned bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(dst), "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(bar), "r"(parity)
        : "memory");
}

// Phase A is organised by UNITS (cgcluster.py): one block of the rank in one
// pass, its B operand (p at the block's columns, all slots) held in
// registers for the whole unit, its strips' A fragments streamed per
// (strip, local-realization group) ITEM. Each warp owns a ring of RSLOT
// 2 KB slots in shared memory that its lane 0 fills with TMA bulk copies
// (8 fragments per slot, an item of more takes two) as far ahead as the ring
// allows -- across units and into the next pass -- so the L2 latency is
// covered by the copies in flight, not by the warp's registers.
struct ItemIt {
    int j;            // unit ordinal of this warp in the pass (unit = wid + KW * j)
    int pass;         // 0, 1; 2 = exhausted
    int k, gi;        // strip in the unit, group of the unit's region
};

// unit record {nd, region, psz, cm_off} {n_strips, first strip, pass, cost}
template <int NP>
__device__ __forceinline__ bool item_next(ItemIt &it, const int4 *units, int n_u1, int n_units,
                                          const int *gcnt, const unsigned *gmask,
                                          unsigned live, unsigned &m) {
    const int wid = threadIdx.x >> 5;
    for (;;) {
        if (it.pass > 1) return false;
        const int lo = it.pass ? n_u1 : 0, hi = it.pass ? n_units : n_u1;
        const int u = lo + wid + KW * it.j;
        if (u >= hi) { ++it.pass; it.j = 0; it.k = 0; it.gi = -1; continue; }
        const int4 U0 = units[2 * u], U1 = units[2 * u + 1];
        const int reg = U0.y, ngrp = reg < 0 ? 1 : gcnt[reg];
        for (++it.gi;; ++it.gi) {
            if (it.gi >= ngrp) { ++it.k; it.gi = 0; }
            if (it.k >= U1.x) break;
            m = reg < 0 ? live : (gmask[reg * NP + it.gi] & live);
            if (m) return true;
        }
        ++it.j; it.k = 0; it.gi = -1;
    }
}

// per-warp ring state (warp-uniform registers)
struct Ring {
    unsigned base;    // shared address of slot 0 of this warp
    unsigned bar;     // shared address of the slot 0 mbarrier (8 bytes apart)
    int head, used;   // next slot to fill, slots filled and not yet consumed
    unsigned par;     // per-slot wait parity bits
    ItemIt pit;       // producer position
};

// issue copies for the next items while the ring has room
template <int NP>
__device__ __forceinline__ void ring_fill(Ring &rg, const int4 *units, const int4 *strips,
                                          int n_u1, int n_units, const int *gcnt,
                                          const int *gloc, const unsigned *gmask, unsigned live,
                                          const double *__restrict__ packed) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        ItemIt nx = rg.pit;
        unsigned m;
        if (!item_next<NP>(nx, units, n_u1, n_units, gcnt, gmask, live, m)) return;
        const int lo = nx.pass ? n_u1 : 0;
        const int u = lo + (threadIdx.x >> 5) + KW * nx.j;
        const int4 U0 = units[2 * u], U1 = units[2 * u + 1];
        const int nt4 = (U0.x + 3) >> 2, need = nt4 > 8 ? 2 : 1;
        if (rg.used + need > RSLOT) return;
        const int l = U0.y < 0 ? 0 : gloc[U0.y * NP + nx.gi];
        const int4 st = strips[U1.y + nx.k];
        const double *src = packed + st.x + (long long)l * U0.z;
        if (lane == 0) {
            if (g_cl_dbg_nofence == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const int s0 = rg.head, s1 = (rg.head + 1) % RSLOT;
            const int n0 = nt4 > 8 ? 8 : nt4;
            bulk_load(rg.base + s0 * SLOT_D * 8, src, n0 * 256, rg.bar + 8 * s0);
            if (need == 2)
                bulk_load(rg.base + s1 * SLOT_D * 8, src + 8 * 32, (nt4 - 8) * 256,
                          rg.bar + 8 * s1);
        }
        __syncwarp();
        rg.head = (rg.head + need) % RSLOT;
        rg.used += need;
        rg.pit = nx;
    }
}

// the A fragments of the item in slot s (and s+1) into registers, after its
// copies landed
template <int NT, bool GEN>
__device__ __forceinline__ int ring_take(Ring &rg, int nt4, double (&a)[16]) {
    const int lane = threadIdx.x & 31;
    const int tail = (rg.head - rg.used + RSLOT) % RSLOT;
    const int need = nt4 > 8 ? 2 : 1;
    mbar_wait(rg.bar + 8 * tail, (rg.par >> tail) & 1u);
    rg.par ^= 1u << tail;
    const int t2 = (tail + 1) % RSLOT;
    if (need == 2) {
        mbar_wait(rg.bar + 8 * t2, (rg.par >> t2) & 1u);
        rg.par ^= 1u << t2;
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        if (GEN && t >= nt4) break;
        const int sl = t < 8 ? tail : t2;
        a[t] = lds_f64(rg.base + (unsigned)(sl * SLOT_D * 8 + (t & 7) * 256 + lane * 8));
    }
    rg.used -= need;
    return need;
}

// MMAs of one item for N-tiles HM: acc[h] += (A x B) for the member slots
template <int NP, int NT, bool GEN, int HM>
__device__ __forceinline__ void item_mma(int nt4, const double (&a)[16],
                                         const double (&Bv)[16][NP / 8], unsigned m,
                                         double (&acc)[NP / 8][2]) {
    constexpr int NH = NP / 8;
    const int q = threadIdx.x & 3;
    double e[NH][2], o[NH][2];
#pragma unroll
    for (int h = 0; h < NH; ++h) e[h][0] = e[h][1] = o[h][0] = o[h][1] = 0.0;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        if (GEN && t >= nt4) break;
#pragma unroll
        for (int h = 0; h < NH; ++h) {
            if (!((HM >> h) & 1)) continue;
            if (t & 1)
                dmma884(o[h][0], o[h][1], a[t], Bv[t][h]);
            else
                dmma884(e[h][0], e[h][1], a[t], Bv[t][h]);
        }
    }
#pragma unroll
    for (int h = 0; h < NH; ++h) {
        if (!((HM >> h) & 1)) continue;
        const unsigned mh = m >> (8 * h + 2 * q);
        if (mh & 1u) acc[h][0] += e[h][0] + o[h][0];
        if (mh & 2u) acc[h][1] += e[h][1] + o[h][1];
    }
}

// consume every item of unit u (this warp's), the B operand in registers;
// rows leave per strip: pass 1 S := acc, pass 2 S += acc or the owner's cut
// buffer (DSMEM)
template <int NP, int NT, bool GEN>
__device__ __forceinline__ void unit_consume(int u, Ring &rg, const int4 *units,
                                             const int4 *strips, int n_u1, int n_units,
                                             const int *gcnt, const int *gloc,
                                             const unsigned *gmask, unsigned live,
                                             const double *__restrict__ packed, unsigned psh,
                                             unsigned cmbase, double *S, double *CB,
                                             cg::cluster_group &cl) {
    constexpr int NH = NP / 8;
    const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
    const int4 U0 = units[2 * u], U1 = units[2 * u + 1];
    const int nd = U0.x, nt4 = (nd + 3) >> 2, reg = U0.y;
    const int ngrp = reg < 0 ? 1 : gcnt[reg];
    double Bv[16][NH];
    {
        const unsigned cma = cmbase + 4u * (U0.w + q);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            if (GEN && t >= nt4) break;
            const int cv = (4 * t + q < nd ? lds_s32(cma + 16u * t) : 0) + g;
#pragma unroll
            for (int h = 0; h < NH; ++h) Bv[t][h] = lds_f64(psh + 8u * (unsigned)(cv ^ (h << 3)));
        }
    }
    for (int k = 0; k < U1.x; ++k) {
        double acc[NH][2];
#pragma unroll
        for (int h = 0; h < NH; ++h) acc[h][0] = acc[h][1] = 0.0;
        for (int gi = 0; gi < ngrp; ++gi) {
            const unsigned m = reg < 0 ? live : (gmask[reg * NP + gi] & live);
            if (!m) continue;
            const long long c0 = clock64();
            ring_fill<NP>(rg, units, strips, n_u1, n_units, gcnt, gloc, gmask, live, packed);
            const long long c1 = clock64();
            double a[16];
            ring_take<NT, GEN>(rg, nt4, a);
            const long long c2 = clock64();
            const int hm = NH == 1 ? 1 : ((m & 0xffu) ? 1 : 0) | ((m >> 8) ? 2 : 0);
            if (NH == 1 || hm == 1)
                item_mma<NP, NT, GEN, 1>(nt4, a, Bv, m, acc);
            else if (hm == 2)
                item_mma<NP, NT, GEN, 2>(nt4, a, Bv, m, acc);
            else
                item_mma<NP, NT, GEN, 3>(nt4, a, Bv, m, acc);
            if (g_trace_on && blockIdx.x == 0 && (threadIdx.x >> 5) == 0) {
                const double s_ = acc[0][0];
                const long long c3 = clock64();
                const int i = g_trace_n;
                if (i < 256 && (threadIdx.x & 31) == 0) {
                    g_cl_prof[i * 6 + 0] = c1 - c0;
                    g_cl_prof[i * 6 + 1] = c2 - c1;
                    g_cl_prof[i * 6 + 2] = c3 - c2 + (s_ == 12345.0);
                    g_cl_prof[i * 6 + 3] = nt4;
                    g_cl_prof[i * 6 + 4] = __popc(m);
                    g_cl_prof[i * 6 + 5] = hm;
                }
                g_trace_n = i + 1;
            }
        }
        const int4 st = strips[U1.y + k];
        const int R = st.y & 0xff, kind = (st.y >> 8) & 0xf, ow = st.y >> 12;
        if (g < R) {
            const int row = st.z + g;
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                const int sl = 8 * h + 2 * q;
                if (kind & 4) {
                    *reinterpret_cast<double2 *>(cl.map_shared_rank(CB, ow) + row * NP + sl) =
                        make_double2(acc[h][0], acc[h][1]);
                } else {
                    double2 *dp = reinterpret_cast<double2 *>(S + pel<NP>(row, sl));
                    if (kind & 2) {
                        const double2 v = *dp;
                        *dp = make_double2(v.x + acc[h][0], v.y + acc[h][1]);
                    } else {
                        *dp = make_double2(acc[h][0], acc[h][1]);
                    }
                }
            }
        }
    }
}

template <int NP>
__device__ __forceinline__ void unit_dispatch(int u, Ring &rg, const int4 *units,
                                              const int4 *strips, int n_u1, int n_units,
                                              const int *gcnt, const int *gloc,
                                              const unsigned *gmask, unsigned live,
                                              const double *__restrict__ packed, unsigned psh,
                                              unsigned cmbase, double *S, double *CB,
                                              cg::cluster_group &cl) {
    switch (units[2 * u].x) {
    case 16: unit_consume<NP, 4, false>(u, rg, units, strips, n_u1, n_units, gcnt, gloc, gmask, live, packed, psh, cmbase, S, CB, cl); break;
    case 24: unit_consume<NP, 6, false>(u, rg, units, strips, n_u1, n_units, gcnt, gloc, gmask, live, packed, psh, cmbase, S, CB, cl); break;
    case 32: unit_consume<NP, 8, false>(u, rg, units, strips, n_u1, n_units, gcnt, gloc, gmask, live, packed, psh, cmbase, S, CB, cl); break;
    case 48: unit_consume<NP, 12, false>(u, rg, units, strips, n_u1, n_units, gcnt, gloc, gmask, live, packed, psh, cmbase, S, CB, cl); break;
    case 64: unit_consume<NP, 16, false>(u, rg, units, strips, n_u1, n_units, gcnt, gloc, gmask, live, packed, psh, cmbase, S, CB, cl); break;
    default: unit_consume<NP, 16, true>(u, rg, units, strips, n_u1, n_units, gcnt, gloc, gmask, live, packed, psh, cmbase, S, CB, cl); break;
    }
}

enum { SLOT_RUN = 0, SLOT_NEW = 1, SLOT_DONE = 2 };

// per-slot sums of the slot pair a thread accumulated (pair = tid % (NP/2),
// fixed): xor tree over the lanes with the same pair, the warps in order,
// then the cluster's ranks in order (every CTA computes the same totals).
// Returns, in threads tid < NP, the total of slot tid. Ends with a cluster
// barrier (everything stored to peers before the call is visible after it).
template <int NP>
__device__ __forceinline__ double cluster_sum(double v0, double v1, double (*red)[NP],
                                              double *gbuf, cg::cluster_group &cl, int C,
                                              int rank) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = NP / 2; o < 32; o <<= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, o);
        v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    }
    if (lane < NP / 2) {
        red[wid][2 * lane] = v0;
        red[wid][2 * lane + 1] = v1;
    }
    __syncthreads();
    if (threadIdx.x < NP) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < KW; ++w) t += red[w][threadIdx.x];
        for (int r = 0; r < C; ++r) cl.map_shared_rank(gbuf, r)[rank * NP + threadIdx.x] = t;
    }
    cl.sync();
    double tot = 0.0;
    if (threadIdx.x < NP)
        for (int r = 0; r < C; ++r) tot += gbuf[r * NP + threadIdx.x];
    return tot;
}

template <int NP>
__global__ void __launch_bounds__(KT, 1) cg_cluster_kernel(ClArgs A) {
    constexpr int NPR = NP / 2;                    // slot pairs per row
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int *H = A.hdr + rank * HDR;
    const int n_own = H[0], n_units = H[2], n_cut = H[3], n_cm = H[4], n_strips = H[10];
    const int n_u1 = H[12];
    const int *own = A.tab + H[5];
    const int2 *peer = reinterpret_cast<const int2 *>(A.tab + H[6]);
    const int4 *units_g = reinterpret_cast<const int4 *>(A.tab + H[7]);
    const int4 *strips_g = reinterpret_cast<const int4 *>(A.tab + H[11]);
    const int *cut = A.tab + H[9];
    const int n = A.n_lambda;
    const int npair = n_own * NPR;
    const int sp2 = tid % NPR;                     // this thread's slot pair (vector phases)
    const int NR = A.n_regions;

    // one layout for every rank (sized by the largest rank), so a peer's
    // arrays are at the same offsets as ours (map_shared_rank):
    // p [used][NP] | S p [own][NP] (unless in global) | cut [cut][NP] | r, x
    // [own][NPR] (double2, when in shared memory) | A ring [warps][RSLOT][256] |
    // column maps | group tables | units | strips
    extern __shared__ double smem[];
    double *P = smem;
    double *S = A.s_glob ? A.ss + (size_t)blockIdx.x * A.own_max * NP
                         : P + (size_t)A.used_max * NP;
    double *CB = (A.s_glob ? P + (size_t)A.used_max * NP : S + (size_t)A.own_max * NP);
    double *tail = CB + (size_t)A.cut_max * NP;
    double2 *R2, *X2;
    if (A.r_smem) { R2 = reinterpret_cast<double2 *>(tail); tail += (size_t)A.own_max * NP; }
    else R2 = reinterpret_cast<double2 *>(A.rs + (size_t)blockIdx.x * A.own_max * NP);
    if (A.x_smem) { X2 = reinterpret_cast<double2 *>(tail); tail += (size_t)A.own_max * NP; }
    else X2 = reinterpret_cast<double2 *>(A.xs + (size_t)blockIdx.x * A.own_max * NP);
    double *RING = tail;
    tail += (size_t)KW * RSLOT * SLOT_D;
    int *CM = reinterpret_cast<int *>(tail);
    int *s_loc = CM + A.cm_max;                    // [regions][NP]
    int *s_gloc = s_loc + NR * NP;                 // [regions][NP]
    unsigned *s_gmask = reinterpret_cast<unsigned *>(s_gloc + NR * NP);   // [regions][NP]
    int *s_gcnt = reinterpret_cast<int *>(s_gmask + NR * NP);             // [regions]
    int4 *units = reinterpret_cast<int4 *>(
        (reinterpret_cast<uintptr_t>(s_gcnt + NR) + 15) & ~uintptr_t(15));  // [unit_max][2]
    int4 *strips = units + 2 * A.unit_max;                                  // [strip_max]
    __shared__ int s_k[NP], s_it[NP], s_state[NP], s_stat[NP], s_mail[NP], s_seg[NP];
    __shared__ double s_rr[NP], s_gn[NP], s_a[NP], s_b[NP];
    __shared__ double s_red[KW][NP];
    __shared__ double s_gpsp[KMAXC * NP], s_grr[KMAXC * NP], s_ggg[KMAXC * NP];
    __shared__ int s_tctr;
    __shared__ int s_dbg[4];
    __shared__ __align__(8) unsigned long long s_bar[KW * RSLOT];
    __shared__ unsigned s_par[KW];

    for (int e = tid; e < n_cm; e += KT) CM[e] = pel<NP>(A.tab[H[8] + e], 0);
    for (int e = tid; e < 2 * n_units; e += KT) units[e] = units_g[e];
    for (int e = tid; e < n_strips; e += KT) strips[e] = strips_g[e];
    if (tid < KW * RSLOT) mbar_init(smem_u32(&s_bar[tid]), 1);
    if (tid < KW) s_par[tid] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int e = tid; e < A.used_max * NP; e += KT) P[e] = 0.0;
    if (tid < NP) { s_k[tid] = -1; s_state[tid] = SLOT_DONE; s_it[tid] = 0; s_seg[tid] = -1; }
    if (tid == 0) s_tctr = 0;
    if (tid < 4) s_dbg[tid] = 0;
    cl.sync();
    if (A.dbg == 1) return;
    long long pt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tc = clock64();
#define MFB_PT(i)                                      \
    do {                                               \
        if (A.dbg == 100 && tid == 0) {                \
            const long long t_ = clock64();            \
            pt[i] += t_ - tc;                          \
            tc = t_;                                   \
        }                                              \
    } while (0)

    for (;;) {
        // ---- refill free slots: rank 0 draws the points and mails them -----
        bool need = false;
#pragma unroll
        for (int s = 0; s < NP; ++s) need |= s_k[s] == -1;
        unsigned fresh = 0;
        if (need) {
            if (rank == 0 && tid == 0) {
                for (int s = 0; s < NP; ++s) {
                    if (s_k[s] != -1) continue;
                    const int t = atomicAdd(A.next, 1);
                    const int nk = t < A.n_pts ? t : -2;
                    for (int rr = 0; rr < A.C; ++rr) cl.map_shared_rank(s_mail, rr)[s] = nk;
                }
            }
            cl.sync();
            bool any = false;
#pragma unroll
            for (int s = 0; s < NP; ++s) {
                const int k = s_k[s] == -1 ? s_mail[s] : s_k[s];
                any |= k >= 0;
                if (s_k[s] == -1 && k >= 0) fresh |= 1u << s;
            }
            __syncthreads();
            if (tid < NP && s_k[tid] == -1) {
                s_k[tid] = s_mail[tid];
                s_state[tid] = s_mail[tid] >= 0 ? SLOT_NEW : SLOT_DONE;
                s_it[tid] = 0;
                s_seg[tid] = -1;
            }
            if (!any) break;
            __syncthreads();
        }
        if (fresh) {
            for (int e = tid; e < NR * NP; e += KT) {
                const int s = e % NP;
                if ((fresh >> s) & 1u)
                    s_loc[e] = A.local_idx[(long long)(e / NP) * A.n_real + A.k0 + s_k[s]];
            }
            __syncthreads();
            // per region: the distinct local realizations of the slots holding
            // points, with their slot masks
            for (int rg = tid; rg < NR; rg += KT) {
                int cnt = 0;
                for (int s = 0; s < NP; ++s) {
                    if (s_k[s] < 0) continue;
                    const int l = s_loc[rg * NP + s];
                    int j = 0;
                    while (j < cnt && s_gloc[rg * NP + j] != l) ++j;
                    if (j == cnt) {
                        s_gloc[rg * NP + cnt] = l;
                        s_gmask[rg * NP + cnt] = 0u;
                        ++cnt;
                    }
                    s_gmask[rg * NP + j] |= 1u << s;
                }
                s_gcnt[rg] = cnt;
            }
            // g = 0 + h_lower + h_upper (mortar.jump of the bar traces), x = 0,
            // r = p = g on the owned rows; the peers' halo copies of p too
            const bool f0 = (fresh >> (2 * sp2)) & 1u, f1 = (fresh >> (2 * sp2 + 1)) & 1u;
            double v0 = 0.0, v1 = 0.0;
            for (int e = tid; e < npair && (f0 || f1); e += KT) {
                const int d = e / NPR;
                const int gd = own[d];
                const int4 sd = A.sides[gd];
                const int ri = A.region[sd.x], rj = sd.z >= 0 ? A.region[sd.z] : -1;
                double gv[2] = {0.0, 0.0};
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int s = 2 * sp2 + h;
                    if (!((fresh >> s) & 1u)) continue;
                    const int li = ri < 0 ? 0 : s_loc[ri * NP + s];
                    double gg = A.hbar[A.h_base[sd.x] + (long long)li * A.ndof[sd.x] + sd.y];
                    if (sd.z >= 0) {
                        const int lj = rj < 0 ? 0 : s_loc[rj * NP + s];
                        gg = gg + A.hbar[A.h_base[sd.z] + (long long)lj * A.ndof[sd.z] + sd.w];
                    }
                    gv[h] = gg;
                    if (A.g) A.g[(long long)s_k[s] * n + gd] = gg;
                }
                const int pe = pel<NP>(d, 2 * sp2);
                double2 p2 = *reinterpret_cast<double2 *>(P + pe);
                double2 x2 = X2[e], r2 = R2[e];
                if (f0) { p2.x = gv[0]; r2.x = gv[0]; x2.x = 0.0; v0 += gv[0] * gv[0]; }
                if (f1) { p2.y = gv[1]; r2.y = gv[1]; x2.y = 0.0; v1 += gv[1] * gv[1]; }
                *reinterpret_cast<double2 *>(P + pe) = p2;
                X2[e] = x2;
                R2[e] = r2;
                const int2 pr = peer[d];
                if (pr.x >= 0)
                    *reinterpret_cast<double2 *>(cl.map_shared_rank(P, pr.x) +
                                                 pel<NP>(pr.y, 2 * sp2)) = p2;
            }
            const double tot = cluster_sum<NP>(v0, v1, s_red, s_ggg, cl, A.C, rank);
            if (tid < NP && ((fresh >> tid) & 1u)) {
                s_rr[tid] = tot;
                s_gn[tid] = sqrt(tot);
                s_state[tid] = SLOT_RUN;
                if (s_gn[tid] == 0.0) {           // interface.py:111-113
                    s_state[tid] = SLOT_DONE;
                    s_stat[tid] = MFB_CG_ZERO_RHS;
                }
            }
            __syncthreads();
        }
        unsigned run = 0;
#pragma unroll
        for (int s = 0; s < NP; ++s) run |= (unsigned)(s_state[s] == SLOT_RUN) << s;
        MFB_PT(0);

        // ---- Phase A: S p on the tensor cores. Units of this warp in pass 1
        //      (lower-side rows :=), a CTA barrier, pass 2 (upper-side rows
        //      += / to the owner's cut buffer); A fragments through the warp's
        //      TMA ring ----------------------------------------------------------
        if (run) {
            Ring rg;
            rg.base = smem_u32(RING) + (unsigned)(wid * RSLOT * SLOT_D * 8);
            rg.bar = smem_u32(s_bar) + (unsigned)(wid * RSLOT * 8);
            rg.head = 0;
            rg.used = 0;
            rg.par = s_par[wid];
            rg.pit.j = 0; rg.pit.pass = 0; rg.pit.k = 0; rg.pit.gi = -1;
            const unsigned psh = smem_u32(P), cmb = smem_u32(CM);
            for (int pass = 0; pass < 2; ++pass) {
                const int lo = pass ? n_u1 : 0, hi = pass ? n_units : n_u1;
                for (int u = lo + wid; u < hi; u += KW)
                    unit_dispatch<NP>(u, rg, units, strips, n_u1, n_units, s_gcnt, s_gloc,
                                      s_gmask, run, A.packed, psh, cmb, S, CB, cl);
                __syncthreads();
            }
            if (lane == 0) s_par[wid] = rg.par;
        }
        MFB_PT(1);
        cl.sync();                                  // cut rows landed
        MFB_PT(2);

        // ---- Phase A2: cut rows (lower + upper); p.S p -----------------------
        for (int e = tid; e < n_cut * NPR; e += KT) {
            const int qr = e / NPR, s = 2 * (e % NPR);
            double2 *sp = reinterpret_cast<double2 *>(S + pel<NP>(cut[qr], s));
            const double2 c2 = *reinterpret_cast<const double2 *>(CB + qr * NP + s);
            double2 v = *sp;
            v.x = v.x + c2.x;
            v.y = v.y + c2.y;
            *sp = v;
        }
        if (tid == 0) s_tctr = 0;                   // next Phase A (barriers in between)
        __syncthreads();
        {
            double v0 = 0.0, v1 = 0.0;
            if (((run >> (2 * sp2)) & 3u) != 0) {
#pragma unroll 4
                for (int e = tid; e < npair; e += KT) {
                    const int pe = pel<NP>(e / NPR, 2 * sp2);
                    const double2 p2 = *reinterpret_cast<const double2 *>(P + pe);
                    const double2 s2 = *reinterpret_cast<const double2 *>(S + pe);
                    v0 += p2.x * s2.x;
                    v1 += p2.y * s2.y;
                }
            }
            const double pSp = cluster_sum<NP>(v0, v1, s_red, s_gpsp, cl, A.C, rank);
            if (tid < NP && ((run >> tid) & 1u)) {
                s_it[tid] += 1;
                if (!(pSp > 0.0)) {                  // interface.py:123-126
                    s_state[tid] = SLOT_DONE;
                    s_stat[tid] = MFB_CG_NOT_SPD;
                } else {
                    s_a[tid] = s_rr[tid] / pSp;
                }
            }
            __syncthreads();
        }
        MFB_PT(3);
        unsigned upd = 0;
#pragma unroll
        for (int s = 0; s < NP; ++s) upd |= (unsigned)(((run >> s) & 1u) && s_state[s] == SLOT_RUN) << s;

        // ---- Phase B: x += a p, r -= a S p, r.r --------------------------------
        {
            double v0 = 0.0, v1 = 0.0;
            const bool u0 = (upd >> (2 * sp2)) & 1u, u1 = (upd >> (2 * sp2 + 1)) & 1u;
            if (u0 || u1) {
                const double a0 = s_a[2 * sp2], a1 = s_a[2 * sp2 + 1];
#pragma unroll 4
                for (int e = tid; e < npair; e += KT) {
                    const int pe = pel<NP>(e / NPR, 2 * sp2);
                    const double2 p2 = *reinterpret_cast<const double2 *>(P + pe);
                    const double2 s2 = *reinterpret_cast<const double2 *>(S + pe);
                    double2 x2 = X2[e], r2 = R2[e];
                    if (u0) {
                        x2.x += a0 * p2.x;
                        r2.x -= a0 * s2.x;
                        v0 += r2.x * r2.x;
                    }
                    if (u1) {
                        x2.y += a1 * p2.y;
                        r2.y -= a1 * s2.y;
                        v1 += r2.y * r2.y;
                    }
                    X2[e] = x2;
                    R2[e] = r2;
                }
            }
            const double rr_new = cluster_sum<NP>(v0, v1, s_red, s_grr, cl, A.C, rank);
            if (tid < NP && ((upd >> tid) & 1u)) {
                const double rn = sqrt(rr_new);
                const int it = s_it[tid];
                if (rank == 0) {
                    const int idx = it - 1;
                    if (idx % A.seg == 0) {
                        const long long sg = atomicAdd(A.seg_next, 1);
                        s_seg[tid] = sg < A.seg_cap ? (int)sg : -1;
                        A.seg_tab[(long long)s_k[tid] * A.max_segs + idx / A.seg] = s_seg[tid];
                    }
                    if (s_seg[tid] >= 0)
                        A.hist[(long long)s_seg[tid] * A.seg + idx % A.seg] = rn / s_gn[tid];
                }
                if (rn <= A.tol * s_gn[tid]) {
                    s_state[tid] = SLOT_DONE;
                    s_stat[tid] = MFB_CG_CONVERGED;
                } else if (it >= A.max_iter) {
                    s_state[tid] = SLOT_DONE;
                    s_stat[tid] = MFB_CG_MAX_ITER;
                } else {
                    s_b[tid] = rr_new / s_rr[tid];
                    s_rr[tid] = rr_new;
                }
            }
            __syncthreads();
        }

        MFB_PT(4);
        // ---- Phase C: p = r + beta p (owned rows and the peers' halo rows);
        //      finished slots write their solution ---------------------------
        {
            unsigned cont = 0, fin = 0;
#pragma unroll
            for (int s = 0; s < NP; ++s) {
                cont |= (unsigned)(((upd >> s) & 1u) && s_state[s] == SLOT_RUN) << s;
                fin |= (unsigned)(s_k[s] >= 0 && s_state[s] == SLOT_DONE) << s;
            }
            const bool c0 = (cont >> (2 * sp2)) & 1u, c1 = (cont >> (2 * sp2 + 1)) & 1u;
            const bool z0 = (fin >> (2 * sp2)) & 1u, z1 = (fin >> (2 * sp2 + 1)) & 1u;
            if (c0 || c1) {
                const double b0 = s_b[2 * sp2], b1 = s_b[2 * sp2 + 1];
#pragma unroll 4
                for (int e = tid; e < npair; e += KT) {
                    const int d = e / NPR;
                    const int pe = pel<NP>(d, 2 * sp2);
                    double2 p2 = *reinterpret_cast<double2 *>(P + pe);
                    const double2 r2 = R2[e];
                    if (c0) p2.x = r2.x + b0 * p2.x;
                    if (c1) p2.y = r2.y + b1 * p2.y;
                    *reinterpret_cast<double2 *>(P + pe) = p2;
                    const int2 pr = peer[d];
                    if (pr.x >= 0)
                        *reinterpret_cast<double2 *>(cl.map_shared_rank(P, pr.x) +
                                                     pel<NP>(pr.y, 2 * sp2)) = p2;
                }
            }
            if (z0 || z1) {
                for (int e = tid; e < npair; e += KT) {
                    const double2 x2 = X2[e];
                    const int gd = own[e / NPR];
                    if (z0)
                        A.lam[(long long)s_k[2 * sp2] * n + gd] =
                            s_stat[2 * sp2] == MFB_CG_ZERO_RHS ? 0.0 : x2.x;
                    if (z1)
                        A.lam[(long long)s_k[2 * sp2 + 1] * n + gd] =
                            s_stat[2 * sp2 + 1] == MFB_CG_ZERO_RHS ? 0.0 : x2.y;
                }
            }
            __syncthreads();
            if (tid < NP && ((fin >> tid) & 1u)) {
                if (rank == 0) {
                    A.iters[s_k[tid]] = s_stat[tid] == MFB_CG_ZERO_RHS ? 0 : s_it[tid];
                    A.status[s_k[tid]] = s_stat[tid];
                }
                s_k[tid] = -1;
            }
        }
        MFB_PT(5);
        cl.sync();                                  // halo rows of p landed
        MFB_PT(6);
        pt[7] += (A.dbg == 100 && tid == 0) ? 1 : 0;
    }
    if (A.dbg == 100 && tid == 0 && blockIdx.x < 1024) {
        for (int i = 0; i < 8; ++i) g_cl_prof[blockIdx.x * 8 + i] = pt[i];
        for (int i = 0; i < 4; ++i) g_cl_prof[8 * 1024 - 4 * 1024 + blockIdx.x * 4 + i] = s_dbg[i];
    }
#undef MFB_PT
}

template <int NP>
int launch_cluster(const ClArgs &A, int n_clusters, size_t smem, cudaStream_t st) {
    auto kern = cg_cluster_kernel<NP>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return MFB_ERR_SMEM;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = A.C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(KT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(A.C * n_clusters, 1, 1);
    if (cudaLaunchKernelEx(&cfg, kern, A) != cudaSuccess) return MFB_ERR_LAUNCH;
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}

}  // namespace

extern "C" int mfb_debug_cluster(int v) {
    g_cl_dbg = v;
    const int on = v == 101 || v == 102, z = 0, nf = v == 102;
    cudaMemcpyToSymbol(g_cl_dbg_nofence, &nf, sizeof(int));
    cudaMemcpyToSymbol(g_trace_on, &on, sizeof(int));
    cudaMemcpyToSymbol(g_trace_n, &z, sizeof(int));
    return 0;
}

// per-CTA phase cycle totals of the last profiled launch (mfb_debug_cluster(100))
extern "C" int mfb_debug_cluster_prof(long long *out, int n) {
    if (n > 1024 * 8) n = 1024 * 8;
    return cudaMemcpyFromSymbol(out, g_cl_prof, sizeof(long long) * n) == cudaSuccess ? 0 : 2;
}

// co-resident clusters of C CTAs with `smem` bytes of dynamic shared memory
extern "C" int mfb_cg_cluster_max_clusters(int C, int NP, int n_own_max, long long smem) {
    (void)n_own_max;
    if (C < 1 || C > KMAXC || (NP != 8 && NP != 16) || smem > 227 * 1024) return -MFB_ERR_ARG;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(KT, 1, 1);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(C * 1024, 1, 1);
    int maxc = 0;
    cudaError_t e;
    if (NP == 8) {
        if (cudaFuncSetAttribute(cg_cluster_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess) { cudaGetLastError(); return -MFB_ERR_SMEM; }
        e = cudaOccupancyMaxActiveClusters(&maxc, cg_cluster_kernel<8>, &cfg);
    } else {
        if (cudaFuncSetAttribute(cg_cluster_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess) { cudaGetLastError(); return -MFB_ERR_SMEM; }
        e = cudaOccupancyMaxActiveClusters(&maxc, cg_cluster_kernel<16>, &cfg);
    }
    if (e != cudaSuccess) { cudaGetLastError(); return -MFB_ERR_LAUNCH; }
    return maxc;
}

// dynamic shared memory of the cluster CG for a rank layout (cgcluster.py):
// flags bit 0: r in shared memory, bit 1: x in shared memory
extern "C" long long mfb_cg_cluster_smem(int NP, int n_used_max, int n_own_max, int n_cut_max,
                                         int n_cm_max, int n_unit_max, int n_strip_max,
                                         int n_regions, int flags) {
    long long b = 8LL * NP * (n_used_max + ((flags & 4) ? 0 : n_own_max) +
                              (n_cut_max > 0 ? n_cut_max : 1));
    if (flags & 1) b += 8LL * NP * n_own_max;
    if (flags & 2) b += 8LL * NP * n_own_max;
    b += 8LL * KW * RSLOT * SLOT_D;
    b += 4LL * n_cm_max + 4LL * (3LL * n_regions * NP + n_regions);
    b = (b + 15) / 16 * 16 + 32LL * n_unit_max + 16LL * n_strip_max;
    return b;
}

extern "C" int mfb_cg_cluster(int n_lambda, int C, int NP, const int *hdr, const int *tab,
                              int n_own_max, int n_used_max, int n_cut_max, int n_cm_max,
                              int n_unit_max, int n_strip_max, int flags, long long smem, const int *ndof, const int *region,
                              int n_regions, const long long *h_base, const int *local_idx,
                              int n_real, const double *hbar, const int *sides,
                              const double *packed, int k0, int n_pts, double tol, int max_iter,
                              double *lam, int *iters, int *status, double *g, double *xs,
                              double *rs, double *ss, int n_clusters, int *counter, double *hist, int seg,
                              long long seg_cap, int *seg_tab, int max_segs, int *seg_counter,
                              void *stream) {
    if (n_pts <= 0) return n_pts == 0 ? MFB_OK : MFB_ERR_ARG;
    if (n_lambda <= 0 || C < 1 || C > KMAXC || (NP != 8 && NP != 16) || n_own_max < 0 ||
        n_used_max < n_own_max || n_cut_max < 0 || n_regions < 0 || max_iter < 1 || seg < 1 ||
        max_segs < (max_iter + seg - 1) / seg || n_clusters < 1 ||
        smem < mfb_cg_cluster_smem(NP, n_used_max, n_own_max, n_cut_max, n_cm_max, n_unit_max,
                                   n_strip_max, n_regions, flags) ||
        smem > 227 * 1024 || (!(flags & 1) && !rs) || (!(flags & 2) && !xs) ||
        ((flags & 4) && !ss))
        return MFB_ERR_ARG;
    cudaStream_t st = mfb_stream(stream);
    if (cudaMemsetAsync(counter, 0, sizeof(int), st) != cudaSuccess) return MFB_ERR_LAUNCH;
    if (cudaMemsetAsync(seg_counter, 0, sizeof(int), st) != cudaSuccess) return MFB_ERR_LAUNCH;
    ClArgs A = {};
    A.n_lambda = n_lambda; A.n_regions = n_regions; A.n_real = n_real; A.k0 = k0;
    A.n_pts = n_pts; A.max_iter = max_iter; A.C = C;
    A.own_max = n_own_max; A.used_max = n_used_max; A.cut_max = n_cut_max > 0 ? n_cut_max : 1;
    A.cm_max = n_cm_max; A.unit_max = n_unit_max; A.strip_max = n_strip_max; A.r_smem = flags & 1; A.x_smem = (flags >> 1) & 1;
    A.s_glob = (flags >> 2) & 1;
    A.tol = tol;
    A.hdr = hdr; A.tab = tab; A.local_idx = local_idx; A.ndof = ndof; A.region = region;
    A.sides = reinterpret_cast<const int4 *>(sides);
    A.h_base = h_base; A.hbar = hbar; A.packed = packed;
    A.lam = lam; A.g = g; A.xs = xs; A.rs = rs; A.ss = ss; A.hist = hist;
    A.iters = iters; A.status = status; A.next = counter; A.seg_tab = seg_tab;
    A.seg_next = seg_counter; A.seg = seg; A.max_segs = max_segs; A.seg_cap = seg_cap;
    A.dbg = g_cl_dbg;
    return NP == 8 ? launch_cluster<8>(A, n_clusters, (size_t)smem, st)
                   : launch_cluster<16>(A, n_clusters, (size_t)smem, st);
}
