// Batched interface CG for large interfaces: MP collocation points per CTA.
//
// When a point's gathered flux-basis blocks no longer fit in shared memory
// (cfg4: n_lambda = 2,720, 128 subdomains, 2.1 MB of blocks per point), the
// one-CTA-per-point kernel (mfb_cg.cu) re-reads every block from L2 on every
// CG iteration, and the sweep runs at the L2 bandwidth (~11 TB/s, 27 us per
// point-iteration on cfg4). This kernel keeps MP = 8 points of the sweep in
// flight per CTA, in lockstep: each block tile is read from L2 ONCE per
// iteration and applied to every slot whose local realization uses it (all
// slots for the frozen Stokes blocks; the slots sharing a Darcy local
// realization otherwise). Slots are refilled from a global work counter as
// their points converge (persistent CTAs), so points with long iteration
// counts do not hold the others back.
//
// Per point the algorithm is the reference's (interface.py:107-139, 238-247)
// and the arithmetic is independent of which slot / CTA / neighbours a point
// gets: the row products accumulate over the block's columns in order,
// Sp[d] = row_lower + row_upper (basis_apply's ascending-sid scatter from
// zero), and the dot products use a fixed shuffle tree + fixed warp order.
// Same stopping test, breakdown test, zero-rhs exit and outputs as
// mfb_cg_batched.
//
// S p runs on the FP64 tensor cores: with MP = 8 the slots are exactly the
// N dimension of mma.m8n8k4.f64 -- a warp multiplies an 8-row tile of a
// block (A, read from L2 once per iteration) by the 4 x 8 tile of the slots'
// p at those columns (B, from shared memory) into an 8 (rows) x 8 (slots)
// accumulator. A slot on another local realization gets a zero B column,
// which leaves its accumulator untouched, so per slot the result is the same
// sequence of MMA updates whatever the other slots hold.
//
// Layout: p of the MP slots in shared memory, interleaved [n_lambda][MP]
// (64 bytes per mortar dof, slot halves of every other dof pair exchanged:
// conflict-free B operands); r in the SM's tensor memory (tcgen05.ld / .st,
// thread-private); x and S p in a per-CTA global scratch with p's layout
// (2 x 174 KB per CTA at cfg4, L2 resident). Work items ("tasks") are runs of
// <= 8 (task loop) or <= 16 (streamed walk) mortar dofs of one interface: the
// warp computes both sides' row tiles (an interface's dofs are contiguous in
// both adjacent subdomains' local orders) and adds them, lower subdomain
// first. The vector phases run elementwise over (dof, slot pair) with
// 16-byte accesses. Two forms of S p: the task loop (side_mma / strip_pass,
// any configuration) and the streamed walk over per-warp pass lists
// (stream_walk, when the lists fit in shared memory: the cfg4 path).
#include "mfb_common.cuh"

namespace {

constexpr int MP = 8;            // points in flight per CTA (= the MMA's N)
constexpr int MNT = 512;         // threads per CTA
constexpr int MW = MNT / 32;
constexpr int MREG = 64;         // KL regions cached per slot
constexpr int MPF = 8;           // A fragments prefetched per side (32 columns)
constexpr int VB_STREAM = 3;     // vector phases: elements per thread with loads in flight together

struct CgMultiArgs {
    int n_lambda, n_sub, n_regions, n_real, k0, n_pts, max_iter, hist_cap, n_tasks;
    double tol;
    const int *ndof, *dof_ptr, *dof_map, *region, *local_idx;
    const long long *blk_base, *h_base;
    const double *blocks, *hbar;
    const int4 *tasks;           // {d0, strip lower, strip upper, i | (j + 1) << 12 | R << 24}
    const int4 *trec;            // per task 3 int4: the run, side metadata, side strips
    const double *packed;        // blocks as MMA-fragment strips (mfb_cg_pack)
    const long long *pk_base;    // per sid: packed block of loc l at pk_base + l * pk_size
    const int *pk_size;
    const int4 *sides;           // per dof {i, a_i, j, a_j} (j = -1: one side)
    double *lam, *res_hist, *g, *scratch;
    int *seg_tab, *seg_next;       // segmented histories (seg_tab != NULL; hist_cap = segment)
    int max_segs;
    long long seg_cap;
    int *iters, *status, *next;
    const int *chunk_ptr;          // claims of <= MP consecutive points (NULL: one point per claim)
    int n_chunks;
    int list_cap;                  // pass-list entries per warp (streamed S p); 0: task loop
    const int *dm_tab;             // the dof list as the kernel reads it (p offsets, see below)
    int n_dm;
};

// p of the MP slots lives in shared memory as [dof][slot], 64 bytes per dof,
// with the two slot halves of every other dof PAIR exchanged: slot s of dof d
// at double d * 8 + (s ^ ((d & 2) << 1)). The B operand of an MMA reads, per
// half warp, slots 0-3 (4-7) of four consecutive dofs -- 32 bytes at a
// 64-byte stride, a two-way bank conflict in the plain layout; exchanged,
// the four dofs cover all 32 banks. The dof lists hold d * 8 + ((d & 2) << 1),
// so a lane's address is list ^ g; the vector phases see a permutation
// within each dof's 64 bytes (pidx).
__device__ __forceinline__ int pidx(int e) { return e ^ ((e >> 2) & 2); }

// ---- r in tensor memory -----------------------------------------------------
// The vector phases and phase A's A stream share one limit, the L2 -> SM
// bandwidth (x, r, S p round trips: 1 MB of the 3.6 MB a CTA moves per
// iteration at cfg4). r is private to the thread that updates it -- element
// e = tid + k * MNT in every phase -- so it lives in the SM's tensor memory
// (256 KB, idle in an FP64 kernel) instead of the global scratch: warp w owns
// lanes 32 (w % 4) .. + 31 (the quadrant its tcgen05.ld / .st may touch) and
// 4 columns (one double2) per element at column 4 KA (w / 4) + 4 k.
__device__ __forceinline__ void tm_ld(unsigned ta, double2 (&v)[1]) {
    unsigned a, b, c, d;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
                 "tcgen05.wait::ld.sync.aligned;"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(ta) : "memory");
    v[0] = make_double2(__hiloint2double(b, a), __hiloint2double(d, c));
}
__device__ __forceinline__ void tm_st(unsigned ta, double2 v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};"
                 :: "r"(ta), "r"(__double2loint(v.x)), "r"(__double2hiint(v.x)),
                    "r"(__double2loint(v.y)), "r"(__double2hiint(v.y)) : "memory");
}
// issue / wait / fence pieces for batches (the fence ties the registers to
// the wait: volatile asms keep their order, the uses read the fenced values)
#define TM_LD4(ta, v)                                                            \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];" \
                 : "=r"((v)[0]), "=r"((v)[1]), "=r"((v)[2]), "=r"((v)[3]) : "r"(ta) : "memory")
#define TM_WAIT_LD() asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory")
#define TM_FENCE4(v) \
    asm volatile("" : "+r"((v)[0]), "+r"((v)[1]), "+r"((v)[2]), "+r"((v)[3]) :: "memory")
__device__ __forceinline__ double2 tm_d2(const unsigned (&v)[4]) {
    return make_double2(__hiloint2double(v[1], v[0]), __hiloint2double(v[3], v[2]));
}
#ifdef MFB_A_NOALLOC
__device__ __forceinline__ double2 ldg_a(const double2 *p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                 : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
#else
__device__ __forceinline__ double2 ldg_a(const double2 *p) { return __ldg(p); }
#endif
#ifdef MFB_SCRATCH_CG
#define SC_LD(p) __ldcg(p)
#define SC_ST(p, v) __stcg(p, v)
#else
#define SC_LD(p) (*(p))
#define SC_ST(p, v) (*(p) = (v))
#endif
// B operand of the streamed walk: the dof lists hold absolute shared-memory
// byte addresses (p is 128-byte aligned), a lane's address is list ^ (g << 3)
__device__ __forceinline__ double lds_f64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void tm_st_wait() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}


__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// per-slot sums of the two slots (2 q, 2 q + 1) a thread accumulated, with
// q = threadIdx.x & 3 fixed for the thread: fixed xor tree over the lanes
// sharing q, then the warps in order
__device__ __forceinline__ void reduce_pairs(double &v0, double &v1, double (*red)[MP],
                                             double *out) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, o);
        v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    }
    if (lane < 4) {
        red[wid][2 * lane] = v0;
        red[wid][2 * lane + 1] = v1;
    }
    __syncthreads();
    if (threadIdx.x < MP) {
        double t = 0.0;
        for (int w = 0; w < MW; ++w) t += red[w][threadIdx.x];
        out[threadIdx.x] = t;
    }
    __syncthreads();
}

// acc += the 8-row strip at `soff` of subdomain sid's packed block (slot
// n's block: local realization s_loc[region][n]) times the slots' p. A strip
// holds the A fragments of its MMAs in lane order: fragment t of lane
// (g, q) = B[r0 + g][4 t + q] at strip[32 t + lane] (zero-padded), so every
// A load is one coalesced 256-byte warp access.
// One pass over a strip for the slots of mask m (block of local realization
// l): NT4 > 0 is the compile-time fragment count (ndof == 4 NT4, no bounds
// checks), 0 the generic path.
template <int NT4>
__device__ __forceinline__ void strip_pass(const double *__restrict__ Sl, const int *dm, int nd,
                                           const double *__restrict__ ps, int m,
                                           double &d0, double &d1) {
    const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
    const int nt4 = NT4 > 0 ? NT4 : (nd + 3) >> 2;
    // Two accumulator chains (even / odd fragments) halve the MMA dependency
    // chain; their sum is the row product
    double e0 = 0.0, e1 = 0.0, o0 = 0.0, o1 = 0.0;
#pragma unroll
    for (int t0 = 0; t0 < (NT4 > 0 ? NT4 : nt4); t0 += MPF) {
        double af[MPF];
        int dv[MPF];
#pragma unroll
        for (int t = 0; t < MPF; ++t) {
            if (NT4 > 0 ? (t0 + t < NT4) : (t0 + t < nt4)) {
                af[t] = __ldg(Sl + 32 * (t0 + t));
                const int c = 4 * (t0 + t) + q;
                dv[t] = (NT4 > 0 || c < nd) ? dm[c] ^ g : g;
            }
        }
#pragma unroll
        for (int t = 0; t < MPF; t += 2) {
            if (NT4 > 0 ? (t0 + t >= NT4) : (t0 + t >= nt4)) break;
            dmma884(e0, e1, af[t], ps[dv[t]]);
            if (NT4 > 0 ? (t0 + t + 1 < NT4) : (t0 + t + 1 < nt4))
                dmma884(o0, o1, af[t + 1], ps[dv[t + 1]]);
        }
    }
    // B was every slot's p: a column only feeds its own slot's outputs, so the
    // group's members take the products and the other slots keep their
    // accumulators (what a zero B column gives: x + 0 = x)
    if ((m >> (2 * q)) & 1) d0 += e0 + o0;
    if ((m >> (2 * q + 1)) & 1) d1 += e1 + o1;
}

// acc += the 8-row strip at `soff` of subdomain sid's packed block (slot
// n's block: local realization of its region) times the slots' p. A strip
// holds the A fragments of its MMAs in lane order: fragment t of lane
// (g, q) = B[r0 + g][4 t + q] at strip[32 t + lane] (zero-padded), so every
// A load is one coalesced 256-byte warp access. The slots are visited by
// local-realization group (g_cnt / g_loc / g_mask per region, rebuilt when
// slots are refilled); the frozen Stokes blocks are one group.
__device__ __forceinline__ void side_mma(const double *__restrict__ packed, int nd, int reg,
                                         int dmo, int pkb, int psz,
                                         const double *__restrict__ ps, const int *sdm,
                                         const int *g_cnt, const int *g_loc, const int *g_mask,
                                         int live, double &d0, double &d1) {
    const int lane = threadIdx.x & 31;
    const int *dm = sdm + dmo;                  // shared: dof * MP
    const double *base = packed + pkb + lane;
    const int ngrp = reg < 0 ? 1 : g_cnt[reg];
    for (int gi = 0; gi < ngrp; ++gi) {
        const int m = reg < 0 ? live : (g_mask[reg * MP + gi] & live);
        if (!m) continue;
        const int l = reg < 0 ? 0 : g_loc[reg * MP + gi];
        const double *Sl = base + (long long)l * psz;
        switch (nd) {
        case 16: strip_pass<4>(Sl, dm, nd, ps, m, d0, d1); break;
        case 24: strip_pass<6>(Sl, dm, nd, ps, m, d0, d1); break;
        case 32: strip_pass<8>(Sl, dm, nd, ps, m, d0, d1); break;
        case 40: strip_pass<10>(Sl, dm, nd, ps, m, d0, d1); break;
        case 48: strip_pass<12>(Sl, dm, nd, ps, m, d0, d1); break;
        case 56: strip_pass<14>(Sl, dm, nd, ps, m, d0, d1); break;
        case 64: strip_pass<16>(Sl, dm, nd, ps, m, d0, d1); break;
        default: strip_pass<0>(Sl, dm, nd, ps, m, d0, d1); break;
        }
    }
}

// strips[e] = {sid, r0, rows, strip offset}: copy rows r0..r0+rows-1 of every
// local realization's block of sid (column-major Bt[c*nd + r]) into
// fragment order (zero-padded to 8 rows x 4-column multiples)
__global__ void cg_pack_kernel(const int4 *__restrict__ strips, const int *__restrict__ ndof,
                               const int *__restrict__ n_loc, const long long *__restrict__ blk_base,
                               const long long *__restrict__ pk_base,
                               const int *__restrict__ pk_size, const double *__restrict__ blocks,
                               double *__restrict__ packed, int layout) {
    const int4 S = strips[blockIdx.x];
    const int sid = S.x, nd = ndof[sid];
    const int nt4 = (((nd + 3) >> 2) + 1) & ~1;      // strips hold an even number of fragments
    for (int l = blockIdx.y; l < n_loc[sid]; l += gridDim.y) {
        const double *B = blocks + blk_base[sid] + (long long)l * nd * nd;
        double *D = packed + pk_base[sid] + (long long)l * pk_size[sid] + S.w;
        for (int e = threadIdx.x; e < 32 * nt4; e += blockDim.x) {
            const int lane = e & 31, g = lane >> 2, c = 4 * (e >> 5) + (lane & 3);
            // layout 1: the lane's fragments 2 k, 2 k + 1 adjacent (one 16-byte load)
            // (a paired strip alternates with its partner: 128 doubles per pair)
            const int dst = layout ? ((S.z >> 8) ? 128 : 64) * (e >> 6) + 2 * lane + ((e >> 5) & 1)
                                   : e;
            D[dst] = (g < (S.z & 0xff) && c < nd) ? B[(long long)c * nd + S.y + g] : 0.0;
        }
    }
}


// ---- streamed S p --------------------------------------------------------
// The task loop above issues a pass's A loads and then waits a full L2
// round trip before its first MMA: with 16 warps x 8 fragments the loads in
// flight average about half of what the 32 KB could be. The streamed form
// keeps a ROLLING window instead: every warp walks a flat list of its passes
// (rebuilt in shared memory when the slots' local realizations change), and
// each step -- two fragments, the even / odd accumulator chains -- multiplies
// the two oldest fragments of an 8-fragment register window and at once
// re-issues their slots for the step four ahead, across pass and task
// boundaries. Same MMA sequence per (slot, row) as the task loop: same bits.
//
// list entry (int2): x = offset of the pass's strip in fragment pairs (packed
// + 64 x), y = steps | side << 5 | task end << 6 | list end << 7 | slot mask
// << 8 | the block's offset in the (padded, pair-interleaved) dof list << 16. A task-end entry is followed by
// the task's record {first dof, rows | has upper << 8}.
constexpr int PL_SIDE = 1 << 5, PL_TEND = 1 << 6, PL_END = 1 << 7;
constexpr int PL_DBL = 1 << 30, PL_XMASK = PL_DBL - 1;   // in x: a 16-row pass

__device__ __forceinline__ void build_pass_list(const CgMultiArgs &A, int2 *L, int run,
                                                const int *g_cnt, const int *g_loc,
                                                const int *g_mask) {
    int n = 0;
    for (int ti = threadIdx.x >> 5; ti < A.n_tasks; ti += MW) {
        const int4 T = __ldg(A.trec + 3 * ti), U = __ldg(A.trec + 3 * ti + 1),
                   V = __ldg(A.trec + 3 * ti + 2);
        if (T.w < 0) continue;                      // (no task at this position)
        const int j = ((T.w >> 12) & 0xfff) - 1, Rr = T.w >> 24;
        int last = -1;
        for (int side = 0; side < (j >= 0 ? 2 : 1); ++side) {
            const int ndr = side ? U.y : U.x, dmo = side ? U.w : U.z;
            const int pkb = side ? V.y : V.x, psz = side ? V.w : V.z;
            const int nd = ndr & 0xffff, reg = (ndr >> 16) - 1;
            const int steps = (((nd + 3) >> 2) + 1) >> 1;
            const int ngrp = reg < 0 ? 1 : g_cnt[reg];
            for (int gi = 0; gi < ngrp; ++gi) {
                const int m = reg < 0 ? 0xff : g_mask[reg * MP + gi];
                if (!(m & run)) continue;
                const int l = reg < 0 ? 0 : g_loc[reg * MP + gi];
                last = n;
                L[n++] = make_int2((int)(((long long)pkb + (long long)l * psz) >> 6) |
                                       (Rr > 8 ? PL_DBL : 0),
                                   (int)((unsigned)steps | (side ? PL_SIDE : 0) | (m << 8) |
                                         ((unsigned)dmo << 16)));
            }
        }
        if (last >= 0) {
            L[last].y |= PL_TEND;
            L[n++] = make_int2(T.x, Rr | (j >= 0 ? 256 : 0));
        }
    }
    L[n] = make_int2(0, PL_END);
}

// One warp's S p over its pass list from entry i0; returns this thread's
// p . S p partials (slots 2 q, 2 q + 1) in v0 / v1 and the entry it stopped
// at. The packed strips are pair-interleaved (mfb_cg_pack layout 1: fragments
// 2 k, 2 k + 1 of lane l adjacent, one 16-byte load per step) and so is the
// dof list (the two fragments' rows of lane q adjacent, one 8-byte load per
// step). DBL: the 16-row passes at the head of the list -- two strips whose
// fragment pairs alternate in memory, every B operand feeding both (four
// MMAs per step); the walk stops at the first 8-row pass.
template <bool DBL>
__device__ __forceinline__ int stream_walk(const CgMultiArgs &A, const int2 *L, int i0, int run,
                                           const double *__restrict__ ps, const int *sdm,
                                           double2 *__restrict__ S2, const double2 *P2,
                                           double &v0, double &v1) {
    const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3, g8 = g << 3;
    const double2 *__restrict__ pk = reinterpret_cast<const double2 *>(A.packed) + lane;
    const int2 *dmq = reinterpret_cast<const int2 *>(sdm) + q;
    int iL = i0, iC = i0;
    int2 eC = L[i0];
#define PL_STOP(e) (((e).y & PL_END) || (DBL && !((e).x & PL_DBL)))
    if (PL_STOP(eC)) return i0;
    int yL = eC.y, nL = yL & 31, nC = nL;
    const double2 *pL = pk + ((long long)(eC.x & PL_XMASK) << 5);
    // The B operands are fetched by the LOAD cursor too, four steps ahead
    // (p does not change during the walk): the dof-list entry of the next
    // step to issue is already in ddL, so a step's MMAs wait on nothing but
    // the tensor pipe -- the list -> p -> MMA chain of two shared-memory
    // latencies is off the critical path.
    const int2 *dmL = dmq + ((unsigned)eC.y >> 17);
    int2 ddL = *dmL;
    dmL += 4;
    double2 af[4], ag[DBL ? 4 : 1], bq[4];
    double e0 = 0.0, e1 = 0.0, o0 = 0.0, o1 = 0.0, lo0 = 0.0, lo1 = 0.0, up0 = 0.0, up1 = 0.0;
    double E0 = 0.0, E1 = 0.0, O0 = 0.0, O1 = 0.0, LO0 = 0.0, LO1 = 0.0, UP0 = 0.0, UP1 = 0.0;
    // the list walk is a loop so that it stays a (rarely taken) branch
    // instead of a dozen predicated instructions in every step
#define PL_ISSUE(s)                                                      \
    do {                                                                 \
        af[s] = ldg_a(pL);                                               \
        if (DBL) ag[s] = ldg_a(pL + 32);                                 \
        pL += DBL ? 64 : 32;                                             \
        bq[s].x = lds_f64(ddL.x ^ g8);                                   \
        bq[s].y = lds_f64(ddL.y ^ g8);                                   \
        --nL;                                                            \
        while (nL == 0) {                                                \
            iL += 1 + ((yL >> 6) & 1);                                   \
            const int2 eN = L[iL];                                       \
            yL = eN.y;                                                   \
            nL = PL_STOP(eN) ? -1 : (yL & 31);                           \
            pL = pk + ((long long)(eN.x & PL_XMASK) << 5);               \
            dmL = dmq + ((unsigned)yL >> 17);                            \
        }                                                                \
        ddL = *dmL;                                                      \
        dmL += 4;                                                        \
    } while (0)
    PL_ISSUE(0); PL_ISSUE(1); PL_ISSUE(2); PL_ISSUE(3);
    for (;;) {
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            dmma884(e0, e1, af[s].x, bq[s].x);
            dmma884(o0, o1, af[s].y, bq[s].y);
            if (DBL) {
                dmma884(E0, E1, ag[s].x, bq[s].x);
                dmma884(O0, O1, ag[s].y, bq[s].y);
            }
            PL_ISSUE(s);
            if (--nC == 0) {
                // a column of B only feeds its own slot: the group's members
                // take the products, the other slots keep their accumulators
                const int m = (eC.y >> 8) & run;
                const bool m0 = (m >> (2 * q)) & 1, m1 = (m >> (2 * q + 1)) & 1;
                const double t0 = e0 + o0, t1 = e1 + o1;
                if (eC.y & PL_SIDE) {
                    if (m0) up0 += t0;
                    if (m1) up1 += t1;
                } else {
                    if (m0) lo0 += t0;
                    if (m1) lo1 += t1;
                }
                e0 = e1 = o0 = o1 = 0.0;
                if (DBL) {
                    const double T0 = E0 + O0, T1 = E1 + O1;
                    if (eC.y & PL_SIDE) {
                        if (m0) UP0 += T0;
                        if (m1) UP1 += T1;
                    } else {
                        if (m0) LO0 += T0;
                        if (m1) LO1 += T1;
                    }
                    E0 = E1 = O0 = O1 = 0.0;
                }
                if (eC.y & PL_TEND) {
                    const int2 rec = L[iC + 1];
                    iC += 2;
                    const int rows = rec.y & 0xff;
                    if (g < rows) {
                        const double2 sp = (rec.y & 256) ? make_double2(lo0 + up0, lo1 + up1)
                                                         : make_double2(lo0, lo1);
                        const int e = (rec.x + g) * (MP / 2) + q;
                        SC_ST(S2 + e, sp);
                        const double2 pp = P2[pidx(e)];
                        v0 += pp.x * sp.x;
                        v1 += pp.y * sp.y;
                    }
                    lo0 = lo1 = up0 = up1 = 0.0;
                    if (DBL) {
                        if (g + 8 < rows) {
                            const double2 sp = (rec.y & 256)
                                                   ? make_double2(LO0 + UP0, LO1 + UP1)
                                                   : make_double2(LO0, LO1);
                            const int e = (rec.x + 8 + g) * (MP / 2) + q;
                            SC_ST(S2 + e, sp);
                            const double2 pp = P2[pidx(e)];
                            v0 += pp.x * sp.x;
                            v1 += pp.y * sp.y;
                        }
                        LO0 = LO1 = UP0 = UP1 = 0.0;
                    }
                } else {
                    iC += 1;
                }
                eC = L[iC];
                if (PL_STOP(eC)) return iC;
                nC = eC.y & 31;
            }
        }
    }
#undef PL_ISSUE
#undef PL_STOP
}

__device__ __forceinline__ void stream_passes(const CgMultiArgs &A, const int2 *L, int run,
                                              const double *__restrict__ ps, const int *sdm,
                                              double2 *__restrict__ S2, const double2 *P2,
                                              double &v0, double &v1) {
    const int i1 = stream_walk<true>(A, L, 0, run, ps, sdm, S2, P2, v0, v1);
    stream_walk<false>(A, L, i1, run, ps, sdm, S2, P2, v0, v1);
}

enum { SLOT_RUN = 0, SLOT_NEW = 1, SLOT_DONE = 2 };

__device__ int g_multi_dbg;
__device__ long long g_multi_prof[148 * 8];
__device__ long long g_multi_warp[MW];          // phase A clocks per warp of CTA 0 (MFB_PHASE_PROF)
// phase clocks (tools/multi_phases.py) only in a -DMFB_PHASE_PROF build: the
// counters cost registers the production kernel needs
#ifdef MFB_PHASE_PROF
#define MP_T(i)                                                     \
    do {                                                            \
        if (dbg && threadIdx.x == 0) {                              \
            const long long t_ = clock64();                         \
            pt[i] += t_ - tc;                                       \
            tc = t_;                                                \
        }                                                           \
    } while (0)
#define MP_PROF 1
#else
#define MP_T(i) do { } while (0)
#define MP_PROF 0
#endif

template <bool STREAM>
__global__ void __launch_bounds__(MNT, 1) cg_multi_kernel(CgMultiArgs A) {
    extern __shared__ __align__(128) double ps[];   // [n_lambda][MP], then the dof lists
    __shared__ int s_k[MP], s_it[MP], s_state[MP], s_stat[MP], s_seg[MP];
    __shared__ double s_rr[MP], s_gn[MP], s_a[MP], s_b[MP], s_tot[MP];
    __shared__ int s_loc[MREG * MP];
    __shared__ int s_gcnt[MREG], s_gloc[MREG * MP], s_gmask[MREG * MP];
    __shared__ double s_red[MW][MP];
    __shared__ int s_any, s_q0, s_q1;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int n = A.n_lambda;
    const int npair = n * (MP / 2);
    const int sq = 2 * (tid & 3);                  // this thread's slot pair (vector phases)
    double *Xs = A.scratch + (long long)blockIdx.x * 3 * n * MP;
    double *Rs = Xs + (long long)n * MP;
    double *Ss = Rs + (long long)n * MP;
    // x, r, S p: disjoint thirds of this CTA's scratch
    double2 *__restrict__ X2 = reinterpret_cast<double2 *>(Xs);
    double2 *__restrict__ S2 = reinterpret_cast<double2 *>(Ss);
    double2 *P2 = reinterpret_cast<double2 *>(ps);
    int *sdm = reinterpret_cast<int *>(ps + (long long)n * MP);   // the dof list (A.dm_tab)
    int2 *plist = reinterpret_cast<int2 *>(sdm + ((A.n_dm + 1) & ~1)) +
                  (long long)wid * A.list_cap;        // this warp's pass list (STREAM)
    int prev_run = -1;
    constexpr int VB = STREAM ? VB_STREAM : 2;
    // tensor memory for r: all 512 columns (one CTA per SM)
    __shared__ unsigned s_tmem;
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                     :: "r"((unsigned)__cvta_generic_to_shared(&s_tmem)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // elements per thread, uniform over the warp (lanes past npair idle), and
    // the warp's column range
    const int kw = (npair - (wid << 5) + MNT - 1) / MNT;
    const int ka = ((npair + MNT - 1) / MNT + VB - 1) / VB * VB;
    const unsigned tr = s_tmem + ((unsigned)(32 * (wid & 3)) << 16) + (unsigned)((wid >> 2) * 4 * ka);
    if (tid < MP) { s_k[tid] = -1; s_state[tid] = SLOT_DONE; }
    if (tid == 0) { s_q0 = 0; s_q1 = 0; }
    for (int e = tid; e < n * MP; e += MNT) ps[e] = 0.0;
    {
        // streamed: absolute shared-memory byte addresses of the dofs' p
        const unsigned ps_sa = (unsigned)__cvta_generic_to_shared(ps);
        for (int e = tid; e < A.n_dm; e += MNT)
            sdm[e] = STREAM ? (int)(ps_sa + ((unsigned)A.dm_tab[e] << 3)) : A.dm_tab[e];
    }

#if MP_PROF
    const int dbg = g_multi_dbg;
    long long pt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tc = clock64();
#endif
    bool refill = true;               // a slot was freed (or the first trip)
    for (;;) {
        if (refill) {
        __syncthreads();
        // ---- refill empty slots from the global work counter --------------
        // A claim is a chunk of <= MP consecutive points of the sweep order
        // (the host groups points that share local realizations, so a CTA's
        // slots visit few distinct Darcy blocks per region); the chunk's
        // points go to this CTA's slots as they free up.
        if (tid == 0) {
            int any = 0, q0 = s_q0, q1 = s_q1;
            for (int s = 0; s < MP; ++s) {
                if (s_k[s] == -1) {
                    if (q0 == q1 && q1 >= 0) {
                        const int c = atomicAdd(A.next, 1);
                        if (A.chunk_ptr) {
                            if (c < A.n_chunks) { q0 = A.chunk_ptr[c]; q1 = A.chunk_ptr[c + 1]; }
                            else q0 = q1 = -1;
                        } else if (c < A.n_pts) { q0 = c; q1 = c + 1; }
                        else q0 = q1 = -1;
                    }
                    const int t = q0 < q1 ? q0++ : -2;
                    s_k[s] = t;
                    s_state[s] = t >= 0 ? SLOT_NEW : SLOT_DONE;
                    s_it[s] = 0;
                }
                any |= s_k[s] >= 0;
            }
            s_q0 = q0; s_q1 = q1;
            s_any = any;
        }
        __syncthreads();
        }
        if (!s_any) break;
        int fresh = 0;
#pragma unroll
        for (int s = 0; s < MP; ++s) fresh |= (s_state[s] == SLOT_NEW) << s;
        const bool f0 = (fresh >> sq) & 1, f1 = (fresh >> (sq + 1)) & 1;
        double v0 = 0.0, v1 = 0.0;
        if (fresh) {
            for (int e = tid; e < A.n_regions * MP; e += MNT) {
                const int s = e % MP;
                if ((fresh >> s) & 1)
                    s_loc[e] = A.local_idx[(long long)(e / MP) * A.n_real + A.k0 + s_k[s]];
            }
            __syncthreads();
            // per region: the distinct local realizations among the slots
            // holding points, with their slot masks (read after the barriers
            // of the reduction below)
            for (int r = tid; r < A.n_regions; r += MNT) {
                int cnt = 0;
                for (int s = 0; s < MP; ++s) {
                    if (s_k[s] < 0) continue;
                    const int l = s_loc[r * MP + s];
                    int j = 0;
                    while (j < cnt && s_gloc[r * MP + j] != l) ++j;
                    if (j == cnt) {
                        s_gloc[r * MP + cnt] = l;
                        s_gmask[r * MP + cnt] = 0;
                        ++cnt;
                    }
                    s_gmask[r * MP + j] |= 1 << s;
                }
                s_gcnt[r] = cnt;
            }
            // g = 0 + h_lower + h_upper (mortar.jump of the bar traces), x = 0
            for (int k = 0; k < kw; ++k) {
                const int e = tid + k * MNT;
                double2 rv[1];
                tm_ld(tr + 4 * k, rv);           // (the whole warp: .sync.aligned)
                if ((f0 || f1) && e < npair) {
                    const int d = e >> 2;
                    const int4 sd = A.sides[d];
                    const int ri = A.region[sd.x], rj = sd.z >= 0 ? A.region[sd.z] : -1;
                    double gv[2] = {0.0, 0.0};
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int s = sq + h;
                        if (!((fresh >> s) & 1)) continue;   // s_loc is only set for fresh slots
                        const int li = ri < 0 ? 0 : s_loc[ri * MP + s];
                        double gg = A.hbar[A.h_base[sd.x] + (long long)li * A.ndof[sd.x] + sd.y];
                        if (sd.z >= 0) {
                            const int lj = rj < 0 ? 0 : s_loc[rj * MP + s];
                            gg = gg + A.hbar[A.h_base[sd.z] + (long long)lj * A.ndof[sd.z] + sd.w];
                        }
                        gv[h] = gg;
                    }
                    double2 p2 = P2[pidx(e)], x2 = X2[e];
                    if (f0) {
                        p2.x = gv[0]; rv[0].x = gv[0]; x2.x = 0.0; v0 += gv[0] * gv[0];
                        if (A.g) A.g[(long long)s_k[sq] * n + d] = gv[0];
                    }
                    if (f1) {
                        p2.y = gv[1]; rv[0].y = gv[1]; x2.y = 0.0; v1 += gv[1] * gv[1];
                        if (A.g) A.g[(long long)s_k[sq + 1] * n + d] = gv[1];
                    }
                    P2[pidx(e)] = p2; X2[e] = x2;
                }
                tm_st(tr + 4 * k, rv[0]);
            }
            tm_st_wait();
            reduce_pairs(v0, v1, s_red, s_tot);
            if (tid < MP && ((fresh >> tid) & 1)) {
                s_rr[tid] = s_tot[tid];
                s_gn[tid] = sqrt(s_tot[tid]);
                s_state[tid] = SLOT_RUN;
                if (s_gn[tid] == 0.0) {          // interface.py:111-113
                    s_state[tid] = SLOT_DONE;
                    s_stat[tid] = MFB_CG_ZERO_RHS;
                }
            }
            __syncthreads();
        }
        int run = 0;
#pragma unroll
        for (int s = 0; s < MP; ++s) run |= (s_state[s] == SLOT_RUN) << s;
        MP_T(0);

        // ---- Phase A: S p on the tensor cores; p.S p --------------------------
        v0 = 0.0; v1 = 0.0;
        if (STREAM) {
            if (run) {
                if (fresh || run != prev_run) {     // the slots' blocks changed
                    if (lane == 0) build_pass_list(A, plist, run, s_gcnt, s_gloc, s_gmask);
                    __syncwarp();
                }
#if MP_PROF
                const long long tw0 = clock64();
#endif
                stream_passes(A, plist, run, ps, sdm, S2, P2, v0, v1);
#if MP_PROF
                if (dbg && lane == 0 && blockIdx.x == 0) g_multi_warp[wid] += clock64() - tw0;
#endif
            }
            prev_run = run;
        } else
        if (run) {
            const int g8 = lane >> 2;
            // task records {run}{nd | region + 1 << 16 per side, dof_ptr per side}
            // {packed strip base per side, packed block size per side}: the
            // next task's record is fetched while this task runs
            const int4 *rec = A.trec;
            for (int ti = wid; ti < A.n_tasks; ti += MW) {
                const int4 T = __ldg(rec + 3 * ti), U = __ldg(rec + 3 * ti + 1),
                           V = __ldg(rec + 3 * ti + 2);
                const int j = ((T.w >> 12) & 0xfff) - 1, Rr = T.w >> 24;
                double lo0 = 0.0, lo1 = 0.0, up0 = 0.0, up1 = 0.0;
                side_mma(A.packed, U.x & 0xffff, (U.x >> 16) - 1, U.z, V.x, V.z, ps, sdm, s_gcnt,
                         s_gloc, s_gmask, run, lo0, lo1);
                if (j >= 0)
                    side_mma(A.packed, U.y & 0xffff, (U.y >> 16) - 1, U.w, V.y, V.w, ps, sdm,
                             s_gcnt, s_gloc, s_gmask, run, up0, up1);
                if (g8 < Rr) {
                    const int d = T.x + g8;
                    const double2 sp = j >= 0 ? make_double2(lo0 + up0, lo1 + up1)
                                              : make_double2(lo0, lo1);
                    const int e = d * (MP / 2) + (lane & 3);
                    S2[e] = sp;
                    const double2 pp = P2[pidx(e)];
                    v0 += pp.x * sp.x;
                    v1 += pp.y * sp.y;
                }
            }
        }
        MP_T(1);
        reduce_pairs(v0, v1, s_red, s_tot);
        MP_T(2);
        if (tid < MP && ((run >> tid) & 1)) {
            const double pSp = s_tot[tid];
            s_it[tid] += 1;
            if (!(pSp > 0.0)) {                  // interface.py:123-126
                s_state[tid] = SLOT_DONE;
                s_stat[tid] = MFB_CG_NOT_SPD;
            } else {
                s_a[tid] = s_rr[tid] / pSp;
            }
        }
        __syncthreads();
        int upd = 0;
#pragma unroll
        for (int s = 0; s < MP; ++s) upd |= (((run >> s) & 1) && s_state[s] == SLOT_RUN) << s;

        // ---- Phase B: x += a p, r -= a S p, r.r (elementwise) -----------------
        v0 = 0.0; v1 = 0.0;
        const bool u0 = (upd >> sq) & 1, u1 = (upd >> (sq + 1)) & 1;
        if (upd) {                        // (uniform: r moves through tensor memory)
            const double a0 = s_a[sq], a1 = s_a[sq + 1];
            const bool act = u0 || u1;
            // VB elements per trip, their scratch loads issued together
            for (int k0 = 0; k0 < kw; k0 += VB) {
                double2 s2[VB], x2[VB], r2[VB];
                unsigned rr[VB][4];
#pragma unroll
                for (int k = 0; k < VB; ++k) TM_LD4(tr + 4 * (k0 + k), rr[k]);
#pragma unroll
                for (int k = 0; k < VB; ++k) {
                    const int e = tid + (k0 + k) * MNT;
                    if (act && e < npair) {
                        s2[k] = SC_LD(S2 + e);
                        x2[k] = SC_LD(X2 + e);
                    }
                }
                TM_WAIT_LD();
#pragma unroll
                for (int k = 0; k < VB; ++k) {
                    TM_FENCE4(rr[k]);
                    r2[k] = tm_d2(rr[k]);
                }
#pragma unroll
                for (int k = 0; k < VB; ++k) {
                    const int e = tid + (k0 + k) * MNT;
                    if (act && e < npair) {
                        const double2 p2 = P2[pidx(e)];
                        if (u0) {
                            x2[k].x = __dadd_rn(x2[k].x, __dmul_rn(a0, p2.x));
                            r2[k].x = __dsub_rn(r2[k].x, __dmul_rn(a0, s2[k].x));
                            v0 += r2[k].x * r2[k].x;
                        }
                        if (u1) {
                            x2[k].y = __dadd_rn(x2[k].y, __dmul_rn(a1, p2.y));
                            r2[k].y = __dsub_rn(r2[k].y, __dmul_rn(a1, s2[k].y));
                            v1 += r2[k].y * r2[k].y;
                        }
                        SC_ST(X2 + e, x2[k]);
                    }
                    tm_st(tr + 4 * (k0 + k), r2[k]);
                }
            }
            tm_st_wait();
        }
        MP_T(3);
        reduce_pairs(v0, v1, s_red, s_tot);
        MP_T(4);
        if (tid < MP && ((upd >> tid) & 1)) {
            const double rr_new = s_tot[tid];
            const double rn = sqrt(rr_new);
            const int it = s_it[tid];
            if (A.seg_tab) {
                const int idx = it - 1;
                if (idx % A.hist_cap == 0) {
                    const long long sg = atomicAdd(A.seg_next, 1);
                    s_seg[tid] = sg < A.seg_cap ? (int)sg : -1;
                    A.seg_tab[(long long)s_k[tid] * A.max_segs + idx / A.hist_cap] = s_seg[tid];
                }
                if (s_seg[tid] >= 0)
                    A.res_hist[(long long)s_seg[tid] * A.hist_cap + idx % A.hist_cap] =
                        rn / s_gn[tid];
            } else if (it <= A.hist_cap) {
                A.res_hist[(long long)s_k[tid] * A.hist_cap + it - 1] = rn / s_gn[tid];
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

        // ---- Phase C: p = r + beta p; finished slots write their solution ----
        int cont = 0, fin = 0;
#pragma unroll
        for (int s = 0; s < MP; ++s) {
            cont |= (((upd >> s) & 1) && s_state[s] == SLOT_RUN) << s;
            fin |= (s_k[s] >= 0 && s_state[s] == SLOT_DONE) << s;
        }
        const bool c0 = (cont >> sq) & 1, c1 = (cont >> (sq + 1)) & 1;
        const bool z0 = (fin >> sq) & 1, z1 = (fin >> (sq + 1)) & 1;
        if (cont || fin) {
            const double b0 = s_b[sq], b1 = s_b[sq + 1];
            if (cont) {                   // (uniform)
                for (int k0 = 0; k0 < kw; k0 += VB) {
                    double2 r2[VB];
                    unsigned rr[VB][4];
#pragma unroll
                    for (int k = 0; k < VB; ++k) TM_LD4(tr + 4 * (k0 + k), rr[k]);
                    TM_WAIT_LD();
#pragma unroll
                    for (int k = 0; k < VB; ++k) {
                        TM_FENCE4(rr[k]);
                        r2[k] = tm_d2(rr[k]);
                    }
#pragma unroll
                    for (int k = 0; k < VB; ++k) {
                        const int e = tid + (k0 + k) * MNT;
                        if (e >= npair || !(c0 || c1)) continue;
                        double2 p2 = P2[pidx(e)];
                        if (c0) p2.x = __dadd_rn(r2[k].x, __dmul_rn(b0, p2.x));
                        if (c1) p2.y = __dadd_rn(r2[k].y, __dmul_rn(b1, p2.y));
                        P2[pidx(e)] = p2;
                    }
                }
            }
            if (z0 || z1) {
                for (int e = tid; e < npair; e += MNT) {
                    const int d = e >> 2;
                    const double2 x2 = X2[e];
                    if (z0)
                        A.lam[(long long)s_k[sq] * n + d] =
                            s_stat[sq] == MFB_CG_ZERO_RHS ? 0.0 : x2.x;
                    if (z1)
                        A.lam[(long long)s_k[sq + 1] * n + d] =
                            s_stat[sq + 1] == MFB_CG_ZERO_RHS ? 0.0 : x2.y;
                }
            }
        }
        __syncthreads();
        MP_T(5);
#if MP_PROF
        pt[6] += dbg && tid == 0;
#endif
        refill = fin != 0;
        if (tid < MP && ((fin >> tid) & 1)) {
            A.iters[s_k[tid]] = s_stat[tid] == MFB_CG_ZERO_RHS ? 0 : s_it[tid];
            A.status[s_k[tid]] = s_stat[tid];
            s_k[tid] = -1;
        }
    }
#if MP_PROF
    if (dbg && threadIdx.x == 0 && blockIdx.x < 148)
        for (int i = 0; i < 8; ++i) g_multi_prof[blockIdx.x * 8 + i] = pt[i];
#endif
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (wid == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;"
                     :: "r"(s_tmem) : "memory");
}

}  // namespace

extern "C" int mfb_debug_multi_warps(long long *out, int reset) {
    long long z[MW] = {0};
    if (reset) return cudaMemcpyToSymbol(g_multi_warp, z, sizeof(z)) == cudaSuccess ? 0 : 2;
    return cudaMemcpyFromSymbol(out, g_multi_warp, sizeof(z)) == cudaSuccess ? 0 : 2;
}

extern "C" int mfb_debug_multi(int on, long long *out) {
    if (out)
        return cudaMemcpyFromSymbol(out, g_multi_prof, sizeof(long long) * 148 * 8) ==
                       cudaSuccess ? 0 : 2;
    return cudaMemcpyToSymbol(g_multi_dbg, &on, sizeof(int)) == cudaSuccess ? 0 : 2;
}

// dynamic shared memory: p of the MP slots, the dof list (n_dm entries) and,
// streamed, MW pass lists of list_cap entries
extern "C" long long mfb_cg_multi_smem(int n_lambda, int n_dm, int list_cap) {
    return (long long)n_lambda * MP * sizeof(double) +
           (long long)((n_dm + 1) & ~1) * sizeof(int) +
           (long long)MW * list_cap * sizeof(int2);
}

extern "C" long long mfb_cg_multi_scratch_doubles(int n_lambda, int n_cta) {
    return (long long)n_cta * 3 * n_lambda * MP;
}

extern "C" int mfb_cg_multi(int n_lambda, int n_sub, int n_rows, const int *ndof,
                            const int *dof_ptr,
                            const int *dof_map, const int *region, int n_regions,
                            const long long *blk_base, const long long *h_base,
                            const int *local_idx, int n_real, const double *blocks,
                            const double *hbar, int k0, int n_pts, double tol, int max_iter,
                            double *lam, int *iters, int *status, double *res_hist,
                            int hist_cap, double *g, const int *tasks, int n_tasks,
                            const int *sides, const double *packed, const long long *pk_base,
                            const int *pk_size, int n_cta, double *scratch, int *counter,
                            int *seg_tab, int max_segs, long long seg_cap, int *seg_counter,
                            const int *trec, const int *chunk_ptr, int n_chunks, int list_cap,
                            const int *dm_tab, int n_dm, void *stream) {
    if (n_pts <= 0) return n_pts == 0 ? MFB_OK : MFB_ERR_ARG;
    if (n_lambda <= 0 || n_sub <= 0 || n_sub >= 4095 || n_rows <= 0 || n_regions > MREG || n_cta <= 0 ||
        max_iter < 1 || hist_cap < 1 || n_tasks <= 0 || (chunk_ptr && n_chunks <= 0) ||
        list_cap < 0 || !dm_tab || n_dm < n_rows || (list_cap > 0 && n_dm >= 65536) ||
        (seg_tab && (max_segs < (max_iter + hist_cap - 1) / hist_cap || !seg_counter)))
        return MFB_ERR_ARG;
    // r of the slots in tensor memory: 16 columns per element a thread owns
    if (((n_lambda * (MP / 2) + MNT - 1) / MNT + VB_STREAM - 1) / VB_STREAM * VB_STREAM > 32)
        return MFB_ERR_SMEM;
    const size_t smem = mfb_cg_multi_smem(n_lambda, n_dm, list_cap);
    if (smem + 8192 > 227 * 1024) return MFB_ERR_SMEM;    // + the kernel's static tables
    if (cudaFuncSetAttribute(list_cap ? cg_multi_kernel<true> : cg_multi_kernel<false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return MFB_ERR_SMEM;
    cudaStream_t st = mfb_stream(stream);
    if (cudaMemsetAsync(counter, 0, sizeof(int), st) != cudaSuccess) return MFB_ERR_LAUNCH;
    CgMultiArgs A;
    A.n_lambda = n_lambda; A.n_sub = n_sub; A.n_regions = n_regions; A.n_real = n_real;
    A.k0 = k0; A.n_pts = n_pts; A.max_iter = max_iter; A.hist_cap = hist_cap;
    A.n_tasks = n_tasks; A.tol = tol;
    A.ndof = ndof; A.dof_ptr = dof_ptr; A.dof_map = dof_map; A.region = region;
    A.local_idx = local_idx; A.blk_base = blk_base; A.h_base = h_base;
    A.blocks = blocks; A.hbar = hbar;
    A.tasks = reinterpret_cast<const int4 *>(tasks);
    A.trec = reinterpret_cast<const int4 *>(trec);
    if (!trec) return MFB_ERR_ARG;
    A.sides = reinterpret_cast<const int4 *>(sides);
    A.packed = packed; A.pk_base = pk_base; A.pk_size = pk_size;
    A.lam = lam; A.res_hist = res_hist; A.g = g; A.scratch = scratch;
    A.iters = iters; A.status = status; A.next = counter;
    A.chunk_ptr = chunk_ptr; A.n_chunks = n_chunks;
    A.seg_tab = seg_tab; A.seg_next = seg_counter; A.max_segs = max_segs; A.seg_cap = seg_cap;
    if (seg_tab && cudaMemsetAsync(seg_counter, 0, sizeof(int), st) != cudaSuccess)
        return MFB_ERR_LAUNCH;
    A.list_cap = list_cap; A.dm_tab = dm_tab; A.n_dm = n_dm;
    if (list_cap)
        cg_multi_kernel<true><<<n_cta, MNT, smem, st>>>(A);
    else
        cg_multi_kernel<false><<<n_cta, MNT, smem, st>>>(A);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}

extern "C" int mfb_cg_pack(int n_strips, const int *strips, const int *ndof, const int *n_loc,
                           int max_loc, const long long *blk_base, const long long *pk_base,
                           const int *pk_size, const double *blocks, double *packed,
                           int layout, void *stream) {
    if (n_strips < 0 || max_loc < 0 || layout < 0 || layout > 1) return MFB_ERR_ARG;
    if (n_strips == 0 || max_loc == 0) return MFB_OK;
    dim3 grid(n_strips, max_loc < 64 ? max_loc : 64);
    cg_pack_kernel<<<grid, 128, 0, mfb_stream(stream)>>>(
        reinterpret_cast<const int4 *>(strips), ndof, n_loc, blk_base, pk_base, pk_size, blocks,
        packed, layout);
    MFB_CHECK_LAUNCH();
    return MFB_OK;
}
