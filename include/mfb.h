/*
 * mfb.h -- C ABI of the B200 (sm_100a) stochastic multiscale-flux-basis path.
 *
 * The reference (sdmortar 0.1.0, pure Python/numpy/scipy) has no FFI; its
 * seam is the Python function API of `sdmortar/interface.py`. Each entry
 * point below replaces one piece of that API's compute; the Python host
 * (paper_1802_06263_b200/interface.py) keeps the reference signatures and
 * binds these through ctypes.
 *
 *   mfb_kl_realize        <- LogPermField.realize / evaluate_log
 *                            (random_field.py:232-243, 125-140)
 *   mfb_kl_realize_ld     <- problem.permeability (problem.py:85-96), S2
 *   mfb_kl_realize_batched   every table of a sweep in one launch
 *   mfb_systems_solve     <- problem.assemble_subdomain + DarcyOperator /
 *                            StokesOperator factor + the N_dof star solves of
 *                            compute_flux_basis and the bar solve
 *                            (problem.py:98-112, darcy.py:67-154,
 *                             stokes.py:112-322, interface.py:218-235, 166-177)
 *   mfb_systems_apply     <- solve_star + side_functionals with stored
 *                            factors (S1's direct_apply, interface.py:180-194)
 *   mfb_s1_cg_begin/_step <- S1's compute_rhs + cg_solve (interface.py:107-139,
 *                            166-177), every point in lock step
 *   mfb_s1_fields         <- S1's recover_fields (interface.py:250-260)
 *   mfb_systems_extract   <- compute_flux_basis readout (interface.py:210-235),
 *                            side_functionals (problem.py:132-148),
 *                            postprocess (problem.py:150-158)
 *   mfb_cg_batched, _multi <- the S3 main loop's compute_rhs + cg_solve with
 *                            basis_apply (interface.py:107-139, 238-247,
 *                            331-334), all collocation points at once
 *   mfb_group_stats,
 *   mfb_group_fields,
 *   mfb_moments_reduce    <- recover_fields + MomentAccumulator for field keys
 *                            (interface.py:250-268, moments.py:25-58)
 *   mfb_lambda_moments    <- MomentAccumulator for the "lambda" key
 *                            (moments.py:25-58), fixed realization order
 *
 * Conventions: every pointer argument is a DEVICE pointer unless named
 * `host_*`; buffers are caller-allocated and never freed by the library;
 * calls are stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 * default stream); return 0 on success or an MFB_ERR_* code. Per-item
 * numerical failures (singular pivots, CG breakdown) are reported in the
 * caller's `info` / `status` arrays, which the Python layer maps onto the
 * reference exceptions (SingularOperatorError, ConvergenceError).
 */
#ifndef MFB_H
#define MFB_H

#ifdef __cplusplus
extern "C" {
#endif

/* shape limits the host checks before launching (interface.py) */
#define MFB_MOMENTS_MAX_NDOF 64   /* mortar dofs per subdomain in mfb_group_stats/fields */
#define MFB_KL_MAX_TERM 64        /* KL terms per region in mfb_kl_realize*[_batched] */

#define MFB_OK 0
#define MFB_ERR_ARG 1
#define MFB_ERR_LAUNCH 2
#define MFB_ERR_SMEM 3

/* term kinds of a parametrised matrix / rhs entry */
#define MFB_TERM_CONST 0      /* c                */
#define MFB_TERM_INV_K 1      /* c / K[k]         */
#define MFB_TERM_INV_SQRT_K 2 /* c / sqrt(K[k])   */

/* CG per-point status */
#define MFB_CG_CONVERGED 0
#define MFB_CG_NOT_SPD 1      /* p.Sp <= 0  (interface.py:123-126) */
#define MFB_CG_MAX_ITER 2     /* budget exhausted (interface.py:137-139) */
#define MFB_CG_ZERO_RHS 3     /* ||g|| = 0, zero iterations (interface.py:111-113) */

/*
 * Structure of one subdomain's linear system (shared by all its local
 * realizations). Interior unknowns 0..n-1 are in banded order (lower/upper
 * half-bandwidths kl, ku); border unknowns n..n+nb-1 (Stokes rigid-body
 * pinning dofs and kernel multipliers) couple densely through E / G.
 * Right-hand sides: ndof mortar columns Q (sparse, CSC) and one bar column.
 * All index/coefficient arrays are device pointers.
 */
typedef struct MfbPattern {
    int n, kl, ku, ldab, nb, ndof, nfield;
    int n_entries;                 /* interior matrix entries          */
    const int *e_row, *e_col;      /* band-order row/col per entry      */
    const int *e_tptr;             /* [n_entries+1] term ranges         */
    const int *t_kind;             /* MFB_TERM_*                        */
    const double *t_c;
    const int *t_k;                /* index into the system's K slice   */
    const double *E;               /* n x nb row-major (constant)       */
    const double *G;               /* nb x nb row-major (constant)      */
    const int *q_ptr, *q_row;      /* CSC of Q: ndof columns, rows < n+nb */
    const double *q_val;
    const double *bar_const;       /* [n+nb] constant bar rhs           */
    int n_bar_rows;                /* parametrised bar rhs rows         */
    const int *b_row, *b_tptr;     /* rows and term ranges              */
    const int *bt_kind;
    const double *bt_c;
    const int *bt_k;
    const double *h_lift;          /* [ndof] bar readout of lifted data */
    const int *p_ptr, *p_col;      /* CSR postprocess: nfield rows      */
    const double *p_val;
    const double *f_lift;          /* [nfield] lifted data in the fields */
} MfbPattern;

/*
 * Hybridised (SPD) Darcy subdomain: unknown edge multipliers 0..n-1 in line
 * order (half-bandwidth w); every cell contributes K_T * Hhat over its
 * (west, east, south, north) edges. Interface edges carry the mortar data
 * through G (gam_*: edge -> mortar dofs; dof_*: the transpose), pressure
 * edges carry p_val. See paper_1802_06263_b200/hybrid.py.
 */
typedef struct MfbHybPattern {
    int n, w, ws, ndof, nfield, n_edges, n_cells, has_src;
    double hx, hy, nu, s2;
    double Hhat[16];
    const int *row_edge, *edge_kind, *edge_idx, *edge_cells, *edge_slot, *edge_noflow;
    const int *cell_edges;
    const int *gam_ptr, *gam_d;
    const double *gam_c;
    const int *dof_ptr, *dof_edge;
    const double *dof_coef;
    const double *p_val, *src_k, *src_c, *cell_f, *cell_q;
    /* assembly term tables (hybrid.py::assembly_tables): window/border row
     * entries (CSR over rows; dest <= w: band offset, else w+1+border col)
     * and the initial border block entries (dest = d1*(ndof+1)+d2); every
     * term is coef*K[cell] (cell >= 0) or coef (cell < 0). */
    int z_n;
    const int *asm_ptr, *asm_row, *asm_dest, *asm_tptr, *asm_cell;
    const double *asm_coef;
    const int *z_dest, *z_tptr, *z_cell;
    const double *z_coef;
    /* the same entries flattened per panel (panel width of the launch): the
     * rows entering the window at panel pi are entries pe_ptr[pi]..
     * pe_ptr[pi+1] of pe_rec (int4 {window offset of the destination, cell
     * of term 0, cell of term 1, terms}) and pe_coef (double2 coefficients) */
    const int *pe_ptr, *pe_rec;
    const double *pe_coef;
} MfbHybPattern;

const char *mfb_version(void);
const char *mfb_strerror(int code);

/* K[l*n_cells + c] = exp(mean[c] + sum_j phi[c*n_term + j] * xi[l*n_term + j]) */
int mfb_kl_realize(const double *phi, const double *mean, int n_cells, int n_term,
                   const double *xi, int n_loc, double *K, void *stream);

/* One KL table of a batched launch: xi holds n_rows + 1 rows of n_term
 * (row 0 = the mean-field point, written at K + dst0; row l >= 1 at K + dst +
 * (l - 1) * ld). All pointers are device pointers. */
typedef struct {
    const double *phi, *mean, *xi;
    long long dst0, dst, ld;
    int n_cells, n_term, n_rows, pad;
} MfbKlTable;

/* Every table in one launch (max_rows = max n_rows, max_cells = max n_cells). */
int mfb_kl_realize_batched(int n_tables, const MfbKlTable *tables, int max_rows,
                           int max_cells, double *K, void *stream);

/* Same with a row stride: K[l*ld + c]. Method S2 writes realization k of a
 * Darcy subdomain into the k-th full-problem K row (problem.permeability(y),
 * problem.py:85-96), so the Stokes BJS terms of realization k read the same
 * row (ld >= n_cells). */
int mfb_kl_realize_ld(const double *phi, const double *mean, int n_cells, int n_term,
                      const double *xi, int n_loc, double *K, long long ld, void *stream);

/*
 * Assemble, factor (banded LU, partial pivoting) and solve every system s
 * in one launch. pats: device array of patterns; sys_pat[s] selects one;
 * the system's K slice is Kbuf + sys_koff[s]; workspace at work +
 * sys_woff[s] holds ldab*n band + n*(nb+ndof+1) doubles; the solution
 * X (n+nb rows x ndof+1 columns, row-major) goes to X + sys_xoff[s].
 * info[s]: 0 ok, j+1 zero pivot at band column j, -1 singular border.
 * threads: 256 or 384 per CTA (panel rows <= 2 x threads); smem_doubles: Pattern.smem_doubles of
 * the widest pattern. group: CTAs per system (>1: cooperative launch of
 * n_sys*group CTAs that split the trailing and rhs columns; `bar` is a
 * device scratch of n_sys counters, zeroed by the call). keep_factors != 0:
 * the panels' pivot positions and multiplier panels are also stored in the
 * workspace for later solves (mfb_systems_apply, Method S1).
 */
int mfb_systems_solve(const MfbPattern *pats, int n_sys, const int *sys_pat,
                      const double *Kbuf, const long long *sys_koff,
                      double *work, const long long *sys_woff,
                      double *X, const long long *sys_xoff, int *info,
                      int threads, int smem_doubles, int group, unsigned int *bar,
                      int keep_factors,
                      void *stream);

/*
 * From X: basis block Bt (column-major ndof x ndof, i.e. Bt[c*ndof+r] =
 * B[r][c] with B = Q^T X_Q), bar jump h = Q^T x_bar + h_lift, field
 * responses M = P X_Q (nfield x ndof row-major) and bar fields
 * Fb = P x_bar + f_lift. Any of the output pointers may be NULL.
 */
int mfb_systems_extract(const MfbPattern *pats, int n_sys, const int *sys_pat,
                        const double *X, const long long *sys_xoff,
                        double *blocks, const long long *sys_boff,
                        double *hbar, const long long *sys_hoff,
                        double *M, const long long *sys_moff,
                        double *Fb, const long long *sys_fboff, void *stream);

/*
 * B <- (B + B^T) / 2 for the basis blocks of n_sys systems (blocks at
 * sys_boff, ndof from the pattern). The flux-basis block of a subdomain is
 * symmetric (the reference's SuperLU blocks are symmetric to
 * 3e-13); a banded LU with partial pivoting leaves ~1e-12 of asymmetry in
 * the Stokes blocks, which costs the unpreconditioned interface CG ~10% more
 * iterations at tol 1e-11 (cfg2: 710 against 641; the reference: 694). The
 * Darcy condensation's blocks are symmetric by construction.
 */
int mfb_blocks_symmetrize(const MfbPattern *pats, int n_sys, const int *sys_pat, double *blocks,
                          const long long *sys_boff, void *stream);

/*
 * Solves with the factors mfb_systems_solve left in the work buffer (Method
 * S1's star solves): item t applies system item_sys[t] to v = V[t*ldv ..]
 * (one coefficient per local mortar dof): x = S^-1 (Q v) (rigid-body kernel
 * projected out like the factorization's own solves) into X[t*ldx ..] (n+nb
 * entries, may be NULL) and the readout Q^T x into R[t*ldr ..] (ndof
 * entries, may be NULL). max_n: max n + nb over the items' systems.
 * item_live (may be NULL): items with item_live[t] == 0 are skipped.
 * item_list (may be NULL): the launch covers items item_list[0..n_items-1]
 * instead of 0..n_items-1 (a size class of systems per launch, so the
 * shared-memory footprint of the short systems is not the longest's).
 */
int mfb_systems_apply(const MfbPattern *pats, int n_items, const int *item_sys,
                      const int *sys_pat, const double *work, const long long *sys_woff,
                      const double *V, long long ldv, double *X, long long ldx, double *R,
                      long long ldr, int max_n, const int *item_live, const int *item_list,
                      void *stream);

/*
 * Method S1's interface CG (cg_solve with direct_apply, interface.py:107-139,
 * 180-194) for n_pts points in lock step. Item of (point pt, subdomain s) =
 * pt*n_sub + s; sides[4d..4d+3] = (i, a_i, j, a_j): mortar dof d is local dof
 * a_i of subdomain i and a_j of j (j < 0: one side). Per point: x, r, p
 * [n_lambda] (x ends as lambda), scal [2] (r.r, ||g||), iters, status
 * (MFB_CG_*; 4 while running). V [items x ldv]: the next apply's input
 * (p restricted to each item's subdomain; x once the point has finished),
 * item_live: 0 once the item's point has finished (mfb_systems_apply skips
 * it), *n_running: points still iterating.
 *   begin: g from the bar readouts hbar[item_hoff[item] + a] (compute_rhs,
 *          interface.py:166-177), x = 0, r = p = g (g_out may be NULL);
 *   step:  Sp from the apply's readouts R[item*ldr + a], then one CG update
 *          (the relative residual of iteration it goes to
 *          res_hist[pt*hist_cap + it-1] while it <= hist_cap).
 */
int mfb_s1_cg_begin(int n_lambda, int n_pts, int n_sub, const int *sides, const double *hbar,
                    const long long *item_hoff, double *x, double *r, double *p, double *scal,
                    int *iters, int *status, double *V, long long ldv, int *item_live,
                    int *n_running, double *g_out, void *stream);
int mfb_s1_cg_step(int n_lambda, int n_pts, int n_sub, const int *sides, const double *R,
                   long long ldr, double tol, int max_iter, double *x, double *r, double *p,
                   double *scal, int *iters, int *status, double *res_hist, int hist_cap,
                   double *V, long long ldv, int *item_live, int *n_running, void *stream);

/*
 * Fields of S1's recovery (recover_fields + postprocess, interface.py:250-260,
 * problem.py:150-158): item t with star solution X[t*ldx ..] (from
 * mfb_systems_apply) writes F[item_foff[t] + f] = Fb[sys_fboff[sys] + f] -
 * (P x)_f for the nfield fields of its system's pattern (x = S^-1 Q v is
 * minus the reference's star solution: Q carries the readout sign).
 */
int mfb_s1_fields(const MfbPattern *pats, int n_items, const int *item_sys, const int *sys_pat,
                  const double *X, long long ldx, const double *Fb, const long long *sys_fboff,
                  double *F, const long long *item_foff, void *stream);

/*
 * Batched interface CG over points k0..k0+n_pts-1 (global indices).
 * Subdomain i: ndof[i] local dofs with global ids dof_map[dof_ptr[i]..],
 * block of point k at blocks + blk_base[i] + loc*ndof[i]^2 and bar jump at
 * hbar + h_base[i] + loc*ndof[i], where loc = local_idx[region[i]*n_real+k]
 * (region[i] < 0: loc = 0). Outputs per point (indexed k-k0): lam
 * [n_lambda], iters, status (MFB_CG_*), rel. residual history res_hist
 * [hist_cap] (entries beyond hist_cap are dropped), g (may be NULL).
 * stage_doubles: sum_i ndof_i^2; when the point's blocks fit (200 KiB of
 * shared memory with the vectors) they are staged per point (0: never).
 * reg_ndof: max_i ndof_i when every ndof_i is a multiple of 4 (else 0):
 * with reg_ndof <= 32 and 2 n_lambda <= 640 every block row lives in one
 * thread's registers for the whole solve and nothing is staged.
 */
int mfb_cg_batched(int n_lambda, int n_sub, const int *ndof, const int *dof_ptr,
                   const int *dof_map, const int *region, const long long *blk_base,
                   const long long *h_base, const int *local_idx, int n_real,
                   const double *blocks, const double *hbar, int k0, int n_pts,
                   double tol, int max_iter, double *lam, int *iters, int *status,
                   double *res_hist, int hist_cap, double *g, long long stage_doubles, int reg_ndof,
                   void *stream);

/*
 * Same contract for interfaces whose per-point blocks exceed shared memory
 * (cfg4): 8 points in flight per CTA over n_cta persistent CTAs, S p on the
 * FP64 tensor cores with the 8 points as the MMA's N dimension, each block
 * read once per iteration for every point using it; points are taken from
 * a work counter (counter: one int of device memory, reset by the call).
 * n_rows = dof_ptr[n_sub]; n_regions: rows of local_idx. tasks[4 * n_tasks]: runs of <= 8 mortar
 * dofs of one interface {first dof, strip offset in the lower subdomain's
 * packed block, same in the upper one, i | (j + 1) << 12 | rows << 24};
 * sides[4 * n_lambda]: per dof {i, row in i, j, row in j} (j = -1: one
 * side). packed: the blocks in strip order (mfb_cg_pack), block of
 * (sid, loc) at pk_base[sid] + loc * pk_size[sid]. scratch:
 * mfb_cg_multi_scratch_doubles(n_lambda, n_cta) doubles (x, r and S p of
 * the points in flight). seg_tab != NULL: residual histories in segments of
 * hist_cap entries, as mfb_cg_cluster's (res_hist = the pool). trec[12 *
 * n_tasks]: per task its run (as tasks[]), per side nd | (region + 1) << 16,
 * dof_ptr, packed strip base (loc 0) and packed block size.
 * chunk_ptr[n_chunks + 1] (device, or NULL): a CTA claims whole chunks of
 * <= 8 consecutive points, [chunk_ptr[c], chunk_ptr[c + 1]), and feeds them
 * to its slots as they free up (the caller orders the points so that a
 * chunk's points share local realizations); NULL: one point per claim.
 * list_cap > 0: S p streamed over per-warp pass lists of list_cap entries in
 * shared memory (a rolling window of A fragments in flight across pass and
 * task boundaries; needs n_rows < 65536, ndof <= 248 and list_cap >= the
 * largest per-warp count of passes + tasks + 1 with 8 passes per Darcy
 * side); 0: the task loop. Dynamic shared memory: mfb_cg_multi_smem(...)
 * + 8 KB of static tables must fit in 227 KB. Strips of the packed pool hold
 * an even number of fragments (zero-padded).
 * dm_tab[n_dm] (device): the dof list as p offsets, d * 8 + ((d & 2) << 1) for
 * mortar dof d (p is kept [dof][slot] with the slot halves of every other
 * dof pair exchanged: conflict-free B operands). list_cap == 0: dm_tab[r]
 * for row r of dof_map (n_dm >= n_rows + 8, zero padding) and packed in
 * layout 0; list_cap > 0: per subdomain its columns padded to a multiple of
 * 8 and pair-interleaved (column 8 k + 4 h + q at 8 k + 2 q + h), the
 * subdomain's offset in trec's dof_ptr fields, and packed in layout 1.
 */
long long mfb_cg_multi_smem(int n_lambda, int n_dm, int list_cap);
long long mfb_cg_multi_scratch_doubles(int n_lambda, int n_cta);
int mfb_cg_multi(int n_lambda, int n_sub, int n_rows, const int *ndof, const int *dof_ptr,
                 const int *dof_map, const int *region, int n_regions,
                 const long long *blk_base, const long long *h_base, const int *local_idx,
                 int n_real, const double *blocks, const double *hbar, int k0, int n_pts,
                 double tol, int max_iter, double *lam, int *iters, int *status,
                 double *res_hist, int hist_cap, double *g, const int *tasks, int n_tasks,
                 const int *sides, const double *packed, const long long *pk_base,
                 const int *pk_size, int n_cta, double *scratch, int *counter, int *seg_tab,
                 int max_segs, long long seg_cap, int *seg_counter, const int *trec,
                 const int *chunk_ptr, int n_chunks, int list_cap, const int *dm_tab,
                 int n_dm, void *stream);

/*
 * Same contract again, on thread-block clusters of C CTAs (C <= 8) holding
 * NP (8 or 16) points in flight per cluster (csrc/mfb_cg_cluster.cu): the
 * subdomains are split into C parts, CTA `rank` applies its part's blocks
 * (packed fragment strips, mfb_cg_pack) and keeps p, S p and r of the mortar
 * dofs it owns on chip; the two dot products are all-gathered over DSMEM.
 * hdr[12 C] / tab: per-rank tables (paper_1802_06263_b200/cgcluster.py:
 * owned dofs, halo peers, tasks, column maps, cut rows); n_own_max,
 * n_used_max, n_cut_max, n_cm_max, n_unit_max, n_strip_max: their largest
 * owned / used / cut row, column-map, unit and strip counts (every rank uses
 * the same shared-memory layout, sized by
 * these); flags bit 0 / bit 1: r / x of the owned rows in shared memory
 * (else in rs / xs: n_clusters * C * n_own_max * NP doubles each); bit 2:
 * S p in ss (same size) instead of shared memory; smem >=
 * mfb_cg_cluster_smem(...) bytes of dynamic shared memory.
 * Residual histories go to a segmented pool: the history of point k, entry
 * i, is hist[seg_tab[k * max_segs + i / seg] * seg + i % seg]; segments are
 * drawn from seg_counter (reset by the call); a segment index >= seg_cap is
 * not stored (seg_tab entry -1) and the final seg_counter says how many
 * segments the sweep needed. max_segs >= ceil(max_iter / seg).
 * mfb_cg_cluster_max_clusters: co-resident clusters for (C, NP, n_own_max,
 * smem) on this device (negative: MFB_ERR_* code).
 */
int mfb_cg_cluster_max_clusters(int C, int NP, int n_own_max, long long smem);
int mfb_debug_cluster(int stop_at);   /* debug: stop the cluster CG at a phase (0: off; 100: phase clocks) */
int mfb_debug_cluster_prof(long long *out, int n);   /* per-CTA phase clocks of the last run */
int mfb_debug_multi(int on, long long *out);   /* multi CG phase clocks: on/off, or read (out) */
int mfb_debug_multi_warps(long long *out, int reset);   /* CTA 0's S p clocks per warp [16] (-DMFB_PHASE_PROF builds) */
long long mfb_cg_cluster_smem(int NP, int n_used_max, int n_own_max, int n_cut_max,
                              int n_cm_max, int n_unit_max, int n_strip_max, int n_regions,
                              int flags);
int mfb_cg_cluster(int n_lambda, int C, int NP, const int *hdr, const int *tab, int n_own_max,
                   int n_used_max, int n_cut_max, int n_cm_max, int n_unit_max,
                   int n_strip_max, int flags, long long smem,
                   const int *ndof, const int *region, int n_regions, const long long *h_base,
                   const int *local_idx, int n_real, const double *hbar, const int *sides,
                   const double *packed, int k0, int n_pts, double tol, int max_iter,
                   double *lam, int *iters, int *status, double *g, double *xs, double *rs,
                   double *ss, int n_clusters, int *counter, double *hist, int seg, long long seg_cap,
                   int *seg_tab, int max_segs, int *seg_counter, void *stream);

/*
 * One interface-operator application out = S p from stored flux-basis blocks
 * (the reference's basis_apply, interface.py:238-247): block of subdomain i
 * column-major at blocks + blk_base[i] (ndof[i]^2), its rows = mortar dofs
 * dof_map[dof_ptr[i]..]; sides[4 n_lambda] per dof {i, row in i, j, row in
 * j} (j = -1: one side); out[d] = 0 + row_i + row_j. rows: dof_ptr[n_sub]
 * doubles of scratch.
 */
int mfb_basis_apply(int n_lambda, int n_sub, const int *ndof, const int *dof_ptr,
                    const int *dof_map, const int *sides, const long long *blk_base,
                    const double *blocks, const double *p, double *rows, double *out,
                    void *stream);

/*
 * Repack the basis pool for mfb_cg_multi: strips[4 * n_strips] = {sid, first
 * row, rows (<= 8), strip offset}; for every local realization l <
 * n_loc[sid] the strip's rows of block (sid, l) (column-major at blk_base[sid]
 * + l * ndof^2) are written as MMA A fragments: fragment t of lane (g, q) =
 * B[row0 + g][4 t + q] at packed[pk_base[sid] + l * pk_size[sid] + offset +
 * 32 t + lane], zero-padded to an even fragment count (layout 0), or with
 * the lane's fragments 2 k, 2 k + 1 adjacent at 64 k + 2 lane (layout 1, the
 * streamed mfb_cg_multi). max_loc = max n_loc.
 */
int mfb_cg_pack(int n_strips, const int *strips, const int *ndof, const int *n_loc,
                int max_loc, const long long *blk_base, const long long *pk_base,
                const int *pk_size, const double *blocks, double *packed, int layout,
                void *stream);

/*
 * Shifted sufficient statistics per group (one subdomain x one local
 * realization): members grp_members[grp_ptr[g]..grp_ptr[g+1]) (increasing
 * k), W = sum w_k, lamstar = lam_{first member}|_i, s = sum w_k d_k,
 * C = sum w_k d_k d_k^T with d_k = lam_k|_i - lamstar.
 */
int mfb_group_stats(int n_groups, const int *grp_sid, const int *grp_ptr,
                    const int *grp_members, const int *ndof, const int *dof_ptr,
                    const int *dof_map, int n_lambda, const double *lam,
                    const double *weights, const long long *grp_voff,
                    const long long *grp_coff, double *W, double *lamstar,
                    double *s, double *C, void *stream);

/* Per group: fstar = Fb - M lamstar, t = -M s, q = diag(M C M^T). */
int mfb_group_fields(int n_groups, const int *grp_sid, const int *ndof,
                     const int *nfield, const double *M, const long long *grp_moff,
                     const double *Fb, const long long *grp_fboff,
                     const long long *grp_voff, const long long *grp_coff,
                     const double *lamstar, const double *s, const double *C,
                     double *fstar, double *t, double *q, void *stream);

/*
 * Per subdomain i, groups gptr[i]..gptr[i+1] in local order: mean =
 * sum_l (W_l fstar_l + t_l); var = sum_l [W_l (fstar_l-m)^2 + 2 (fstar_l-m)
 * t_l + q_l] + m^2 (1 - wtot), unclamped (the host applies the clamp).
 */
int mfb_moments_reduce(int n_sub, const int *gptr, const int *nfield,
                       const long long *grp_fboff, const double *W,
                       const double *fstar, const double *t, const double *q,
                       double wtot, const long long *sid_out_off, double *mean,
                       double *var, void *stream);

/* Streaming s += w*v, q += (w*v)*v in realization order, then m = s,
 * var = q - m*m (unclamped), no FMA contraction (moments.py:34-35, 50). */
int mfb_lambda_moments(int n_lambda, int n_real, const double *lam,
                       const double *weights, double *mean, double *var,
                       double *sumsq, void *stream);

/*
 * Darcy flux basis by static condensation of the SPD hybridised system in
 * shared memory (band Cholesky, panel width `panel` = 8, trailing
 * updates on DMMA): per system B (column-major into blocks + sys_boff) and
 * the bar jump h. If Lstore != NULL the factor panels are kept for
 * mfb_darcy_backsolve (layout: per panel m*(panel+4) L doubles then
 * panel*Cp rhs doubles, m = w + panel, Cp = ndof+1 rounded up to 8).
 * info[s] = -(pivot index + 1) if a pivot is not positive. smem_bytes:
 * 8 * (m*ws + m*Cp + Cp*Cp + m*(panel+4) + panel*Cp) for the widest pattern.
 */
int mfb_darcy_condense(const MfbHybPattern *pats, int n_sys, const int *sys_pat,
                       const double *Kbuf, const long long *sys_koff, double *blocks,
                       const long long *sys_boff, double *hbar, const long long *sys_hoff,
                       double *Lstore, const long long *sys_loff, int *info, int panel,
                       int smem_bytes, void *stream);

/* X = H_II^-1 [V | v_b] (n x Cp, row-major) from the stored factor panels;
 * smem_bytes = 8 * (m*Cp + m*(panel+4) + panel*Cp). */
int mfb_darcy_backsolve(const MfbHybPattern *pats, int n_sys, const int *sys_pat,
                        const double *Lstore, const long long *sys_loff, double *X,
                        const long long *sys_xoff, int panel, int smem_bytes, void *stream);

/* Cell-local recovery of the fields: M (nfield x ndof, fields = Fb - M lam)
 * and Fb, in the layout u(edges) | p(cells) | cv(cells x 2) | cp(cells). */
int mfb_darcy_recover(const MfbHybPattern *pats, int n_sys, const int *sys_pat,
                      const double *Kbuf, const long long *sys_koff, const double *X,
                      const long long *sys_xoff, double *M, const long long *sys_moff,
                      double *Fb, const long long *sys_fboff, void *stream);

/* Self test of the FP64 tensor-core (DMMA m8n8k4) fragment layout the
 * elimination kernels rely on; writes max |error| to *err (device). */
int mfb_selftest_dmma(double *err, void *stream);

/* Phase cycle counters of the condense kernel (builds with -DMFB_PROFILE
 * only; returns 1 otherwise). Host pointer, 16 counters. */
int mfb_debug_prof(unsigned long long *out);
/* Same for the banded LU kernel (24 counters; -DMFB_PROFILE builds only). */
int mfb_debug_bprof(unsigned long long *out);
/* -DMFB_PROFILE builds: CG phase cycles of CTA 0 (8 counters). */
int mfb_debug_cgprof(unsigned long long *out);
/* -DMFB_PROFILE builds: per-panel timeline of system 0 (4 x 4096 globaltimer ns). */
int mfb_debug_timeline(unsigned long long *out);

#ifdef __cplusplus
}
#endif
#endif /* MFB_H */
