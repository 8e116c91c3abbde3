/*
 * pbsafe.h — C-ABI of the B200-native p-BiCGSafe hot path (libpbsafe.so).
 *
 * Plain pointers and sizes only; no torch types.  Every entry point returns an
 * int status (PBS_OK or a negative PBS_ERR_*); the solver's own outcome
 * (converged / max_iters / breakdown / non_finite) travels in pbs_result.
 * A context is bound to one CUDA device and is not thread-safe: one host
 * thread drives it (the reference's "one control thread per solve",
 * SPEC.md:304).  Host pointers are borrowed for the duration of a call;
 * device copies are owned by the context.
 *
 * Reference interfaces each group replaces (paths under
 * /root/reference/pkg/src/pipesafe/):
 *   pbs_solve / pbs_solve_dev  — solve(), solve_pbicgsafe(),
 *                                solve_pbicgsafe_rr(), solve_ssbicgsafe2(),
 *                                solve_bicgstab(), solve_gpbicg()
 *                                (solvers.py:791-803, 742-779, 485-592,
 *                                210-327, 330-460), plus the paper's
 *                                p-BiCGStab comparator (not in
 *                                the reference — PBS_METHOD_PBICGSTAB), with
 *                                SolverConfig fields (solvers.py:51-78) in
 *                                pbs_config and SolveOutcome / IterationRecord
 *                                (solvers.py:81-114) in pbs_result + history
 *   pbs_csr_upload             — CsrMatrix (linalg.py:27-71) moved to HBM
 *   pbs_stencil_create         — matrix-free operator for the generated grids
 *                                (linalg.py:175-209 gen_poisson and the
 *                                BASELINE configs' stencils)
 *   pbs_spmv_dev               — linalg.spmv (linalg.py:149-161) incl. the
 *                                check_finite scan (linalg.py:142-146)
 *   pbs_k_*                    — the kernel backend table kernels._TABLES
 *                                (kernels.py:140-174): spmv_range, dot_range,
 *                                lincomb2/3/4, lincomb_nested, add_scaled_diff,
 *                                add_scaled_damped_diff (kernels.py:95-137)
 *   pbs_dot_batch_dev          — ReductionEngine.submit_batch over a DotBatch
 *                                (reduction.py:344-382), labels a..h,r
 *   pbs_step_dev               — one iteration of _solve_pipelined
 *                                (solvers.py:639-734) from a given state: the
 *                                single-iteration parity seam
 */
#ifndef PBSAFE_H_
#define PBSAFE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes */
#define PBS_OK 0
#define PBS_ERR_INVALID -1   /* ValueError in the reference */
#define PBS_ERR_CUDA -2      /* CUDA runtime failure (message in pbs_last_error) */
#define PBS_ERR_NONFINITE -3 /* NonFiniteVectorError: see pbs_result.nonfinite_* */
#define PBS_ERR_NOMEM -4
#define PBS_ERR_NCCL -5
#define PBS_ERR_UNSUPPORTED -6

/* methods (solvers.py:782-788) */
#define PBS_METHOD_PBICGSAFE 0
#define PBS_METHOD_PBICGSAFE_RR 1
#define PBS_METHOD_SSBICGSAFE2 2
#define PBS_METHOD_BICGSTAB 3  /* two reduction phases (solvers.py:210-327) */
#define PBS_METHOD_GPBICG 4    /* three reduction phases (solvers.py:330-460) */
#define PBS_METHOD_PBICGSTAB 5 /* pipelined BiCGStab (Cools & Vanroose; not in the reference,
                                  restated in oracle/pbsafe_oracle.c solve_pstab) */

/* SolveStatus (solvers.py:44-48) */
#define PBS_CONVERGED 0
#define PBS_MAX_ITERS 1
#define PBS_BREAKDOWN 2
#define PBS_NON_FINITE 3

/* BreakdownError quantities (coefficients.py:77, 80, 83, 102, 105) */
#define PBS_BD_NONE 0
#define PBS_BD_INITIAL_ALPHA 1 /* "initial alpha denominator (r0*, s)" */
#define PBS_BD_BETA 2          /* "beta denominator zeta_prev * f_prev" */
#define PBS_BD_ALPHA 3         /* "alpha denominator g + beta*h" */
#define PBS_BD_ZETA 4          /* "zeta denominator (s, s)" */
#define PBS_BD_ZETA_ETA 5      /* "zeta/eta denominator a*b - c^2" */
/* product-type comparators (solvers.py:275, 283, 302-303, 434; coefficients.py:130, 134) */
#define PBS_BD_PROD_ALPHA 6    /* "alpha denominator (r0*, Ap)" */
#define PBS_BD_STAB_OMEGA 7    /* "omega denominator (At, At)" */
#define PBS_BD_STAB_BETA 8     /* "beta denominator omega" */
#define PBS_BD_BETA_F 9        /* "beta denominator (r0*, r)" */
#define PBS_BD_GP_ZETA 10      /* "zeta denominator (At, At)" */
#define PBS_BD_GP_ZETA_ETA 11  /* "zeta/eta denominator e*a - d^2" */
#define PBS_BD_GP_BETA 12      /* "beta denominator zeta" */
#define PBS_BD_PSTAB_ALPHA 13  /* "alpha denominator (r0*, w) + beta*((r0*, s) - omega*(r0*, z))" */
#define PBS_BD_PSTAB_OMEGA 14  /* "omega denominator (y, y)" */

/* SpMV tags of NonFiniteVectorError messages (reduction.py:330, 451) */
#define PBS_TAG_AX 1
#define PBS_TAG_AR 2
#define PBS_TAG_AS 3
#define PBS_TAG_AW 4
#define PBS_TAG_AO 5
#define PBS_TAG_AU 6
#define PBS_TAG_AT 7
#define PBS_TAG_AY 8
#define PBS_TAG_AP 9
#define PBS_TAG_AZ 10 /* p-BiCGStab v = A z */

/* reduction orders for the per-iteration dot batch */
#define PBS_REDUCE_TREE 0 /* fixed-shape block tree: deterministic, full speed */
#define PBS_REDUCE_PLAN 1 /* PartitionPlan.balanced(n, plan_workers) chains +
                             left-to-right combine (reduction.py:282-294):
                             bitwise equal to the reference; small n only */

/* history flag bits */
#define PBS_HIST_REPLACED 1
#define PBS_HIST_HAS_COEF 2

typedef struct pbs_ctx pbs_ctx;
typedef struct pbs_mat pbs_mat;

/* trace_hook (solvers.py:725-732): called after each completed iteration with
 * host arrays (valid for the call only): 13 for the Safe methods,
 * x r p u o t w y z s q g l; BiCGStab 6, x r p t Ap At (solvers.py:315);
 * GPBi-CG 8, x r p u t w y z (solvers.py:448).
 * Tracing syncs the device every iteration; it is a parity/debug mode. */
typedef void (*pbs_trace_fn)(int64_t iter, double* const* host_vecs, void* user);

typedef struct {
  double tol;            /* SolverConfig.tol */
  int64_t max_iters;     /* SolverConfig.max_iters */
  int64_t rr_epoch;      /* SolverConfig.rr_epoch (m) */
  int64_t rr_cutoff;     /* SolverConfig.rr_cutoff; < 0 means max_iters */
  int32_t record_history;
  int32_t reduce_mode;   /* PBS_REDUCE_* */
  int32_t plan_workers;  /* ranges for PBS_REDUCE_PLAN */
  int32_t use_graphs;    /* capture iterations into CUDA graphs */
  int32_t timing;        /* per-kernel CUDA-event timing (no graphs) */
  int32_t pad;
  pbs_trace_fn trace_fn; /* NULL: no tracing */
  void* trace_user;
  /* schedule evidence (multi-GPU schedule, timing mode): records of
   * (iter, kind, tag, t_ms) as 4 doubles, kind 0 reduce_start 1 reduce_end
   * 2 spmv_start 3 spmv_end 4 coeff_ready, tag = PBS_TAG_* (spmv) or 0;
   * t_ms from the solve's first event.  NULL: off. */
  double* events_out;
  int64_t events_cap;
  int64_t* events_count;
  /* multi-GPU schedule evidence from the device clock (%globaltimer): per
   * partition and iteration i < stamps_cap, 8 doubles in ns from the solve's
   * first stamp (-1: absent): As start/end, Aw start/end, publish of check i
   * start/end, finalize of check i start/end.  NULL: off. */
  double* stamps_out;
  int64_t stamps_cap;
  int64_t* stamps_count;
} pbs_config;

#define PBS_NUM_KERNEL_KINDS 8 /* K1 As, K2 update, K3 Aw+epilogue, F finalize,
                                  R rr elementwise, RS rr SpMV, S setup, D dots */

typedef struct {
  int32_t status;           /* PBS_CONVERGED ... */
  int32_t breakdown;        /* PBS_BD_* */
  int64_t iterations;
  int64_t failure_iter;     /* -1: None */
  int64_t n_records;        /* history length */
  double r0_norm;
  int32_t nonfinite_tag;    /* != 0 when PBS_ERR_NONFINITE was returned */
  int32_t pad;
  int64_t nonfinite_index;  /* first non-finite row of that SpMV output */
  int64_t n_spmv;           /* SpMVs executed (reference counting) */
  int64_t n_replacements;   /* residual-replacement iterations executed */
  int32_t stop_stage;       /* product-type methods: where the stopping
                               iteration ended (0 loop-top check, 1 after the
                               alpha step, 2 omega/zeta, 3 after the x/r
                               update, 4 complete) */
  int32_t pad2;
  double device_ms;         /* CUDA-event time from setup to the last check */
  int64_t kernel_launches;  /* kernels launched by this solve */
  double kernel_ms[PBS_NUM_KERNEL_KINDS];    /* timing mode: summed durations */
  int64_t kernel_count[PBS_NUM_KERNEL_KINDS];
} pbs_result;

/* ---- context ---------------------------------------------------------- */
int pbs_init(int device, pbs_ctx** ctx);
int pbs_destroy(pbs_ctx* ctx);
const char* pbs_last_error(pbs_ctx* ctx); /* ctx may be NULL (global error) */
int pbs_device_info(pbs_ctx* ctx, int* sm_count, int* cc_major, int* cc_minor);
/* bind the context's work to an external stream (e.g. torch's current
 * stream); 0 restores the context's own stream */
int pbs_set_stream(pbs_ctx* ctx, uintptr_t stream);

/* ---- operators ---------------------------------------------------------- */
/* CSR: row_ptr int64[n_rows+1]; col_idx int64 or int32 (col_bytes 8/4);
 * values f64[nnz].  Validated cheaply (sizes, endpoints); column indices
 * must fit int32 on the device. */
int pbs_csr_upload(pbs_ctx* ctx, int64_t n_rows, int64_t n_cols, int64_t nnz,
                   const int64_t* row_ptr, const void* col_idx, int32_t col_bytes,
                   const double* values, pbs_mat** mat);
/* constant-coefficient stencil on a k^dim grid, C order (last axis fastest);
 * offsets int32[npts*dim] ((dz,)dy,dx per point) sorted by flattened offset,
 * coeffs f64[npts].  npts <= 27. */
/* upload new arrays of the same shape (n_rows, nnz) into an existing CSR
 * operator (e.g. a resident partition slab): its workspace and halo plan
 * stay */
int pbs_csr_update(pbs_mat* mat, const int64_t* row_ptr, const void* col_idx, int32_t col_bytes,
                   const double* values);
int pbs_stencil_create(pbs_ctx* ctx, int32_t dim, int64_t k, int32_t npts,
                       const int32_t* offsets, const double* coeffs, pbs_mat** mat);
/* CSR of a stencil operator built on the device (rows in C order, columns
 * ascending, out-of-grid neighbours dropped) — the same arrays as
 * problems.stencil_csr builds on the host, without the host round trip
 * (config 4's 1.5e9 nonzeros). */
int pbs_stencil_to_csr(pbs_mat* stencil, pbs_mat** csr);
int pbs_mat_free(pbs_mat* mat);
int pbs_mat_info(pbs_mat* mat, int64_t* n_rows, int64_t* n_cols, int64_t* nnz,
                 int32_t* is_stencil);
/* The device layout the SpMV engines stream for this operator (there is no
 * counterpart in the reference: linalg.py:28-48 keeps the three CSR arrays;
 * this is what bench.py's byte accounting and the layout tests read).
 * out[0] layout: 0 CSR order, int32 col_idx, x gathered; 1 CSR order, u16
 *        window-local columns; 2 CSR order, band mode; 3 sliced ELL, f64
 *        values; 4 sliced ELL, u8 dictionary values; 5 sliced ELL, u8 (value,
 *        relative column) pair dictionary; 10 matrix-free stencil
 * out[1] entries streamed per product (nonzeros + padding)
 * out[2] bytes per entry (value + column)
 * out[3] bytes per row besides (8: int64 row_ptr; 1: u8 row length)
 * out[4] dictionary entries in use (layouts 4, 5)
 * out[5] longest row of a 256-row block (layouts 3, 4, 5)
 * out[6] x windows per row block, out[7] staged x elements per row block */
int pbs_mat_layout(pbs_mat* mat, int64_t out[8]);

/* y = A x with device pointers; reports the first non-finite row (check_finite)
 * through *nonfinite_index (-1 when all finite). */
int pbs_spmv_dev(pbs_mat* mat, const double* d_x, double* d_y, int64_t* nonfinite_index);

/* ---- solver ------------------------------------------------------------ */
/* Host buffers (the e2e drop-in): b, x0 (NULL = zeros) -> x_out;
 * hist_rel f64[max_iters+1], hist_flags u8[max_iters+1] (PBS_HIST_* bits),
 * hist_coef f64[4*(max_iters+1)] (alpha beta zeta eta); any may be NULL. */
int pbs_solve(pbs_mat* mat, int32_t method, const double* b, const double* x0,
              const pbs_config* cfg, double* x_out, double* hist_rel, uint8_t* hist_flags,
              double* hist_coef, pbs_result* result);
/* Device-resident inputs/outputs (HBM-resident timing); history to host. */
int pbs_solve_dev(pbs_mat* mat, int32_t method, const double* d_b, const double* d_x0,
                  const pbs_config* cfg, double* d_x_out, double* hist_rel,
                  uint8_t* hist_flags, double* hist_coef, pbs_result* result);

/* One p-BiCGSafe iteration from an explicit state (single-step parity seam).
 * d_state: 16 device vectors of n doubles, in this order:
 *   x r p u o t w y z s q g l r0s b As
 * updated in place to the state after the iteration (o, q, As filled);
 * scalars f64[6] in: iter, alpha_prev, zeta_prev, f_prev, r0_norm, replace;
 * out f64[14]: alpha beta zeta eta + the 9 dots (a..h,r) + status(-1=ran). */
int pbs_step_dev(pbs_mat* mat, double* const* d_state, const double* scalars_in,
                 int32_t reduce_mode, int32_t plan_workers, double* scalars_out);

/* ---- kernel backend table (host pointers; parity seam) ------------------ */
int pbs_k_spmv_range(pbs_ctx* ctx, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                     const int64_t* col_idx, const double* values, const double* x,
                     double* out, int64_t lo, int64_t hi);
int pbs_k_dot_range(pbs_ctx* ctx, const double* x, const double* y, int64_t lo, int64_t hi,
                    double* result);
/* kind: 2 lincomb2, 3 lincomb3, 4 lincomb4, 5 lincomb_nested,
 *       6 add_scaled_diff (base=a; s=sc[0]; a=b; b=c),
 *       7 add_scaled_damped_diff (base=a; s=sc[0]; a=b; w=sc[1]; b=c) */
int pbs_k_lincomb(pbs_ctx* ctx, int32_t kind, int64_t n, double* out, const double* sc,
                  const double* a, const double* b, const double* c, const double* d);

/* ---- multi-GPU row partition (one process per GPU) --------------------- */
/* The row-partitioned path of SURVEY §8(e): each rank owns rows [lo, hi) of
 * PartitionPlan.balanced(n, nranks) (reduction.py:55-87).  Its local CSR is
 * uploaded with pbs_csr_upload using columns remapped to the extended space
 * [left halo (hl) | own (hi-lo) | right halo (hr)]; pbs_mat_set_partition
 * attaches the halo transfer plan.  Solves on a partitioned operator take
 * and return the rank's own segments of b / x0 / x; the history, status and
 * iteration count are identical on every rank.  NCCL is loaded at run time
 * (libnccl.so.2, e.g. the copy torch already loaded). */
typedef struct pbs_dist pbs_dist;
#define PBS_TRANSPORT_P2P 0  /* halos: copy-engine pushes into IPC-mapped peer
                                memory + stream-memory-op flags; reduction:
                                peer stores of each rank's record + flags */
#define PBS_TRANSPORT_NCCL 1 /* ncclSend/Recv halos, ncclAllGather of the records */
#define PBS_DIST_BLOB_BYTES 256
int pbs_nccl_unique_id(void* out128);
/* a partition's link to its group of nranks (at most 64).  The NCCL
 * transport needs two unique ids (halo exchange and the record all-gather run
 * on different streams, so they must not share a communicator); P2P ignores
 * them (NULL). */
int pbs_dist_init(pbs_ctx* ctx, int32_t nranks, int32_t rank, int32_t transport, const void* id_halo128,
                  const void* id_reduce128, pbs_dist** dist);
int pbs_dist_destroy(pbs_dist* dist);
/* SMs this partition's kernels may fill (0: all): a loopback group of N on
 * one device gives each partition sms / N, like N smaller GPUs */
int pbs_dist_set_sm_limit(pbs_dist* dist, int32_t sms);
/* sends: nsend quadruples (peer, offset within the own segment, length,
 * extended-space offset on the peer); recvs: nrecv triples (peer,
 * extended-space offset, length).  Allocates the partition's workspace. */
int pbs_mat_set_partition(pbs_mat* mat, pbs_dist* dist, int64_t n_global, int64_t row_lo, int64_t hl,
                          int64_t hr, int32_t nsend, const int64_t* sends, int32_t nrecv,
                          const int64_t* recvs);
/* one process per GPU: export this partition (PBS_DIST_BLOB_BYTES: IPC
 * handles of its workspace and mailbox), gather every rank's blob (rank
 * order), connect (maps the peers), then barrier before the first solve */
int pbs_dist_export(pbs_mat* mat, void* blob_out);
int pbs_dist_connect(pbs_mat* mat, const void* blobs);
/* loopback group: partitions 0..n-1 of one system held by this process on
 * one device, linked directly (the same schedule, kernels and transport) */
int pbs_dist_connect_local(pbs_mat** mats, int32_t n);
/* solve on a loopback group: per-partition device pointers to the own
 * segments of b, x0 (NULL: zero) and x; history and result as pbs_solve.
 * (One process per GPU: pbs_solve / pbs_solve_dev on its partition.) */
int pbs_solve_group(pbs_mat** mats, int32_t n, int32_t method, const double* const* d_b,
                    const double* const* d_x0, const pbs_config* cfg, double* const* d_x, double* hist_rel,
                    uint8_t* hist_flags, double* hist_coef, pbs_result* result);
/* partitioned SpMV y = A x (own segments; halos exchanged by the group's
 * transport); nonfinite_index[p]: first non-finite local row or -1 */
int pbs_spmv_group(pbs_mat** mats, int32_t n, const double* const* d_x, double* const* d_y,
                   int64_t* nonfinite_index);
/* rows [row_lo, row_hi) of a whole-grid stencil operator as a partition slab:
 * SpMV inputs in the extended space [pad | hl | own | hr] (like a CSR slab);
 * pbs_stencil_to_csr of a slab gives its CSR with extended-space columns */
int pbs_stencil_slab(pbs_mat* stencil, int64_t row_lo, int64_t row_hi, int64_t hl, int64_t hr, pbs_mat** slab);

/* ---- device batch reduction --------------------------------------------- */
/* 9 dots of the safe batch over device vectors s y r r0s t, packed a..h,r */
int pbs_dot_batch_dev(pbs_ctx* ctx, int64_t n, const double* d_s, const double* d_y,
                      const double* d_r, const double* d_r0s, const double* d_t,
                      int32_t reduce_mode, int32_t plan_workers, double* out9);

#ifdef __cplusplus
}
#endif
#endif /* PBSAFE_H_ */
