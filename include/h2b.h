/*
 * h2b.h — C ABI of the B200-native H² boundary-operator matvec (libh2b.so).
 *
 * This is the drop-in boundary for the reference's H² application path:
 *
 *   strayfield.hmatrix.h2.h2_matvec(op: H2Matrix, x) -> y
 *       /root/reference/pkg/src/strayfield/hmatrix/h2.py:186-244
 *   H2Matrix.matvec(self, x)                       h2.py:74-75
 *   H2Matrix.storage_bytes(self)                   h2.py:77-83
 *   BoundaryOperator.apply / apply_operator        bem.py:255-256, 277-284
 *
 * The reference is pure Python and has no FFI of its own; these entry points
 * are what its ctypes layer binds.  Every argument is a
 * plain pointer or integer — no torch, no numpy, no C++ types.
 *
 * Conventions
 *  - All matrices are C-contiguous little-endian float64, exactly as the
 *    reference stores them in H2Matrix (h2.py:35-42):
 *      row_basis[c]     V_c  (|c| x k_row(c))   for leaf clusters
 *      col_basis[c]     W_c  (|c| x k_col(c))   for leaf clusters
 *      row_transfer[c]  E_c  (k_row(c) x k_row(parent(c)))   keyed by child c
 *      col_transfer[c]  F_c  (k_col(c) x k_col(parent(c)))   keyed by child c
 *      coupling b       S_b  (k_row(t) x k_col(s))
 *      near b           N_b  (|t| x |s|)   (includes D = Psi/4pi - 1 on the
 *                                          diagonal blocks, bem.py:232-234)
 *  - Cluster ids are the reference's preorder ids (cluster.py:385-393).
 *  - x / y are in ORIGINAL node order; perm maps tree position -> node
 *    (cluster.py:42-59).  Multi-RHS vectors are node-major (n x nrhs).
 *  - Return codes: 0 ok, H2B_EINVAL invalid argument (message in
 *    h2b_last_error()), H2B_ECUDA CUDA error, H2B_ENCCL NCCL error,
 *    H2B_ENOMEM host allocation failure, H2B_ENODEV no CUDA device.
 *  - h2b_last_error() is thread-local.
 */
#ifndef H2B_H_
#define H2B_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define H2B_ABI_VERSION 4

#define H2B_OK 0
#define H2B_EINVAL (-1)
#define H2B_ECUDA (-2)
#define H2B_ENCCL (-3)
#define H2B_ENOMEM (-4)
#define H2B_ENODEV (-5)
#define H2B_EIO (-6)     /* corrupt or incompatible operator file (OperatorIOError) */
#define H2B_ECONV (-7)   /* solver breakdown (ConvergenceError, errors.py) */

/* One H2Matrix, as the reference holds it (h2.py:23-42, cluster.py:13-59).
 * Host arrays; they are only read during h2b_create / h2b_plan_create and may
 * be freed afterwards. */
typedef struct h2b_desc {
  int64_t n;                    /* H2Matrix.n == len(tree.perm)             */
  int64_t nclusters;            /* len(tree.clusters), preorder             */
  const int64_t* perm;          /* [n] tree.perm                            */
  const int64_t* cl_start;      /* [nclusters] Cluster.start                */
  const int64_t* cl_end;        /* [nclusters] Cluster.end                  */
  const int64_t* cl_child;      /* [2*nclusters] children cids, -1 = none   */
  const int64_t* k_row;         /* [nclusters] H2Matrix.row_rank(c)         */
  const int64_t* k_col;         /* [nclusters] H2Matrix.col_rank(c)         */
  const double* const* row_basis;    /* [nclusters] leaf V_c, NULL otherwise */
  const double* const* col_basis;    /* [nclusters] leaf W_c, NULL otherwise */
  const double* const* row_transfer; /* [nclusters] E_c for non-root c        */
  const double* const* col_transfer; /* [nclusters] F_c for non-root c        */
  int64_t ncoupling;            /* len(H2Matrix.coupling)                   */
  const int64_t* cp_row;        /* [ncoupling] row cid                      */
  const int64_t* cp_col;        /* [ncoupling] col cid                      */
  const double* const* cp_data; /* [ncoupling] S_b                          */
  int64_t nnear;                /* len(H2Matrix.near)                       */
  const int64_t* nr_row;        /* [nnear] row cid                          */
  const int64_t* nr_col;        /* [nnear] col cid                          */
  const double* const* nr_data; /* [nnear] N_b                              */
} h2b_desc;

/* sched_flags bit 3: take the flags literally.  Without it, an operator
   whose near-field and coupling bytes per rank are at least
   H2B_STREAM_DEFAULT_BYTES gets the streaming defaults for the fields left
   zero: every warp a ring warp with 4 KB stages, 6 near-priority warps,
   leaf mix 4, 8 KB far-field and 256 KB near-field pieces, evict-first
   ring copies; smaller operators,
   whose time is the far-field chain's latency, keep plain scheduling. */
#define H2B_SCHED_EXPLICIT 8
/* sched_flags bit 1 (planning): the final items (y rows) go to the slack
   queue instead of the chain queue, so leaves whose last dependency lands
   together do not pull every warp off the near-field stream at once */
#define H2B_SCHED_FINAL_SLACK 2
/* sched_flags bit 2: arrival counts by release-only atomics; only a warp
   that completes a successor acquires (fence), instead of every arrival
   being an acquire (which invalidates the SM's L1) */
#define H2B_SCHED_RELEASE_ARRIVALS 4
#define H2B_STREAM_DEFAULT_BYTES (1LL << 30)
/* Below this many near-field and coupling bytes per rank the plan uses the
   level-skipping chain by default (plan_flags H2B_PLAN_NO_SKIP: off), and
   plain scheduling (below H2B_STREAM_DEFAULT_BYTES) gets leaf mix 2. */
#define H2B_SKIP_DEFAULT_BYTES (4LL << 30)
/* sched_flags: run the near item a warp claimed ahead before the coupling
   rows of inner clusters (default: inner coupling rows first). */
#define H2B_SCHED_NEAR_FIRST 1
/* sched_flags bits 4-7: single-vector products give the top k warps of each
   CTA a two-stage 8 KB TMA ring for streamed items (16 KB in flight each, no
   registers); 0: register streaming only */
#define H2B_SCHED_RING_WARPS(k) (((k) & 0xf) << 4)
/* sched_flags bits 18-19: single-vector ring stage payload: 0 -> 8 KB,
   1 -> 6 KB, 2 -> 4 KB (smaller stages fit more ring warps per CTA) */
#define H2B_SCHED_RING_STAGE(s) (((s) & 3) << 18)
/* sched_flags bits 8-15: warps per CTA that take near-field items (0: all) */
#define H2B_SCHED_NEAR_WARPS(k) (((k) & 0xff) << 8)
/* sched_flags bits 16-17: columns in flight per lane of a streamed item:
   0 -> 8 (default), 2 -> 4 */
#define H2B_SCHED_STREAM(s) (((s) & 3) << 16)
/* sched_flags bits 20-23: serve the leaf coupling rows before the near item
   a warp claimed ahead once it has run m near items in a row (15: always;
   0: after it, the round-1 behaviour) */
#define H2B_SCHED_LEAF_MIX(m) (((m) & 0xf) << 20)
/* sched_flags bit 24: multi-RHS items stream through registers instead of
   the per-warp TMA ring (A/B switch) */
#define H2B_SCHED_NO_RING (1 << 24)
/* sched_flags bit 25: TMA-ring copies carry an L2 evict-first hint (the
   streamed matrix is read once; the gathered sources should stay in L2) */
#define H2B_SCHED_STREAM_EVICT_FIRST (1 << 25)
/* sched_flags bit 30: near-priority warps take no chain-queue items (only
   continuations): the leaf-level downward items, which become ready
   together, then do not pull every warp off the near-field stream */
#define H2B_SCHED_PRIO_NO_CHAIN (1 << 30)
/* sched_flags bit 31: the near-priority warps' mix (H2B_SCHED_LEAF_MIX)
   serves the coupling rows of inner clusters (they gate the downward chain)
   before the leaf coupling rows */
#define H2B_SCHED_MIX_INNER ((int)(1u << 31))
/* sched_flags bits 26-29: the top k warps of each CTA take near-field items
   before the up-leaf items and the coupling queues (0: none) */
#define H2B_SCHED_NEAR_PRIO(k) (((k) & 0xf) << 26)

/* Execution-plan knobs.  Zero-initialise for defaults. */
typedef struct h2b_options {
  int64_t task_bytes;   /* max bytes per near-field work item (def. 65536)   */
  int64_t far_task_bytes; /* max bytes per far-field item (default 4096): each
                             is staged to shared memory by one TMA bulk copy */
  int32_t warps_per_cta;/* persistent CTA width in warps (default 8, <= 8)   */
  int32_t ctas_per_sm;  /* 0 = occupancy-derived                             */
  int32_t max_nrhs;     /* largest nrhs the op will be called with (def. 16) */
  int32_t sched_flags;  /* H2B_SCHED_* bits; 0 = default scheduling          */
  int32_t band_depth;   /* plans only (h2b_plan_create): group D tree levels
                           of the far-field chain into fused runs; 0/1 = none.
                           h2b_create rejects D > 1 (measured slower)       */
  /* Multi-GPU (one process per GPU).  world_size <= 1: whole operator. */
  int32_t rank;
  int32_t world_size;
  const void* nccl_unique_id; /* 128-byte ncclUniqueId shared by all ranks  */
  int32_t near_phase0_pct; /* multi-GPU: share (percent of bytes, 1-100) of
                              the rank's near field run in phase 0, beside the
                              latency-bound upward pass; 0 = default (90),
                              -1 = none (all in phase 1)                    */
  int32_t plan_flags;   /* H2B_PLAN_* bits; 0 = defaults                      */
} h2b_options;

/* plan_flags: the level-skipping far-field chain: upward
   coefficients of even-height clusters from their grandchildren through
   transfer products, downward coefficients of every other level from the
   grandparent -- half the dependency links, one extra product matrix per
   skipped link (h2b_stats.extra_bytes).  SKIP forces it on, NO_SKIP off. */
#define H2B_PLAN_SKIP_LEVELS 1
#define H2B_PLAN_NO_SKIP 2
/* plan_flags (h2b_plan_create only): also plan the split multi-RHS product
   (the near field alone, then the rest), exposed as phases 1 and 2 of a
   single-GPU plan; h2b_create plans it whenever max_nrhs >= 8. */
#define H2B_PLAN_NEAR_SPLIT 4
/* plan_flags bits 4-7 (v > 0): leaf coupling rows cut into pieces of at
   most 1 KB << v (default: task_bytes, the near-field piece size) */
#define H2B_PLAN_COUPLING_PIECE(v) (((v) & 0xf) << 4)
/* plan_flags bit 8: coupling rows whose inputs are all upward coefficients
   drop their per-source dependencies and are released together once every
   upward item has finished (one counter instead of one arrival per edge);
   bit 9 forces it off */
#define H2B_PLAN_GATE (1 << 8)
#define H2B_PLAN_NO_GATE (1 << 9)
/* plan_flags bit 10: the staged product.  The clusters of at
   most H2B_PLAN_SWEEP_NODES nodes root "bottom subtrees"; their upward items
   run first in a sweep kernel (one CTA per subtree, block barriers between
   tree levels, no arrival counters), one dataflow launch then runs the near
   field, every coupling row and the short far-field chain of the clusters
   above the subtrees, and a second sweep runs the subtrees' downward
   transfers and the finals.  Bit 11 forces it off. */
#define H2B_PLAN_STAGED (1 << 10)
#define H2B_PLAN_NO_STAGED (1 << 11)
/* plan_flags bits 12-15 (v > 0): bottom subtrees hold at most 64 << v nodes
   (default: the power of two giving about 256 subtrees per rank, between 128
   and 16384 nodes; multi-GPU plans shrink it until there are 8 subtrees per
   rank, since ranks own whole subtrees) */
#define H2B_PLAN_SWEEP_NODES(v) (((v) & 0xf) << 12)

typedef struct h2b_op h2b_op;      /* device-resident operator             */
typedef struct h2b_plan h2b_plan;  /* host-only execution plan (no device) */

typedef struct h2b_stats {
  int64_t n;
  int64_t stream_bytes;     /* == H2Matrix.storage_bytes() (h2.py:77-83)   */
  int64_t pool_bytes;       /* matrix pool incl. alignment padding         */
  int64_t coef_doubles;     /* coefficient workspace (x^, y^, partials)    */
  int64_t ntasks;           /* work items in the persistent queue          */
  int64_t nsegs;
  int64_t ndeps;
  int64_t tasks_by_kind[5]; /* up-leaf, up-node, down, near, final         */
  int64_t bytes_by_kind[5];
  int32_t grid;             /* persistent CTAs                             */
  int32_t warps_per_cta;
  int32_t rank, world_size;
  int64_t local_bytes;      /* bytes this rank streams                     */
  int32_t sched_flags;      /* effective scheduling (defaults applied)     */
  int32_t ring_warps;       /* single-vector TMA-ring warps per CTA        */
  int64_t extra_bytes;      /* pool bytes beyond stream_bytes (transfer
                               products of the level-skipping chain)       */
  int32_t launches;         /* kernel launches per single-vector product (after xp = x[perm]) */
  int32_t resident_mask;    /* bit i: the sweeps of a product with 1 << i
                               right-hand sides run from shared memory
                               (resident sweep kernel); operators only     */
} h2b_stats;

/* Plan arrays for host-side inspection (tests execute them with a numpy
 * interpreter to validate the layout without a GPU).  All pointers stay
 * valid until h2b_plan_destroy.  Task/segment semantics: see DESIGN.md §4. */
typedef struct h2b_plan_view {
  int64_t ntasks, nsegs, ndeps, mat_len, coef_len;
  const double* mat;        /* [mat_len] packed column-major matrix pool    */
  const int64_t* t_data;    /* [ntasks] mat offset of (row0, col0)          */
  const int64_t* t_out;     /* [ntasks] coef offset or tree position        */
  const int64_t* t_bias;    /* [ntasks] coef offset of bias slot 0, or -1   */
  const int32_t* t_m;       /* [ntasks] rows                                */
  const int32_t* t_ld;      /* [ntasks] column stride                       */
  const int32_t* t_ncols;   /* [ntasks]                                     */
  const int32_t* t_kind;    /* [ntasks] 0 up-leaf 1 up-node 2 down 3 near 4 final */
  const int32_t* t_seg0;    /* [ntasks+1] CSR into segments                 */
  const int32_t* t_dep0;    /* [ntasks+1] CSR into deps                     */
  const int32_t* t_bias_nslots;  /* [ntasks] */
  const int32_t* t_bias_stride;  /* [ntasks] */
  const int64_t* s_src;     /* [nsegs] tree position (x) or coef offset     */
  const int32_t* s_ncols;   /* [nsegs]                                      */
  const int32_t* s_kind;    /* [nsegs] 0 = x[perm[src+c]], 1 = coef slots   */
  const int32_t* s_nslots;  /* [nsegs] slots summed (coef)                  */
  const int32_t* s_stride;  /* [nsegs] slot stride (coef)                   */
  const int32_t* deps;      /* [ndeps] task indices, all < dependent        */
  const int32_t* t_mlen;    /* [ntasks] fused run length at its first item,
                               0 for the run's other items (1: unfused)     */
  const int32_t* gated;     /* [ngated] gated coupling rows (H2B_PLAN_GATE):
                               no dependencies listed, released once all
                               n_up upward items have finished              */
  int64_t ngated;
  int32_t n_gated1;         /* gated[0:n_gated1) are inner clusters' rows   */
  int32_t n_up;
  /* the launch this phase is: mode 0 dataflow kernel, 1 sweep (units of
     items run wave by wave by one CTA, a block barrier between waves), 2
     near-field items only; group 0 before the x^ exchange of a multi-GPU
     product, 1 after it */
  int32_t mode, group;
  int32_t split;            /* 1: a launch of the split multi-RHS product
                               (H2B_PLAN_NEAR_SPLIT), 0: of the plain one    */
  int32_t resident;         /* sweeps: every unit's inputs are contiguous
                               ranges (u_range), so a CTA can run it from
                               shared memory                                */
  int64_t nunits, nwaves;
  const int32_t* unit0;     /* [nunits+1] sweeps: unit u = waves [unit0[u], unit0[u+1]) */
  const int32_t* wave0;     /* [nwaves+1] sweeps: wave w = items [wave0[w], wave0[w+1]) */
  const int64_t* u_range;   /* [8*nunits] sweeps, per unit (offset, doubles):
                               matrices in the pool; the x^ (upward) or y^
                               (downward) slots of its clusters; the near-field
                               partial slots of its leaves (downward); its
                               tree-position range of x (upward)            */
  int64_t res_mat_max;      /* sweeps: the largest unit's matrix doubles ...  */
  int64_t res_vec_max;      /* ... its coefficient + partial + x doubles ...  */
  int64_t res_items_max;    /* ... and the most items of a unit               */
} h2b_plan_view;

int h2b_abi_version(void);
const char* h2b_last_error(void);

/* Host-only planning (no CUDA calls; works on machines without a GPU). */
int h2b_plan_create(const h2b_desc* d, const h2b_options* opt, h2b_plan** out);
int h2b_plan_view_get(const h2b_plan* p, h2b_plan_view* out);
int h2b_plan_stats(const h2b_plan* p, h2b_stats* out);
/* The launches of the product in order (h2b_plan_view.mode / group): one
   dataflow launch for a single-GPU plan, two (group 0, group 1) for a
   multi-GPU rank plan; staged plans add an upward sweep before
   and a downward sweep after.  With H2B_PLAN_NEAR_SPLIT the
   launches of the split multi-RHS product follow those of the plain one. */
int h2b_plan_phases(const h2b_plan* p);
int h2b_plan_phase_view(const h2b_plan* p, int phase, h2b_plan_view* out);
/* rank_lo_hi[2*world]: tree-position range of each rank's leaves;
 * exchange[2]: {offset, doubles per rank} of the x^ exchange regions. */
int h2b_plan_partition(const h2b_plan* p, int64_t* rank_lo_hi, int64_t* exchange);
void h2b_plan_destroy(h2b_plan* p);

/* Device operator on the current CUDA device (cudaSetDevice beforehand).
 *
 * Concurrency: an operator is shareable between host threads and streams,
 * but runs ONE product at a time (its scheduler state and coefficient
 * workspace are per operator, like the single workspace of the reference's
 * per-call dicts).  Every product waits on the device for the previous
 * product of the same operator (an event chain across streams) and the
 * host-side calls are serialised by a per-operator lock, so products issued
 * from several threads or streams run one after another in issue order.
 * For concurrent products create several operators. */
int h2b_create(const h2b_desc* d, const h2b_options* opt, h2b_op** out);
/* y = M x with x, y device pointers (n x nrhs, node-major); asynchronous on
 * `stream` (cudaStream_t, NULL = legacy default).  The timed path. */
int h2b_matvec_dev(h2b_op* op, const double* x_dev, double* y_dev, int nrhs, void* stream);
/* Restore the scheduler state of a freshly created operator (synchronises
 * the device first).  Called automatically when a launch fails part-way;
 * exposed for callers recovering from an error of their own. */
int h2b_reset(h2b_op* op);
/* Synchronous host convenience (the drop-in path): copies x in, y out.
 * Multi-GPU rank operators return the full y on every rank. */
int h2b_matvec(h2b_op* op, const double* x_host, double* y_host, int64_t n, int nrhs);
/* One phase of a (multi-GPU) product -- 0: every launch before the x^
 * exchange, 1: every launch after it -- and the exchange region between them
 * (for drivers that move the x^ regions themselves instead of NCCL). */
int h2b_matvec_phase(h2b_op* op, int phase, const double* x_dev, double* y_dev, int nrhs, void* stream);
int h2b_exchange_region(h2b_op* op, int nrhs, double** base, int64_t* count_per_rank);
/* Copy src's own exchange region into dst (same layout; async on stream). */
int h2b_exchange_copy(h2b_op* dst, const h2b_op* src, int nrhs, void* stream);
int64_t h2b_stream_bytes(const h2b_op* op);
int h2b_stats_get(const h2b_op* op, h2b_stats* out);
/* The kernel launches of a product with `nrhs` right-hand sides, in order
 * (launch 0 is xp = x[perm]): h2b_launch_count returns how many; per launch
 * its kind (-1 permutation gather, 0 dataflow kernel, 1 sweep kernel, 2 lean
 * near-field kernel), its work items and the matrix bytes they stream.
 * h2b_launch_times runs `steps` products on `stream` with CUDA events around
 * every launch and returns the mean milliseconds of each (measurement aid:
 * bench.py reports the dominant kernel's roofline from it; single GPU). */
int h2b_launch_count(const h2b_op* op, int nrhs);
int h2b_launch_info(const h2b_op* op, int nrhs, int launch, int32_t* kind, int64_t* items, int64_t* bytes);
int h2b_launch_times(h2b_op* op, const double* x_dev, double* y_dev, int nrhs, int steps, void* stream,
                     double* ms_per_launch);
void h2b_destroy(h2b_op* op);

/* ---- Operator files: the reference's "H2MS" v1 format (persist.py:22-199)
 * and its CRC-64/XZ (persist.py:24-38; check value 0x995DC9BBDF1939FA for
 * "123456789").  Errors: H2B_EIO with the reference's OperatorIOError texts. */
uint64_t h2b_crc64(const void* data, uint64_t len);  /* all host cores above 8 MiB */
typedef struct h2b_h2ms h2b_h2ms;
/* Read, verify (checksum first, like load_h2) and parse a file; expected_n < 0
 * skips the node-count check.  The operator stays in host memory until
 * h2b_h2ms_close. */
int h2b_h2ms_open(const char* path, int64_t expected_n, h2b_h2ms** out);
/* Descriptor view of an opened file (pointers into it): pass to h2b_create. */
int h2b_h2ms_desc(const h2b_h2ms* f, h2b_desc* out);
/* Cluster boxes [nclusters*6] (lo xyz, hi xyz) and leaf flags [nclusters]. */
int h2b_h2ms_tree(const h2b_h2ms* f, double* bbox, uint8_t* leaf);
void h2b_h2ms_close(h2b_h2ms* f);
/* save_h2 (persist.py:117-135): the same bytes the reference writes. */
int h2b_h2ms_write(const h2b_desc* d, const double* bbox, const char* path);

/* Diagnostics: per-work-item timeline of the next products, 8 words per item
 * ({start, end, (smid << 32) | warp, continuation+1, compute done, fence
 * done, 0, 0}, globaltimer ns) and item kinds. */
int h2b_trace_enable(h2b_op* op, int on);
int h2b_trace_read(const h2b_op* op, uint64_t* out, int64_t nitems);
int h2b_item_kinds(const h2b_op* op, int32_t* out, int64_t nitems);

/* Multi-GPU helper: fill a 128-byte NCCL unique id (rank 0 calls this and
 * broadcasts the bytes to the other ranks, e.g. over torch.distributed). */
int h2b_nccl_unique_id(void* out128);

/* ---- Operator construction helper (not on the matvec path) ----------------
 * Collocation entries of M = K + D (bem.py:99-153, 207-235) evaluated on the
 * GPU for the operator builder.  `panels` holds 34 doubles per triangle:
 * v0 v1 v2 (9), unit normal (3), shape-function gradients (9), gradient .
 * edge-normal table (9), coplanarity scale (1), edge lengths (3)
 * (bem.py:67-96).  inc_ptr/inc_tri/inc_loc: node -> incident triangles CSR
 * (ascending triangle id) with the node's local vertex index. */
typedef struct h2b_colloc h2b_colloc;
int h2b_colloc_create(int64_t n, int64_t ntri, const double* panels, const int64_t* inc_ptr,
                      const int64_t* inc_tri, const int8_t* inc_loc, const double* diag,
                      h2b_colloc** out);
/* Row job j: point points[3j..3j+2]; columns colidx[col_begin[j] .. +col_count[j]];
 * diag[diag_node[j]] is added on the column equal to diag_node[j] (-1: none);
 * values land in out[out_off[j] + c].  Host arrays; synchronous. */
int h2b_colloc_eval(h2b_colloc* c, int64_t njobs, const double* points, const int64_t* col_begin,
                    const int32_t* col_count, const int64_t* diag_node, const int64_t* out_off,
                    int64_t ncolidx, const int64_t* colidx, int64_t out_len, double* out);
void h2b_colloc_destroy(h2b_colloc* c);

/* ---- FEM solves either side of the boundary operator --
 * Jacobi-preconditioned CG with optional deflation of the constant mode:
 * solver.py:44-98 cg_solve(a, b, tol, max_iter, deflate_constants,
 * precond=jacobi_preconditioner(a)), as called by fem.py:79-121 solve_u1
 * (deflate = 1) and solve_u2 (deflate = 0, on the interior block).  The
 * matrix is CSR (int64 row_ptr, int32 columns), symmetric positive
 * (semi-)definite with a zero-free diagonal (else H2B_EINVAL, like
 * jacobi_preconditioner's ValueError).  max_iter <= 0 means 10 n.  A
 * non-positive p'Ap returns H2B_ECONV.  The caller checks the deflated
 * right-hand side's compatibility (solver.py:68-70).  An h2b_cg owns its
 * work vectors: one solve at a time per object. */
typedef struct h2b_cg h2b_cg;
int h2b_cg_create(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val, h2b_cg** out);
int h2b_cg_solve(h2b_cg* c, const double* b_host, double* x_host, double tol, int deflate, int64_t max_iter,
                 int64_t* iterations, double* residual);
int h2b_cg_solve_dev(h2b_cg* c, const double* b_dev, double* x_dev, double tol, int deflate, int64_t max_iter,
                     int64_t* iterations, double* residual, void* stream);
void h2b_cg_destroy(h2b_cg* c);

/* ---- H -> H^2 recompression on the device -------------
 * hmatrix/h2.py:86-183 (_basis_side, recompress_h2), restated level by level
 * with projected factors: paper_1811_05731_b200/assembly/gpu_recompress.py
 * drives these launches; oracle/rc_ops_ref.py restates each in numpy.  All
 * pointers are DEVICE pointers; every call only enqueues one kernel on
 * `stream` and returns.  One CTA per cluster, no atomics (deterministic).
 *
 * Tree arrays, indexed by cluster id: start/end (tree positions), depth,
 * anc[c * nanc + j] = the ancestor of c at depth j (j <= depth[c], anc = c at
 * j = depth[c]), child[2c], child[2c+1] (-1 for leaves), parent.
 * One side's factors: the blocks anchored at cluster a packed side by side
 * as one row-major (end[a]-start[a]) x cown[a] matrix at fac + foff[a], their
 * column weights at wts + woff[a]; ccur[c] = sum of cown over c's ancestors
 * and c.  k[c]: kept rank.  P: the projected factors of one tree depth,
 * P_c = V_c^T [weighted factor rows] as k[c] x ccur[c] column-major at
 * P + poff[c].  Matrices of a batch: G + i * ldg * ldg, row-major, leading
 * dimension ldg, for the i-th id of the call. */

/* G_i = sum_a R_a diag(w_a^2) R_a^T over the ancestors a of leaf ids[i]
 * (at most 64 rows), R_a = the leaf's rows of a's packed block. */
int h2b_rc_leaf_gram(int64_t nleaf, const int64_t* ids, const int64_t* start, const int64_t* end, const int32_t* anc,
                     const int64_t* depth, const int64_t* foff, const int64_t* cown, int32_t nanc, const int64_t* woff,
                     const double* fac, const double* wts, int32_t ldg, double* G, void* stream);
/* Eigenpairs of nmat symmetric matrices (nvec[i] <= ldg <= 128 rows) by
 * cyclic Jacobi, in place: column j of G_i becomes the eigenvector of the
 * j-th largest eigenvalue lam[i * ldg + j].  max_sweeps <= 0: 30. */
int h2b_rc_eigh(int64_t nmat, const int64_t* nvec, double* G, int32_t ldg, double* lam, int32_t max_sweeps, void* stream);
/* P_c = V(:, :k[c])^T [R_a diag(w_a)]_a for the leaves ids[i], V = V + i ldg^2. */
int h2b_rc_leaf_project(int64_t nleaf, const int64_t* ids, const int64_t* start, const int64_t* end, const int32_t* anc,
                        const int64_t* depth, const int64_t* foff, const int64_t* cown, int32_t nanc, const int64_t* woff,
                        const double* fac, const double* wts, const double* V, int32_t ldg, const int64_t* k, double* P,
                        const int64_t* poff, const int64_t* ccur, void* stream);
/* G_i = Z Z^T, Z = the children's P (depth below: Pc, poffc) stacked, first
 * ccur[c] columns; k[child 1] + k[child 2] <= 128. */
int h2b_rc_inner_gram(int64_t n, const int64_t* ids, const int64_t* child, const int64_t* k, const int64_t* ccur,
                      const double* Pc, const int64_t* poffc, double* G, int32_t ldg, void* stream);
/* P_c = V(:, :k[c])^T Z. */
int h2b_rc_inner_project(int64_t n, const int64_t* ids, const int64_t* child, const int64_t* k, const int64_t* ccur,
                         const double* Pc, const int64_t* poffc, const double* V, int32_t ldg, double* P,
                         const int64_t* poff, void* stream);
/* Q_c = the last cown[c] columns of P_c with the weights divided out (a zero
 * weight gives a zero column), k[c] x cown[c] column-major at Q + qoff[c]. */
int h2b_rc_extract_own(int64_t n, const int64_t* ids, const int64_t* parent, const int64_t* k, const int64_t* ccur,
                       const int64_t* cown, const int64_t* woff, const double* wts, const double* P, const int64_t* poff,
                       double* Q, const int64_t* qoff, void* stream);
/* Coupling matrices (h2.py:171-176): S_b = Qr_t(:, rcol[b] .. + kb[b]) Qc_s(:, ccol[b] .. + kb[b])^T,
 * kr[t] x kc[s] row-major at S + soff[b], t = bt[b], s = bs[b]. */
int h2b_rc_coupling(int64_t nb, const int64_t* bt, const int64_t* bs, const int64_t* rcol, const int64_t* ccol,
                    const int64_t* kb, const double* Qr, const int64_t* qoffr, const int64_t* kr, const double* Qc,
                    const int64_t* qoffc, const int64_t* kc, double* S, const int64_t* soff, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* H2B_H_ */
