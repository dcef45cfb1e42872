// plan.h — host-side execution plan of the H² matvec (no CUDA dependencies).
//
// The reference applies the operator with four Python loops over small
// GEMVs (h2.py:195-240).  Here every one of those GEMVs becomes a "work item"
// of one uniform shape:
//
//     out[0:m] (+)= bias[0:m] + A[0:m, 0:ncols] @ gather(segments)
//
// where A is a column-major slice of one packed matrix pool and the gathered
// source vector is the concatenation of the item's segments (x through the
// cluster permutation, or cluster coefficients x^ / y^ held in a workspace).
// Items are stored in a topologically ordered queue; each lists the items it
// depends on.  A persistent CUDA kernel drains the queue.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../../include/h2b.h"

namespace h2b {

enum TaskKind : int32_t {
  kUpLeaf = 0,   // x^_t = W_t^T x|_t                       h2.py:199-200
  kUpNode = 1,   // x^_p = sum_c F_c^T x^_c                 h2.py:201-205
  kDown = 2,     // y^_t = E_t y^_parent + sum_b S_b x^_s    h2.py:211-218, 231-233
  kNear = 3,     // partial_t = sum_s N_ts x|_s              h2.py:237-240
  kFinal = 4,    // y[perm[t]] = sum partial_t + V_t y^_t    h2.py:227-229, 242-243
};

enum SegKind : int32_t {
  kSegX = 0,     // xp[src + c], xp = x[perm] (permutation gather, h2.py:192-193)
  kSegCoef = 1,  // sum_j coef[src + j*stride + c], j < nslots
};

constexpr int kMaxRows = 64;  // rows per work item (lanes own rows l, l+32)
constexpr int kMaxSegs = 32;  // source segments per work item (one per lane)
constexpr int kMaxNearPieces = 32;  // near-field items per leaf row at most

// One launch of the persistent kernel: a work-item queue (queue order, all
// dependencies earlier) with its scheduling metadata.
struct Phase {
  // tasks (queue order)
  std::vector<int64_t> t_data, t_out, t_bias;
  std::vector<int32_t> t_m, t_ld, t_ncols, t_kind, t_seg0, t_dep0;
  std::vector<int32_t> t_bias_nslots, t_bias_stride;
  std::vector<int8_t> t_qclass;     // 0: far-field chain, 1: inner coupling, 2: leaf coupling / near
  // Fused runs: item i with t_mlen[i] = L > 0 is scheduled as
  // one unit that runs items i .. i+L-1 in order on one warp; its deps and
  // successors are the run's external ones.  t_mlen = 0 marks the members
  // after the first (never scheduled on their own, no deps of their own).
  std::vector<int32_t> t_mlen;
  int64_t nnodes = 0;               // scheduled units (items with t_mlen > 0)
  // segments
  std::vector<int64_t> s_src;
  std::vector<int32_t> s_ncols, s_kind, s_nslots, s_stride;
  // dependencies
  std::vector<int32_t> deps;
  // successors (inverse of deps, CSR) and the initially ready items in
  // issue order: the kernel's dynamic scheduler
  std::vector<int32_t> succ0, succ;
  std::vector<int32_t> ready0;
  int32_t n_ready0_hi = 0;          // ready0[0:n_ready0_hi) are class 0
  // Gated coupling rows (PlanOptions::gate_coupling): down items whose only
  // inputs are upward coefficients carry no dependencies; they are claimed
  // from these lists (inner clusters' rows first, then the leaves' rows,
  // longest first) once all `n_up` upward items of the phase have finished.
  std::vector<int32_t> gated;
  int32_t n_gated1 = 0;             // gated[0:n_gated1) are class 1
  int32_t n_up = 0;
  int64_t tasks_by_kind[5] = {0, 0, 0, 0, 0};
  // Launch kind and position in the product (staged plans).
  // mode 0: the completion-driven dataflow kernel; 1: a sweep -- CTA-
  // cooperative units (bottom subtrees of the cluster tree) whose items run
  // wave by wave with a block barrier between waves, no arrival counters;
  // 2: near-field items only (multi-RHS: the lean near kernel).
  // group 0: before the x^ exchange of a multi-GPU product, 1: after it.
  int32_t mode = 0, group = 0;
  // sweeps: unit u is waves [unit0[u], unit0[u+1]); wave w is the items
  // [wave0[w], wave0[w+1]) of the queue (a unit's items are contiguous and
  // form one fused run: t_mlen = its length at its first item)
  std::vector<int32_t> unit0, wave0;
  // Resident sweeps: everything a unit reads is a few contiguous ranges that
  // its CTA copies into shared memory before running the waves from there.
  // Per unit 8 numbers (doubles, pool / workspace / tree positions): matrices
  // [0] + [1]; main coefficients (the unit's x^ or y^ slots) [2] + [3]; the
  // near-field partial slots of its leaves (downward sweep) [4] + [5]; its
  // tree-position range of x (upward sweep) [6] + [7].  `resident` is false
  // when some unit's ranges are not contiguous (the generic sweep runs then).
  std::vector<int64_t> u_range;
  // ... and, for the kernel, one 128-byte record per unit (16 x int64): the
  // 8 range numbers; first item | items << 32; number of waves; then the
  // waves' end items (relative to the unit's first) as 12 x int32
  std::vector<int64_t> u_rec;
  bool resident = false;
  int64_t res_mat_max = 0, res_vec_max = 0;  // largest unit: matrix doubles; coefficient + partial + x doubles
  int32_t res_items_max = 0;                 // most items in a unit

  int64_t ntasks() const { return (int64_t)t_m.size(); }
  int64_t nsegs() const { return (int64_t)s_ncols.size(); }
};

// One packed matrix of the pool: the column blocks of a work-item group
// (m rows, column-major, ld = m), copied from the descriptor's host arrays
// when the pool is materialised (pack_pool).  base < 0: not used by this
// rank's plan (multi-GPU) and not packed.
struct PackSeg {
  const double* a;   // source block
  int64_t ncols;
  bool transpose;    // false: a is (ncols x m) row-major == (m x ncols) col-major
  int64_t a_ld;      // row stride of a when transposed
};
struct Group {
  int64_t base = -1;
  int32_t m = 0;
  int64_t ncols = 0;
  // staged plans: 1 the matrices of an upward sweep unit, 2 of a downward
  // sweep unit (`unit`: the tree position where its subtree starts), 0 others;
  // the pool is laid out region by region and unit by unit, so that a unit's
  // matrices are one contiguous range (one bulk copy into shared memory)
  int32_t region = 0;
  int64_t unit = 0;
  std::vector<PackSeg> segs;
  int64_t size() const { return (int64_t)m * ncols; }
};

// The execution plan of one operator on one rank.  Single GPU: one phase.
// world_size > 1: phase 0 computes the upward coefficients
// x^ of the clusters this rank owns into its exchange region of the
// coefficient workspace, the regions are all-gathered (every rank's region
// has exch_count doubles, rank r's at exch_off + r * exch_count), and phase 1
// runs the rest of this rank's rows: the clusters spanning several ranks
// (replicated), the downward pass, the near field and the finals of its
// leaves.
struct Plan {
  int64_t n = 0;
  std::vector<int64_t> perm;
  std::vector<Group> groups;  // the pool's matrices (pointers into the descriptor or `owned`)
  // transfer products of the level-skipping chain (PlanOptions::skip_levels),
  // computed at planning time; groups point into them
  std::vector<std::unique_ptr<std::vector<double>>> owned;
  int64_t extra_bytes = 0;    // pool bytes beyond storage_bytes (the products)
  int64_t mat_len = 0;        // doubles of this rank's pool
  std::vector<double> mat;    // host copy of the pool (pack_pool; empty after a streamed upload)
  int64_t coef_len = 0;     // doubles per right-hand side
  int64_t stream_bytes = 0; // == H2Matrix.storage_bytes()
  int64_t bytes_by_kind[5] = {0, 0, 0, 0, 0};
  int32_t rank = 0, world_size = 1;
  int64_t local_bytes = 0;  // matrix bytes streamed by this rank
  std::vector<Phase> ph;
  // Single GPU, PlanOptions::near_split: the same items in two launches --
  // the near field alone (no dependencies: the lean multi-RHS kernel), then
  // everything else (its near-field dependencies satisfied by the first).
  std::vector<Phase> ph_split;
  int64_t exch_off = 0, exch_count = 0;
  std::vector<int64_t> rank_lo, rank_hi;  // tree-position range of each rank's leaves
};

struct PlanOptions {
  int64_t task_bytes = 65536;     // near-field items (and leaf coupling rows)
  int64_t far_task_bytes = 4096;  // up-leaf, up-node and down items
  int32_t band_depth = 1;         // tree levels fused into one run of the far-field chain (1: none)
  int32_t final_class = 0;        // queue class of the final items (0: chain, 2: slack)
  int32_t near_phase0_pct = 90;   // multi-GPU: percent of the rank's near bytes in phase 0 (0: none)
  bool interleave = true;
  bool near_split = false;        // also plan Plan::ph_split (single GPU)
  // Level-skipping far-field chain: the upward coefficients of clusters of
  // even height come from their grandchildren through transfer products
  // (F_g F_c)^T, and the downward coefficients of every other level from
  // their grandparent through E_c E_p (the level between contributes only its
  // own coupling sum), so the dependency chain through the tree has half the
  // links.  Extra pool bytes: one product per skipped link.
  bool skip_levels = false;
  // pieces of the leaf clusters' coupling rows (0: task_bytes); a heavy row
  // cut finer runs on more warps at once instead of forming the tail
  int64_t coupling_task_bytes = 0;
  // release coupling rows behind one counter of finished upward items
  // instead of one arrival per (source, row) edge
  bool gate_coupling = false;
  // Staged product: the clusters of at most `sweep_nodes`
  // nodes whose parents are larger root "bottom subtrees".  Their upward
  // items run first as a sweep (one CTA per subtree, block barriers between
  // tree levels), then one dataflow launch runs the near field, every
  // coupling row and the far-field chain of the clusters above the subtrees,
  // then a second sweep runs the subtrees' downward transfers and the finals.
  // Only the short top chain keeps arrival counters; near items and the
  // coupling rows of bottom clusters have neither inputs to wait for nor
  // successors to notify.  Multi-GPU: ranks own whole subtrees.
  bool staged = false;
  // the split multi-RHS product (near_split) also runs the bottom subtrees as
  // sweeps: [up sweep] near kernel, dataflow launch [down sweep]
  bool split_sweeps = false;
  int64_t sweep_nodes = 0;        // 0: default (about 256 subtrees per rank)
  int32_t rank = 0;
  int32_t world_size = 1;
};

// Validates the descriptor and builds the plan.  Returns H2B_OK or an error
// code with a message in *err.  The pool itself is not packed (the groups
// point into the descriptor's arrays): see pack_pool / pack_groups.
int build_plan(const h2b_desc* d, const PlanOptions& opt, Plan* out, std::string* err);

// Copies groups [g0, g1) of the pool to dst, which corresponds to pool offset
// groups[g0].base (the used groups are contiguous in group order); skips
// unused groups.  Uses up to `threads` host threads.
void pack_groups(const Plan& P, size_t g0, size_t g1, double* dst, int threads);
// Materialises the whole pool in P.mat (host).
void pack_pool(Plan* P, int threads);

}  // namespace h2b
