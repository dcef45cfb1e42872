// h2b.cu — B200 (sm_100a) H² matvec: one persistent dataflow kernel + C ABI.
//
// The whole product y = M x (h2.py:186-244) is one permutation-gather launch
// (xp = x[perm]) plus ONE persistent kernel.  The host planner (plan.cpp)
// turns every small GEMV of the reference's four loops into a work item
//
//     out[0:m] = bias[0:m] + A[0:m, 0:ncols] @ gather(segments)
//
// over a column-major slice of one packed matrix pool.  Scheduling is
// completion driven: items without inputs (up-leaf, near field) start in a
// static queue; each finished item counts itself into its successors, and
// the warp that completes a successor's count pushes it onto a dynamic
// ready queue, which warps serve first (the far-field tree chain is the
// critical path).  No warp ever waits on an unfinished item.
//
// Streaming: lanes own rows (r = lane, lane + 32) so every column is one
// contiguous, coalesced read with no cross-lane reduction.  A warp either
// keeps 8 columns of 64-bit ld.global.nc.L1::no_allocate loads in flight
// (the first ones issued before the item's sources are gathered), or -- a
// "ring warp" -- moves the item through a two-stage shared-memory ring by
// 1-D TMA bulk copies (more bytes in flight, no registers); both run the
// same column-ordered FMA chain.  Items with m <= 16 pack 32/m columns per
// warp instruction and reduce once.  8 and 16 right-hand sides multiply on
// the FP64 tensor cores (DMMA).  Split rows write partial slots that the
// consumer adds in a fixed order: deterministic, no floating-point atomics.
// Scheduling and streaming variants: h2b_options.sched_flags.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdio>
#include <functional>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <string>
#include <type_traits>
#include <vector>

#include <nccl.h>

#include "../../include/h2b.h"
#include "plan.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define H2B_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(H2B_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));        \
  } while (0)

struct __align__(16) DTask {
  int64_t data;   // mat offset of (row0, col0)
  int64_t out;    // coef offset (slot) or tree position (final)
  int64_t bias;   // coef offset or -1
  int32_t m, ld, ncols, kind;
  int32_t seg0, seg1;
  int32_t pad0_, pad1_;
  int32_t bias_nslots, bias_stride;
};
static_assert(sizeof(DTask) == 64, "DTask layout");

struct __align__(8) DSeg {
  int64_t src;
  int32_t ncols;
  int32_t kind;
  int32_t nslots;
  int32_t stride;
};
static_assert(sizeof(DSeg) == 24, "DSeg layout");

// Scheduler state (one per operator).  Every counter is reset by the last
// warp to leave a launch and `epoch` counts launches, so nothing is cleared
// between products.  Each hot counter sits on its own 128-byte line.
constexpr int kQueues = 3;  // 0: far-field chain, 1: upper coupling, 2: leaf coupling
struct Line {
  unsigned v;
  unsigned pad[31];
};
struct Ctl {
  Line head[kQueues];    // dynamic queue q: next slot to claim
  Line tail[kQueues];    // dynamic queue q: next slot to push
  unsigned static_head;  // next initially-ready up-leaf item to claim
  unsigned pad2[31];
  unsigned near_head;    // next initially-ready near-field item to claim
  unsigned pad5[31];
  unsigned dyn_started;  // dynamic items taken (queue or continuation)
  unsigned pad4[31];
  unsigned exited;       // warps that left the scheduler loop
  unsigned epoch;        // launches completed so far
  unsigned pad3[30];
  Line gate;             // upward items finished (gated coupling rows wait for n_up)
  Line g_head[2];        // gated lists: next item to claim (inner rows, leaf rows)
};

struct KParams {
  const DTask* __restrict__ tasks;
  const DSeg* __restrict__ segs;
  const DSeg* __restrict__ seg_inline;  // [ntasks * kInlineSegs]: segments of items with few of them
  const int32_t* __restrict__ succ0;    // [ntasks+1] successor CSR
  const int2* __restrict__ succ;         // (successor, its dependency count)
  const int32_t* __restrict__ ready0;   // initially ready items, issue order
  const double* __restrict__ mat;
  double* coef;
  const int64_t* __restrict__ perm;
  const double* __restrict__ xp;        // x in tree order (written by the gather launch)
  double* y;
  unsigned long long* arrived;          // per item: finished predecessors, all launches
  int32_t* ready_q;                     // dynamic ready queue (item ids)
  unsigned* ready_flag;                 // per slot: epoch+1 once the id is written
  Ctl* ctl;
  int32_t ntasks;
  int32_t nnodes;                       // scheduled units (fused runs count once)
  int32_t nready0;
  int32_t nready0_hi;                   // ready0[0:nready0_hi) are class 0
  int32_t flags;                        // kFlag* scheduling switches (h2b_options.sched_flags)
  int32_t ring_warps;                   // NRHS < 8: warps per CTA (the top ones) with a TMA ring
  int32_t ring_stage;                   // NRHS < 8: ring stage payload bytes (8192, 6144, 4096)
  int32_t mrhs_stage;                   // NRHS >= 8: ring stage payload bytes (8192; 6144 with 12 warps per CTA)
  unsigned long long* trace;            // diagnostics: per item {start ns, end ns, sm|warp, 0}
  const int32_t* __restrict__ gated;    // gated coupling rows (Phase::gated)
  int32_t ngated, ngated1, nup_gate;
  // sweeps (Phase::mode 1): units of waves of items
  const int32_t* __restrict__ unit0;
  const int32_t* __restrict__ wave0;
  int32_t nunits;
  // resident sweeps: per-unit ranges (Phase::u_range) and the shared-memory
  // capacities (doubles; items) the launch was sized for
  const int64_t* __restrict__ u_range;
  int32_t cap_mat, cap_vec, cap_items;
  int32_t sweep_prefetch;               // generic sweep: the next item's static inputs prefetched to L2
  // programmatic dependent launch (H2B_PDL=1): bit 0, a sweep lets the next
  // launch start while it runs; bit 1, a dataflow launch started that way
  // waits for the sweep before its first item that is not near field
  int32_t pdl;
};

// scheduling switches
constexpr int kFlagSlackFirst = 1;  // inner coupling rows before the claimed-ahead near item
constexpr int kFlagNoRing = 1 << 24; // multi-RHS: register-staged streaming instead of the TMA ring
constexpr int kFlagReleaseArrivals = 1 << 2;  // release-only arrival atomics, acquire fence on completion
constexpr int kFlagStreamEvictFirst = 1 << 25;  // ring copies with an L2 evict-first hint
constexpr int kFlagMixInner = (int)(1u << 31);  // near-priority warps' mix serves inner coupling rows too
constexpr int kFlagMrhsRingAll = 2;  // 8/16 RHS: far items through the ring too (TMA sources), not staged whole
constexpr int kFlagMrhsSrcInStage = 1 << 4;  // 8/16 RHS rings: TMA-moved sources behind the matrix chunk in the stage
constexpr int kFlagUpMix = 1 << 3;   // near-priority warps' mix takes up-leaf items first (H2B_UP_MIX=1)
constexpr int kFlagPrioNoChain = 1 << 30;       // near-priority warps leave the chain queue to the others
constexpr int kChunkBytes = 4096;  // per-warp shared staging of gathered sources
constexpr int kInlineSegs = 4;     // segments stored per item next to the task
constexpr int kStageBytes = 4096 + 128;  // TMA staging of one far-field item (+ alignment)

// Per-warp shared memory: gathered sources, the item's segment table, the
// small-item reduction scratch and the far-field staging mbarrier (the
// staging buffer or ring itself follows the WarpSmem array, see WarpRing).
struct __align__(128) WarpSmem {
  double xs[kChunkBytes / 8];
  unsigned long long bar;
  unsigned long long dbg[3];  // diagnostics (tracing): segment table, gather, multiply done
  double red[32];
  long long seg_src[h2b::kMaxSegs];
  int seg_off[h2b::kMaxSegs + 1];
  int seg_kind[h2b::kMaxSegs];
  int seg_nslots[h2b::kMaxSegs];
  int seg_stride[h2b::kMaxSegs];
};

// Per-warp TMA ring of streamed items: two stages of 8 KB (+ alignment
// slack).  Ring warps (all warps for NRHS >= 8, the top `ring_warps` of each
// CTA otherwise) stream their items through it; a ring warp stages its
// far-field items in buf[0].  Other warps have a kStageBytes staging buffer.
// Dynamic shared memory: [WarpSmem x nw][staging of non-ring warps][rings].
// Stage payload: 8 KB (multi-RHS, and the single-vector default), or 6 / 4
// KB for single-vector products (sched_flags bits 18-19), which lets more
// warps of a CTA own a ring at two CTAs per SM.
constexpr int kRingStageBytes = 8192;
// 8/16 right-hand sides in the dataflow and sweep kernels: one CTA per SM.
// The far part of such a product is latency-bound (150 k small items on
// config 3), so warps per SM are what counts, and registers decide them:
//   MT 4 (64 rows per pass), 256 threads, 255 registers    16 RHS 4.555 ms
//   MT 4, 384 threads at 168 registers: 2.2 KB of spills   5.27 ms (12 warps)
//   MT 2 (32 rows per pass; taller items in two passes),
//        384 threads at 168 registers, 6 KB ring stages     4.248 ms, 8 RHS 3.598 -> 3.394 ms
//   MT 2, 256 threads x 2 CTAs at 128 registers, 4 KB stages: spills, 5.35 ms
// (profiles/r02_config3_mrhs_warps.jsonl).  H2B_MRHS_WARPS launches fewer
// warps than compiled for.
#ifndef H2B_MRHS_MT
#define H2B_MRHS_MT 2
#endif
#ifndef H2B_MRHS_THREADS
#define H2B_MRHS_THREADS 384
#endif
constexpr int kMrhsMT = H2B_MRHS_MT;
constexpr int kMrhsStage = 8192;
constexpr int kMrhsCtas = (kMrhsMT >= 4 || H2B_MRHS_THREADS > 256) ? 1 : 2;
constexpr int kMrhsThreads = H2B_MRHS_THREADS;
// The generic sweep kernel has no scheduler state: with 32-row passes it fits
// 128 registers (16 RHS: 248 bytes of spills), two CTAs per SM.
#ifndef H2B_MRHS_SWEEP_CTAS
#define H2B_MRHS_SWEEP_CTAS 2
#endif
constexpr int kMrhsSweepCtas = H2B_MRHS_SWEEP_CTAS;
struct WarpRing {  // view into dynamic shared memory (no dynamically indexed arrays)
  double* base;     // stage 0; stage 1 follows at base + sdbl
  uint64_t* bars;   // two mbarriers
  int sdbl;         // stage stride in doubles
  __device__ __forceinline__ double* buf(int j) const { return base + (j & 1) * sdbl; }
  __device__ __forceinline__ uint64_t* bar(int j) const { return bars + (j & 1); }
};
__host__ __device__ constexpr int ring_bytes(int stage) { return ((2 * (stage + 32) + 16) + 127) / 128 * 128; }
static_assert(kStageBytes % 128 == 0 && sizeof(WarpSmem) % 128 == 0, "staging alignment");
static_assert(2 * (4096 + 32) >= kStageBytes, "a ring (both stages, contiguous) doubles as far-field staging");
inline size_t smem_bytes(int nw, int ring_warps, int stage) {
  return (size_t)nw * sizeof(WarpSmem) + (size_t)(nw - ring_warps) * kStageBytes +
         (size_t)ring_warps * ring_bytes(stage);
}

__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// Arrival count: releases this warp's outputs (after __syncwarp) and acquires
// the other predecessors' (their arrivals precede ours in the counter's
// modification order), so neither a separate fence before nor after is needed.
__device__ __forceinline__ unsigned long long atom_add_acq_rel(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
// Release-only arrival: publishes this warp's outputs without the L1
// invalidation an acquire costs; the completing warp acquires with a fence.
__device__ __forceinline__ unsigned long long atom_add_release(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.release.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---- 1-D TMA (cp.async.bulk) staging into shared memory, mbarrier completion
__device__ __forceinline__ uint32_t smem_u32(const void* q) { return (uint32_t)__cvta_generic_to_shared(q); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// One lane: copy [src, src + bytes) (16-byte aligned, multiple of 16) to dst,
// completing the current phase of `bar`.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after generic reads of dst
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// The same with an L2 eviction-priority hint (createpolicy): the streamed
// matrix is read once, so it should not evict the gathered sources.
__device__ __forceinline__ void bulk_load_hint(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                               uint64_t policy) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// ring copies: with an evict-first hint when the stream_ef flag is set
__device__ __forceinline__ void ring_load(const KParams& p, void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  if (p.flags & kFlagStreamEvictFirst) bulk_load_hint(dst, src, bytes, bar, evict_first_policy());
  else bulk_load(dst, src, bytes, bar);
}

// mbarrier expecting `bytes` from the bulk copies issued next (one arrival).
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_copy_hint(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                               uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// xp = x[perm] (h2.py:192-193), node-major with NRHS columns.
template <int NRHS>
__global__ void __launch_bounds__(256) h2b_permute_kernel(const double* __restrict__ x,
                                                          const int64_t* __restrict__ perm,
                                                          double* __restrict__ xp, int64_t n) {
  const int64_t total = n * NRHS;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = i / NRHS, r = i - pos * NRHS;
    xp[i] = __ldg(x + __ldg(perm + pos) * NRHS + r);
  }
}

// Multi-GPU host path: this rank's rows (tree positions [lo, lo + cnt)) of
// y, packed in tree order, then every rank's packed rows back to node order.
__global__ void __launch_bounds__(256) h2b_pack_rows_kernel(const double* __restrict__ y,
                                                            const int64_t* __restrict__ perm, int64_t lo,
                                                            int64_t cnt, int nrhs, double* __restrict__ out) {
  const int64_t total = cnt * nrhs;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = i / nrhs, r = i - pos * nrhs;
    out[i] = y[perm[lo + pos] * nrhs + r];
  }
}

__global__ void __launch_bounds__(256) h2b_unpack_rows_kernel(const double* __restrict__ rows,
                                                              const int64_t* __restrict__ perm,
                                                              const int64_t* __restrict__ rank_lo, int world,
                                                              int64_t n, int64_t rows_max, int nrhs,
                                                              double* __restrict__ y) {
  const int64_t total = n * nrhs;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = i / nrhs, r = i - pos * nrhs;
    int q = world - 1;  // owner of tree position pos (ranges ascending)
    while (q > 0 && rank_lo[q] > pos) --q;
    y[perm[pos] * nrhs + r] = rows[((int64_t)q * rows_max + (pos - rank_lo[q])) * nrhs + r];
  }
}

// Source value (NRHS column r) of item column c, through the warp's segment table.
template <int NRHS>
__device__ __forceinline__ double gather_one(const KParams& p, const WarpSmem& w, int c, int r, int& k) {
  while (w.seg_off[k + 1] <= c) ++k;
  const int cs = c - w.seg_off[k];
  if (w.seg_kind[k] == h2b::kSegX) return __ldg(p.xp + (w.seg_src[k] + cs) * NRHS + r);
  const double* q = p.coef + (w.seg_src[k] + cs) * NRHS + r;
  const int64_t st = (int64_t)w.seg_stride[k] * NRHS;
  const int ns = w.seg_nslots[k];
  // partial slots of a split producer, added in slot order; eight loads in
  // flight at a time (split rows of upper clusters have dozens of slots)
  double v = 0.0;
  int s = 0;
  for (; s + 8 <= ns; s += 8) {
    double t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = __ldcg(q + (int64_t)(s + u) * st);
#pragma unroll
    for (int u = 0; u < 8; ++u) v += t[u];
  }
  for (; s < ns; ++s) v += __ldcg(q + (int64_t)s * st);
  return v;
}

__device__ __forceinline__ void add_to(double& a, double b) { a += b; }
__device__ __forceinline__ void add_to(double2& a, double2 b) {
  a.x += b.x;
  a.y += b.y;
}

// Gather the sources of item columns [col, col + cc) (all NRHS values of
// each) into the warp's staging buffer xs, through the segment table.
// VW consecutive values (same column, consecutive right-hand sides: they
// are contiguous in x and in the coefficient slots) per load and UG loads
// per lane in flight: the first (or only) slot of each is one predicated
// load -- x through the read-only path (L1 hits across items on the same
// SM), coefficient slots from L2 -- and split producers' further partial
// slots are added afterwards in slot order (eight loads in flight), so
// every value is slot0 + slot1 + ... in a fixed order.
template <int NRHS>
__device__ __forceinline__ double gather_one(const KParams& p, const WarpSmem& w, int c, int r, int& k);

template <int NRHS>
__device__ __forceinline__ void gather_chunk(const KParams& p, WarpSmem& w, int lane, int col, int cc) {
  if constexpr (NRHS == 1) {
    // single vector: one value per load, the matrix stream already in flight
    int k = 0;
    for (int j = lane; j < cc; j += 32) w.xs[j] = gather_one<1>(p, w, col + j, 0, k);
    return;
  }
  constexpr int VW = NRHS >= 2 ? 2 : 1;
  constexpr int UG = 4;
  using V = typename std::conditional<VW == 2, double2, double>::type;
  const int total = cc * NRHS / VW;
  int k = 0;  // segment cursor (columns increase along a lane)
  for (int j0 = lane; j0 < total; j0 += 32 * UG) {
    V v[UG];
    const V* q[UG];
    int ns[UG];
    bool isx[UG];
    int64_t st[UG];
#pragma unroll
    for (int u = 0; u < UG; ++u) {
      const int j = (j0 + 32 * u) * VW;
      const int c = col + j / NRHS, r = j % NRHS;
      ns[u] = 0;
      isx[u] = false;
      q[u] = reinterpret_cast<const V*>(p.coef);
      st[u] = 0;
      if (j < total * VW) {
        while (w.seg_off[k + 1] <= c) ++k;
        const int64_t e = (w.seg_src[k] + (c - w.seg_off[k])) * NRHS + r;
        isx[u] = w.seg_kind[k] == h2b::kSegX;
        q[u] = reinterpret_cast<const V*>((isx[u] ? p.xp : p.coef) + e);
        ns[u] = isx[u] ? 1 : w.seg_nslots[k];
        st[u] = (int64_t)w.seg_stride[k] * NRHS / VW;
      }
    }
#pragma unroll
    for (int u = 0; u < UG; ++u) {
      if (ns[u] == 0) v[u] = V{};
      else v[u] = isx[u] ? __ldg(q[u]) : __ldcg(q[u]);
    }
#pragma unroll
    for (int u = 0; u < UG; ++u) {
      int s = 1;
      for (; s + 8 <= ns[u]; s += 8) {
        V t[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) t[i] = __ldcg(q[u] + (int64_t)(s + i) * st[u]);
#pragma unroll
        for (int i = 0; i < 8; ++i) add_to(v[u], t[i]);
      }
      for (; s < ns[u]; ++s) add_to(v[u], __ldcg(q[u] + (int64_t)s * st[u]));
    }
    V* xs = reinterpret_cast<V*>(w.xs);
#pragma unroll
    for (int u = 0; u < UG; ++u)
      if (j0 + 32 * u < total) xs[j0 + 32 * u] = v[u];
  }
}

// The item's segment table into the warp's shared memory: one segment per
// lane, column offsets by warp scan.
__device__ __forceinline__ void load_segtable(const KParams& p, const DTask& T, const DSeg& sin, WarpSmem& w,
                                              int lane) {
  const int nseg = T.seg1 - T.seg0;  // <= kMaxSegs (planner)
  int nc = 0;
  if (lane < nseg) {
    // items with few segments carry them inline (fetched with the task)
    const DSeg S = nseg <= kInlineSegs ? sin : p.segs[T.seg0 + lane];
    nc = S.ncols;
    w.seg_src[lane] = S.src;
    w.seg_kind[lane] = S.kind;
    w.seg_nslots[lane] = S.nslots;
    w.seg_stride[lane] = S.stride;
  }
  int incl = nc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane < nseg) w.seg_off[lane] = incl - nc;
  if (lane == nseg - 1 || (nseg == 0 && lane == 0)) w.seg_off[nseg] = incl;
  if (lane == 0 && nseg < h2b::kMaxSegs) w.seg_off[h2b::kMaxSegs] = 0x7fffffff;
  __syncwarp();
}

template <bool SMEM>
__device__ __forceinline__ double ldA(const double* q) {
  if constexpr (SMEM) return *q;
  else return ld_stream(q);
}

// Bias: partial slots of the output rows (lane, lane + 32), summed in slot
// order (loads batched: heavy rows have hundreds of slots).
template <int NRHS>
__device__ __forceinline__ void add_bias(const KParams& p, const DTask& T, double (&acc0)[NRHS],
                                         double (&acc1)[NRHS], int lane) {
  const bool v0 = lane < T.m, v1 = lane + 32 < T.m;
  if (T.bias >= 0) {
    int s = 0;
    constexpr int QB = NRHS == 1 ? 16 : (NRHS == 2 ? 4 : 1);
    for (; s + QB <= T.bias_nslots; s += QB) {
      double b0[QB][NRHS], b1[QB][NRHS];
#pragma unroll
      for (int q = 0; q < QB; ++q) {
        const double* b = p.coef + (T.bias + (int64_t)(s + q) * T.bias_stride) * NRHS;
#pragma unroll
        for (int r = 0; r < NRHS; ++r) {
          b0[q][r] = v0 ? __ldcg(b + (int64_t)lane * NRHS + r) : 0.0;
          b1[q][r] = v1 ? __ldcg(b + (int64_t)(lane + 32) * NRHS + r) : 0.0;
        }
      }
#pragma unroll
      for (int q = 0; q < QB; ++q)
#pragma unroll
        for (int r = 0; r < NRHS; ++r) {
          acc0[r] += b0[q][r];
          acc1[r] += b1[q][r];
        }
    }
    for (; s < T.bias_nslots; ++s) {
      const double* b = p.coef + (T.bias + (int64_t)s * T.bias_stride) * NRHS;
#pragma unroll
      for (int r = 0; r < NRHS; ++r) {
        if (v0) acc0[r] += __ldcg(b + (int64_t)lane * NRHS + r);
        if (v1) acc1[r] += __ldcg(b + (int64_t)(lane + 32) * NRHS + r);
      }
    }
  }
}

// Output rows (lane, lane + 32): a coefficient slot, or y in node order.
template <int NRHS>
__device__ __forceinline__ void store_rows(const KParams& p, const DTask& T, const double (&acc0)[NRHS],
                                           const double (&acc1)[NRHS], int lane) {
  const int m = T.m;
  const bool w0 = lane < m, w1 = lane + 32 < m;
  if (T.kind == h2b::kFinal) {
    if (w0) {
      const int64_t node = __ldg(p.perm + T.out + lane);
#pragma unroll
      for (int r = 0; r < NRHS; ++r) p.y[node * NRHS + r] = acc0[r];
    }
    if (w1) {
      const int64_t node = __ldg(p.perm + T.out + lane + 32);
#pragma unroll
      for (int r = 0; r < NRHS; ++r) p.y[node * NRHS + r] = acc1[r];
    }
  } else {
#pragma unroll
    for (int r = 0; r < NRHS; ++r) {
      if (w0) p.coef[(T.out + lane) * NRHS + r] = acc0[r];
      if (w1) p.coef[(T.out + lane + 32) * NRHS + r] = acc1[r];
    }
  }
}

// One work item with NRHS right-hand sides.  A is the item's column-major
// matrix: staged in shared memory by a TMA bulk copy that completes on `bar`
// (SMEM), or streamed from global memory.
template <int NRHS, bool SMEM, int UC>
__device__ __forceinline__ void run_item(const KParams& p, const DTask& T, const DSeg& sin, WarpSmem& w,
                                         int lane, const double* A, uint64_t* bar, unsigned parity,
                                         unsigned long long& t_gath) {
  constexpr int kCols = kChunkBytes / (8 * NRHS);
  constexpr int U = (NRHS == 1) ? UC : 4;  // columns in flight per lane
  const int m = T.m, ld = T.ld;

  load_segtable(p, T, sin, w, lane);
  if (p.trace && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(w.dbg[0])::"memory");

  const bool grouped = (NRHS == 1) && (m <= 16) && (ld == m) && (m > 0);
  double acc0[NRHS], acc1[NRHS];
#pragma unroll
  for (int r = 0; r < NRHS; ++r) { acc0[r] = 0.0; acc1[r] = 0.0; }

  if (grouped) {
    // G columns per step; lane (g, rr) reads element (rr, c + g): the warp
    // touches G*m consecutive doubles per instruction.
    const int G = 32 / m, g = lane / m, rr = lane - g * m;
    const bool v0 = g < G;
    for (int col = 0; col < T.ncols; col += kCols) {
      const int cc = min(kCols, T.ncols - col);
      gather_chunk<NRHS>(p, w, lane, col, cc);
      __syncwarp();
      if (p.trace && col == 0 && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(w.dbg[1])::"memory");
      if (SMEM && col == 0) mbar_wait(bar, parity);
      if (p.trace && col == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_gath)::"memory");
      const double* Ac = A + (int64_t)col * m;
      int c = g;
      for (; c + 7 * G < cc; c += 8 * G) {
        double a[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = v0 ? ldA<SMEM>(Ac + (int64_t)(c + u * G) * m + rr) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) acc0[0] = fma(a[u], w.xs[c + u * G], acc0[0]);
      }
      for (; c < cc; c += G)
        if (v0) acc0[0] = fma(ldA<SMEM>(Ac + (int64_t)c * m + rr), w.xs[c], acc0[0]);
      __syncwarp();
    }
    w.red[lane] = acc0[0];
    __syncwarp();
    double s = 0.0;
    if (lane < m) {
      for (int q = 0; q < G; ++q) s += w.red[q * m + lane];
      if (T.bias >= 0)
        for (int b = 0; b < T.bias_nslots; ++b)
          s += __ldcg(p.coef + T.bias + (int64_t)b * T.bias_stride + lane);
    }
    __syncwarp();
    acc0[0] = s;
  } else {
    const bool v0 = lane < m, v1 = lane + 32 < m;
    add_bias<NRHS>(p, T, acc0, acc1, lane);
    for (int col = 0; col < T.ncols; col += kCols) {
      const int cc = min(kCols, T.ncols - col);
      const double* Ac = A + (int64_t)col * ld;
      // global path: issue the first U columns before gathering the sources
      const int np = SMEM ? 0 : min(U, cc);
      double a0[U], a1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a0[u] = (u < np && v0) ? ld_stream(Ac + (int64_t)u * ld + lane) : 0.0;
        a1[u] = (u < np && v1) ? ld_stream(Ac + (int64_t)u * ld + lane + 32) : 0.0;
      }
      gather_chunk<NRHS>(p, w, lane, col, cc);
      __syncwarp();
      if (p.trace && col == 0 && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(w.dbg[1])::"memory");
      if (SMEM && col == 0) mbar_wait(bar, parity);
      if (p.trace && col == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_gath)::"memory");
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (u < np) {
#pragma unroll
          for (int r = 0; r < NRHS; ++r) {
            const double xv = w.xs[u * NRHS + r];
            acc0[r] = fma(a0[u], xv, acc0[r]);
            acc1[r] = fma(a1[u], xv, acc1[r]);
          }
        }
      }
      int c = np;
      for (; c + U <= cc; c += U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          a0[u] = v0 ? ldA<SMEM>(Ac + (int64_t)(c + u) * ld + lane) : 0.0;
          a1[u] = v1 ? ldA<SMEM>(Ac + (int64_t)(c + u) * ld + lane + 32) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int r = 0; r < NRHS; ++r) {
            const double xv = w.xs[(c + u) * NRHS + r];
            acc0[r] = fma(a0[u], xv, acc0[r]);
            acc1[r] = fma(a1[u], xv, acc1[r]);
          }
        }
      }
      for (; c < cc; ++c) {
        const double b0 = v0 ? ldA<SMEM>(Ac + (int64_t)c * ld + lane) : 0.0;
        const double b1 = v1 ? ldA<SMEM>(Ac + (int64_t)c * ld + lane + 32) : 0.0;
#pragma unroll
        for (int r = 0; r < NRHS; ++r) {
          const double xv = w.xs[c * NRHS + r];
          acc0[r] = fma(b0, xv, acc0[r]);
          acc1[r] = fma(b1, xv, acc1[r]);
        }
      }
      __syncwarp();
    }
  }

  if (p.trace && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(w.dbg[2])::"memory");
  store_rows<NRHS>(p, T, acc0, acc1, lane);
}


template <int NRHS, int MT>
__device__ __forceinline__ void mma_epilogue(const KParams& p, const DTask& T, double (&acc)[MT][NRHS / 8][4],
                                             int lane, int row0);

// D(16x8) += A(16x4, row) B(4x8, col) in fp64 on the tensor cores (DMMA).
__device__ __forceinline__ void dmma_16x8x4(double (&d)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

// One work item with NRHS = 8 or 16 right-hand sides on the FP64 tensor
// cores: Y(m x NRHS) = A(m x ncols) X(ncols x NRHS) as 16 x 8 x 4 DMMA tiles.
// Lane (g = lane/4, t = lane%4) holds A rows g and g+8 of column t of each
// 16-row tile (eight consecutive doubles per column and tile: coalesced),
// X row t / column g of each 8-column tile from the gathered sources in
// shared memory, and accumulator rows g, g+8 / columns 2t, 2t+1.
template <int NRHS, bool SMEM, int MT = 4>
__device__ __forceinline__ void run_item_mma(const KParams& p, const DTask& T, const DSeg& sin, WarpSmem& w,
                                             int lane, const double* A, uint64_t* bar, unsigned parity,
                                             unsigned long long& t_gath) {
  static_assert(NRHS == 8 || NRHS == 16, "DMMA path: 8 or 16 right-hand sides");
  constexpr int kCols = kChunkBytes / (8 * NRHS);
  constexpr int NT = NRHS / 8;  // 8-column tiles
  // MT 16-row tiles per pass: 4 covers an item (m <= 64) in one pass; the
  // dataflow kernel uses 2 (half the accumulator registers, two CTAs per SM)
  // and runs items of more than 32 rows in two passes over the rows
  const int m = T.m, ld = T.ld;
  const int g = lane >> 2, t = lane & 3;
  load_segtable(p, T, sin, w, lane);
  bool waited = false;
  for (int row0 = 0; row0 < m || row0 == 0; row0 += 16 * MT) {
  const int mtiles = (min(m - row0, 16 * MT) + 15) >> 4;

  double acc[MT][NT][4];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

  for (int col = 0; col < T.ncols; col += kCols) {
    const int cc = min(kCols, T.ncols - col);
    const double* Ac = A + (int64_t)col * ld + row0;
    // A fragments of the first k-step: streamed ones are issued before the
    // gather, staged ones read once the bulk copy has landed
    double a[MT][2];
    auto load_a0 = [&]() {
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int r = 16 * i + g;
        const bool ok = i < mtiles && t < cc;
        a[i][0] = (ok && row0 + r < m) ? ldA<SMEM>(Ac + (int64_t)t * ld + r) : 0.0;
        a[i][1] = (ok && row0 + r + 8 < m) ? ldA<SMEM>(Ac + (int64_t)t * ld + r + 8) : 0.0;
      }
    };
    if (!SMEM) load_a0();
    // (a later pass over the rows of a single-chunk item finds its sources staged)
    if (row0 == 0 || T.ncols > kCols) {
      gather_chunk<NRHS>(p, w, lane, col, cc);
      for (int j = cc * NRHS + lane; j < ((cc + 3) & ~3) * NRHS; j += 32) w.xs[j] = 0.0;  // k padding
    }
    __syncwarp();
    if (SMEM && !waited) {
      mbar_wait(bar, parity);
      waited = true;
    }
    if (SMEM) load_a0();
    if (p.trace && col == 0 && row0 == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_gath)::"memory");
    for (int c = 0; c < cc; c += 4) {
      // next k-step's A fragments in flight while this one multiplies
      double an[MT][2];
      const int cn = c + 4 + t;
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int r = 16 * i + g;
        const bool ok = i < mtiles && cn < cc;
        an[i][0] = (ok && row0 + r < m) ? ldA<SMEM>(Ac + (int64_t)cn * ld + r) : 0.0;
        an[i][1] = (ok && row0 + r + 8 < m) ? ldA<SMEM>(Ac + (int64_t)cn * ld + r + 8) : 0.0;
      }
      double b[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = w.xs[(c + t) * NRHS + 8 * j + g];
#pragma unroll
      for (int i = 0; i < MT; ++i)
        if (i < mtiles)
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma_16x8x4(acc[i][j], a[i][0], a[i][1], b[j]);
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        a[i][0] = an[i][0];
        a[i][1] = an[i][1];
      }
    }
    __syncwarp();
  }

  mma_epilogue<NRHS, MT>(p, T, acc, lane, row0);
  }
}

// Bias slots, then the output rows this lane holds (accumulator rows g, g+8
// of each 16-row tile, columns 2t, 2t+1 of each 8-column tile); the tiles
// cover rows [row0, row0 + 16 MT) of the item.
template <int NRHS, int MT>
__device__ __forceinline__ void mma_epilogue(const KParams& p, const DTask& T, double (&acc)[MT][NRHS / 8][4],
                                             int lane, int row0) {
  constexpr int NT = NRHS / 8;
  const int m = T.m;
  const int mtiles = (min(m - row0, 16 * MT) + 15) >> 4;
  const int g = lane >> 2, t = lane & 3;
  // bias slots (the final items' near-field partials): slots of every row
  // this lane holds in flight at once, added in slot order
  constexpr int QB = (MT >= 4 || NT >= 2) ? 2 : 4;
  if (T.bias >= 0) {
    for (int s = 0; s < T.bias_nslots; s += QB) {
      double2 q[QB][MT][2][NT];
#pragma unroll
      for (int u = 0; u < QB; ++u)
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = row0 + 16 * i + g + 8 * h;
            const bool ok = s + u < T.bias_nslots && i < mtiles && r < m;
            const double* bp = p.coef + (T.bias + (int64_t)(s + u) * T.bias_stride + r) * NRHS + 2 * t;
#pragma unroll
            for (int j = 0; j < NT; ++j)
              q[u][i][h][j] = ok ? __ldcg(reinterpret_cast<const double2*>(bp + 8 * j)) : make_double2(0.0, 0.0);
          }
#pragma unroll
      for (int u = 0; u < QB; ++u)
        if (s + u < T.bias_nslots)
#pragma unroll
          for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int j = 0; j < NT; ++j) {
                acc[i][j][2 * h] += q[u][i][h][j].x;
                acc[i][j][2 * h + 1] += q[u][i][h][j].y;
              }
    }
  }
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    if (i >= mtiles) break;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = row0 + 16 * i + g + 8 * h;
      if (r >= m) continue;
      double2 v[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) v[j] = make_double2(acc[i][j][2 * h], acc[i][j][2 * h + 1]);
      double* dst = T.kind == h2b::kFinal ? p.y + __ldg(p.perm + T.out + r) * NRHS : p.coef + (T.out + r) * NRHS;
#pragma unroll
      for (int j = 0; j < NT; ++j) *reinterpret_cast<double2*>(dst + 8 * j + 2 * t) = v[j];
    }
  }
}

// Sources of one multi-RHS chunk (<= 128 double2 values: 4 per lane),
// split into issue (first slot of each value, loads left in flight in
// registers) and commit (further partial slots in slot order, then the
// store to shared memory), so a chunk's gather overlaps the previous
// chunk's multiplication.  `k` is the lane's segment cursor (columns only
// increase along a lane, across chunks too).
template <int NRHS>
struct GatherBatch {
  double2 v[4];
  const double2* q[4];
  int ns[4];
  int64_t st[4];
};
template <int NRHS>
__device__ __forceinline__ void gather_issue(const KParams& p, const WarpSmem& w, int lane, int col, int cc,
                                             GatherBatch<NRHS>& g, int& k) {
  const int total = cc * NRHS / 2;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int jj = lane + 32 * u;
    g.ns[u] = 0;
    g.v[u] = make_double2(0.0, 0.0);
    if (jj < total) {
      const int j = 2 * jj;
      const int c = col + j / NRHS, r = j % NRHS;
      while (w.seg_off[k + 1] <= c) ++k;
      const int64_t e = (w.seg_src[k] + (c - w.seg_off[k])) * NRHS + r;
      const bool isx = w.seg_kind[k] == h2b::kSegX;
      g.q[u] = reinterpret_cast<const double2*>((isx ? p.xp : p.coef) + e);
      g.ns[u] = isx ? 1 : w.seg_nslots[k];
      g.st[u] = (int64_t)w.seg_stride[k] * NRHS / 2;
      if (g.ns[u] > 0) g.v[u] = isx ? __ldg(g.q[u]) : __ldcg(g.q[u]);
    }
  }
}
template <int NRHS>
__device__ __forceinline__ void gather_commit(GatherBatch<NRHS>& g, int lane, int cc, double* xs) {
  const int total = cc * NRHS / 2;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    for (int s = 1; s < g.ns[u]; ++s) add_to(g.v[u], __ldcg(g.q[u] + (int64_t)s * g.st[u]));
    if (lane + 32 * u < total) reinterpret_cast<double2*>(xs)[lane + 32 * u] = g.v[u];
  }
  for (int j = cc * NRHS + lane; j < ((cc + 3) & ~3) * NRHS; j += 32) xs[j] = 0.0;  // k padding
}

// A streamed multi-RHS item (ld == m <= 64) on the DMMA tiles, its matrix
// moved by TMA bulk copies through the warp's two-stage shared-memory ring:
// chunk j + 2 is in flight while chunk j multiplies, so each warp keeps up
// to 16 KB of the stream outstanding without holding it in registers (the
// register-staged loop above keeps one 4-column k-step in flight, which
// leaves HBM idle).  The sources of chunk j + 1 are gathered into the other
// half of the warp's source buffer while chunk j multiplies.  `rpar` holds
// the ring's mbarrier parities (bit s).
template <int NRHS, int STAGE = kRingStageBytes, int MT = 4>
__device__ __forceinline__ void run_item_mma_ring(const KParams& p, const DTask& T, const DSeg& sin, WarpSmem& w,
                                                  const WarpRing R, unsigned& rpar, int lane,
                                                  unsigned long long& t_gath) {
  constexpr int kHalf = kChunkBytes / (16 * NRHS);  // columns per source half (16 or 32)
  constexpr int NT = NRHS / 8;
  const int m = T.m;
  const int g = lane >> 2, t = lane & 3;
  const double* g0 = p.mat + T.data;
  load_segtable(p, T, sin, w, lane);
  // Sources by TMA too when every segment is one contiguous range: x (a
  // node range of xp) or a coefficient vector with a single slot (the x^ of
  // a source cluster): each chunk's sources are bulk-copied into the source
  // half of its stage with the matrix chunk, no register gathers.
  const int nseg = T.seg1 - T.seg0;
  const bool tma_src = __all_sync(0xffffffffu, lane >= nseg || w.seg_kind[lane] == h2b::kSegX ||
                                                   w.seg_nslots[lane] == 1);
  // columns per stage, a whole number of 4-column k-steps so that the DMMA
  // sums group columns exactly like the register-staged loop.  The sources
  // of a chunk sit in the warp's source buffer (two halves of kHalf columns)
  // or, when they come by TMA and the item has few rows, behind the matrix
  // chunk inside the ring stage itself: a 16-row item then moves 32 columns
  // per stage instead of 16 -- half the round trips of the latency-bound far
  // field (ranks are ~16: most up, transfer and coupling items).
  const int stage = R.sdbl * 8 - 32;  // the ring's stage payload (STAGE, or the run-time multi-RHS stage)
  const int cs_buf = min(kHalf, stage / (8 * m)) & ~3;
  const int cs_stage = (p.flags & kFlagMrhsSrcInStage) ? (min(64, stage / (8 * (m + NRHS))) & ~3) : 0;
  const bool src_in_stage = tma_src && cs_stage > cs_buf;
  const int cs = src_in_stage ? cs_stage : cs_buf;
  const int soff = (cs * m + 3) & ~1;  // doubles: behind the chunk (which may start 8 bytes into the stage)
  const int nch = (T.ncols + cs - 1) / cs;
  int kseg_tma = 0;  // lane 0: segment cursor of the TMA source copies
  auto issue = [&](int j) {  // lane 0: chunk j into stage j % 2
    const double* src = g0 + (int64_t)j * cs * m;
    const int cc = min(cs, T.ncols - j * cs);
    const uintptr_t a0 = (uintptr_t)src & ~(uintptr_t)15;
    const uintptr_t a1 = ((uintptr_t)(src + (int64_t)cc * m) + 15) & ~(uintptr_t)15;
    if (!tma_src) {
      ring_load(p, R.buf(j), (const void*)a0, (unsigned)(a1 - a0), R.bar(j));
      return;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect(R.bar(j), (unsigned)(a1 - a0) + (unsigned)(cc * NRHS * 8));
    if (p.flags & kFlagStreamEvictFirst) bulk_copy_hint(R.buf(j), (const void*)a0, (unsigned)(a1 - a0), R.bar(j),
                                                        evict_first_policy());
    else bulk_copy(R.buf(j), (const void*)a0, (unsigned)(a1 - a0), R.bar(j));
    double* xs = src_in_stage ? R.buf(j) + soff : w.xs + (j & 1) * kHalf * NRHS;
    const int col = j * cs;
    int c = col;
    while (c < col + cc) {
      while (w.seg_off[kseg_tma + 1] <= c) ++kseg_tma;
      const int hi = min(col + cc, w.seg_off[kseg_tma + 1]);
      const int64_t e = (w.seg_src[kseg_tma] + (c - w.seg_off[kseg_tma])) * NRHS;
      const double* sp = (w.seg_kind[kseg_tma] == h2b::kSegX ? p.xp : p.coef) + e;
      bulk_copy(xs + (c - col) * NRHS, sp, (unsigned)((hi - c) * NRHS * 8), R.bar(j));
      c = hi;
    }
  };
  if (tma_src && lane == 0) {
    // the coefficients were written by other warps (generic proxy) and
    // acquired by this warp: order them before the async-proxy reads
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  // MT < 4: items of more than 16 MT rows stream once per pass over the rows
  for (int row0 = 0; row0 < m; row0 += 16 * MT) {
  const int mtiles = (min(m - row0, 16 * MT) + 15) >> 4;
  kseg_tma = 0;
  if (lane == 0) {
    issue(0);
    if (nch > 1) issue(1);
  }

  double acc[MT][NT][4];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

  GatherBatch<NRHS> gb;
  int kseg = 0;
  if (!tma_src) {
    gather_issue<NRHS>(p, w, lane, 0, min(cs, T.ncols), gb, kseg);
    gather_commit<NRHS>(gb, lane, min(cs, T.ncols), w.xs);
    __syncwarp();
  }
  for (int jc = 0; jc < nch; ++jc) {
    const int col = jc * cs;
    const int cc = min(cs, T.ncols - col);
    const bool more = jc + 1 < nch;
    const int cc1 = more ? min(cs, T.ncols - col - cs) : 0;
    if (more && !tma_src) gather_issue<NRHS>(p, w, lane, col + cs, cc1, gb, kseg);
    const int s = jc & 1;
    mbar_wait(R.bar(s), (rpar >> s) & 1u);
    rpar ^= 1u << s;
    if (p.trace && jc == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_gath)::"memory");
    const double* A = R.buf(s) + ((((uintptr_t)(g0 + (int64_t)col * m)) & 15) >> 3);
    const double* xs = src_in_stage ? R.buf(s) + soff : w.xs + (jc & 1) * kHalf * NRHS;
    for (int c = 0; c < cc; c += 4) {
      const bool okc = c + t < cc;
      double a[MT][2];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int r = row0 + 16 * i + g;
        const bool ok = okc && i < mtiles;
        a[i][0] = (ok && r < m) ? A[(c + t) * m + r] : 0.0;
        a[i][1] = (ok && r + 8 < m) ? A[(c + t) * m + r + 8] : 0.0;
      }
      double b[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = okc ? xs[(c + t) * NRHS + 8 * j + g] : 0.0;
#pragma unroll
      for (int i = 0; i < MT; ++i)
        if (i < mtiles)
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma_16x8x4(acc[i][j], a[i][0], a[i][1], b[j]);
    }
    __syncwarp();  // every lane is done with stage s and with this source half
    if (lane == 0 && jc + 2 < nch) issue(jc + 2);
    if (more && !tma_src) {
      gather_commit<NRHS>(gb, lane, cc1, w.xs + ((jc + 1) & 1) * kHalf * NRHS);
      __syncwarp();
    }
  }
  mma_epilogue<NRHS, MT>(p, T, acc, lane, row0);
  __syncwarp();
  }
}


// A streamed single-vector item (ld == m, 16 < m <= 64, ncols <= the gather
// capacity) on a ring warp: its matrix moves through the warp's two-stage
// TMA ring (16 KB in flight without registers), the sources are gathered
// once, and every lane runs the same column-ordered FMA chain as run_item,
// so a ring warp's result is bit-identical to a register-streaming warp's.
__device__ __forceinline__ void run_item_ring1(const KParams& p, const DTask& T, const DSeg& sin, WarpSmem& w,
                                               const WarpRing R, unsigned& rpar, int lane,
                                               unsigned long long& t_gath) {
  const int m = T.m;
  const int cs = p.ring_stage / (8 * m);  // columns per stage (>= 8)
  const int nch = (T.ncols + cs - 1) / cs;
  const double* g0 = p.mat + T.data;
  auto issue = [&](int j) {  // lane 0: chunk j into stage j % 2
    const double* src = g0 + (int64_t)j * cs * m;
    const int cc = min(cs, T.ncols - j * cs);
    const uintptr_t a0 = (uintptr_t)src & ~(uintptr_t)15;
    const uintptr_t a1 = ((uintptr_t)(src + (int64_t)cc * m) + 15) & ~(uintptr_t)15;
    ring_load(p, R.buf(j), (const void*)a0, (unsigned)(a1 - a0), R.bar(j));
  };
  if (lane == 0) {
    issue(0);
    if (nch > 1) issue(1);
  }
  load_segtable(p, T, sin, w, lane);
  double acc0[1] = {0.0}, acc1[1] = {0.0};
  add_bias<1>(p, T, acc0, acc1, lane);
  gather_chunk<1>(p, w, lane, 0, T.ncols);
  __syncwarp();
  const bool v0 = lane < m, v1 = lane + 32 < m;
  double s0 = acc0[0], s1 = acc1[0];
  for (int jc = 0; jc < nch; ++jc) {
    const int col = jc * cs;
    const int cc = min(cs, T.ncols - col);
    const int st = jc & 1;
    mbar_wait(R.bar(st), (rpar >> st) & 1u);
    rpar ^= 1u << st;
    if (p.trace && jc == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_gath)::"memory");
    const double* A = R.buf(st) + ((((uintptr_t)(g0 + (int64_t)col * m)) & 15) >> 3);
    const double* xs = w.xs + col;
    int c = 0;
    for (; c + 8 <= cc; c += 8) {
      double a[8], b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a[u] = v0 ? A[(c + u) * m + lane] : 0.0;
        b[u] = v1 ? A[(c + u) * m + lane + 32] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        s0 = fma(a[u], xs[c + u], s0);
        s1 = fma(b[u], xs[c + u], s1);
      }
    }
    for (; c < cc; ++c) {
      const double a = v0 ? A[c * m + lane] : 0.0;
      const double b = v1 ? A[c * m + lane + 32] : 0.0;
      s0 = fma(a, xs[c], s0);
      s1 = fma(b, xs[c], s1);
    }
    __syncwarp();  // every lane is done with stage st
    if (lane == 0 && jc + 2 < nch) issue(jc + 2);
  }
  acc0[0] = s0;
  acc1[0] = s1;
  store_rows<1>(p, T, acc0, acc1, lane);
}


// The same for 2 or 4 right-hand sides: lanes own rows, NRHS accumulators
// each, columns in the order of run_item (bit-identical to it).
template <int NRHS>
__device__ __forceinline__ void run_item_ring_multi(const KParams& p, const DTask& T, const DSeg& sin, WarpSmem& w,
                                                    const WarpRing R, unsigned& rpar, int lane,
                                                    unsigned long long& t_gath) {
  const int m = T.m;
  const int cs = p.ring_stage / (8 * m);  // columns per stage (>= 8)
  const int nch = (T.ncols + cs - 1) / cs;
  const double* g0 = p.mat + T.data;
  auto issue = [&](int j) {  // lane 0: chunk j into stage j % 2
    const double* src = g0 + (int64_t)j * cs * m;
    const int cc = min(cs, T.ncols - j * cs);
    const uintptr_t a0 = (uintptr_t)src & ~(uintptr_t)15;
    const uintptr_t a1 = ((uintptr_t)(src + (int64_t)cc * m) + 15) & ~(uintptr_t)15;
    ring_load(p, R.buf(j), (const void*)a0, (unsigned)(a1 - a0), R.bar(j));
  };
  if (lane == 0) {
    issue(0);
    if (nch > 1) issue(1);
  }
  load_segtable(p, T, sin, w, lane);
  double acc0[NRHS], acc1[NRHS];
#pragma unroll
  for (int r = 0; r < NRHS; ++r) acc0[r] = acc1[r] = 0.0;
  add_bias<NRHS>(p, T, acc0, acc1, lane);
  // sources in windows of the gather capacity (an item may have more
  // columns than fit), each window starting at a stage boundary
  constexpr int kCap = kChunkBytes / (8 * NRHS);
  int wlo = 0, whi = min(kCap, T.ncols);
  gather_chunk<NRHS>(p, w, lane, 0, whi);
  __syncwarp();
  const bool v0 = lane < m, v1 = lane + 32 < m;
  for (int jc = 0; jc < nch; ++jc) {
    const int col = jc * cs;
    const int cc = min(cs, T.ncols - col);
    if (col + cc > whi) {
      wlo = col;
      whi = min(col + kCap, T.ncols);
      gather_chunk<NRHS>(p, w, lane, wlo, whi - wlo);
      __syncwarp();
    }
    const int st = jc & 1;
    mbar_wait(R.bar(st), (rpar >> st) & 1u);
    rpar ^= 1u << st;
    if (p.trace && jc == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_gath)::"memory");
    const double* A = R.buf(st) + ((((uintptr_t)(g0 + (int64_t)col * m)) & 15) >> 3);
    const double* xs = w.xs + (int64_t)(col - wlo) * NRHS;
    int c = 0;
    for (; c + 4 <= cc; c += 4) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = v0 ? A[(c + u) * m + lane] : 0.0;
        b[u] = v1 ? A[(c + u) * m + lane + 32] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int r = 0; r < NRHS; ++r) {
          const double xv = xs[(c + u) * NRHS + r];
          acc0[r] = fma(a[u], xv, acc0[r]);
          acc1[r] = fma(b[u], xv, acc1[r]);
        }
    }
    for (; c < cc; ++c) {
      const double a = v0 ? A[c * m + lane] : 0.0;
      const double b = v1 ? A[c * m + lane + 32] : 0.0;
#pragma unroll
      for (int r = 0; r < NRHS; ++r) {
        const double xv = xs[c * NRHS + r];
        acc0[r] = fma(a, xv, acc0[r]);
        acc1[r] = fma(b, xv, acc1[r]);
      }
    }
    __syncwarp();  // every lane is done with stage st
    if (lane == 0 && jc + 2 < nch) issue(jc + 2);
  }
  store_rows<NRHS>(p, T, acc0, acc1, lane);
}

template <int NRHS>
__global__ void __launch_bounds__(NRHS >= 8 ? kMrhsThreads : 256, NRHS >= 8 ? kMrhsCtas : 2) h2b_dataflow_kernel(KParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  WarpSmem& w = reinterpret_cast<WarpSmem*>(smem_raw)[wib];
  uint64_t* bar = reinterpret_cast<uint64_t*>(&w.bar);
  if (lane == 0) {
    mbar_init(bar);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // staging: a TMA ring (ring warps) or one far-field buffer
  const int nring = NRHS >= 8 ? nw : p.ring_warps;
  const int first_ring = nw - nring;
  const int rstage = NRHS >= 8 ? p.mrhs_stage : p.ring_stage;
  WarpRing ring_v{nullptr, nullptr, 0};
  bool has_ring = false;
  double* abuf;
  unsigned rpar = 0;  // ring stage parities (all lanes)
  bool pdl_waited = false;  // programmatic dependent launch: this warp has waited for the preceding sweep
  int stage_cap = kStageBytes;  // far-field staging capacity (a ring warp: both stages)
  {
    unsigned char* st = smem_raw + (size_t)nw * sizeof(WarpSmem);
    if (wib >= first_ring) {
      unsigned char* rb = st + (size_t)first_ring * kStageBytes + (size_t)(wib - first_ring) * ring_bytes(rstage);
      ring_v.base = reinterpret_cast<double*>(rb);
      ring_v.sdbl = (rstage + 32) / 8;
      ring_v.bars = reinterpret_cast<uint64_t*>(rb + 2 * (rstage + 32));
      has_ring = true;
      abuf = ring_v.base;
      stage_cap = 2 * (rstage + 32);
      if (lane == 0) {
        mbar_init(ring_v.bars);
        mbar_init(ring_v.bars + 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
    } else {
      abuf = reinterpret_cast<double*>(st + (size_t)wib * kStageBytes);
    }
  }
  __syncwarp();
  unsigned phase = 0;  // parity of the staging mbarrier (all lanes)

  // Completion-driven scheduling (lane 0 decides, the warp executes):
  //  0. a successor this warp just completed (continuation: the critical
  //     far-field chain never waits for a queue round trip);
  //  1. a claimed dynamic slot whose push has landed, or a fresh dynamic
  //     claim (the far-field chain and the finals go first);
  //  2. a static item (up-leaf first, then the near field).
  Ctl* ctl = p.ctl;
  const unsigned e1 = ld_relaxed(&ctl->epoch) + 1u;
  const unsigned n_dynamic = (unsigned)(p.nnodes - p.nready0 - p.ngated);
  // lane-0 state below.  The initially-ready items are two static lists
  // claimed through separate heads: up-leaf items ready0[0, nready0_hi) and
  // the near field ready0[nready0_hi, nready0).
  const unsigned n_up = (unsigned)p.nready0_hi, n_near = (unsigned)(p.nready0 - p.nready0_hi);
  bool up_done = n_up == 0;
  bool near_done = n_near == 0;
  // gated coupling rows: claimable once all nup_gate upward items are done
  bool gate_open = p.nup_gate == 0;
  bool g_done1 = p.ngated1 == 0, g_done2 = p.ngated == p.ngated1;
  int owed = -1;             // claimed dynamic slot whose push is still in flight
  int pend = -1;             // near item claimed ahead (slack work, no priority cost)
  int cont = -1;             // continuation (all lanes)
  // warps allowed to take near-field items (fewer loads in flight lower the
  // memory latency the far-field chain sees)
  const int near_lim = (p.flags >> 8) & 0xff;
  // columns in flight per lane for streamed items: enough to cover the
  // bandwidth-latency product, and no more (excess requests only queue)
  const int u_sel = (p.flags >> 16) & 3;
  const int stream_u = u_sel >= 2 ? 4 : 8;
  const bool near_ok = near_lim == 0 || wib < near_lim;
  // leaf coupling rows (class 2) are served before the claimed-ahead near
  // item once this warp has run `leaf_mix` near items in a row (15: always),
  // so the gather-latency-bound downward rows overlap the near-field stream
  // instead of forming a tail after it
  const int leaf_mix = (p.flags >> 20) & 0xf;
  const int leaf_thr = leaf_mix == 15 ? 0 : leaf_mix;
  int near_run = 0;  // lane-0 state: near items run since the last class-2 item
  // the top `near_prio` warps of each CTA stream near items from the start
  // (after the chain queue only), so HBM is busy while the other warps work
  // through the latency-bound upward pass and coupling rows
  const int near_prio = (p.flags >> 26) & 0xf;
  const bool nprio = near_prio > 0 && wib >= nw - near_prio;
  for (;;) {
    int item = cont;
    if (lane == 0 && item < 0) {
      // claim from dynamic queue q (0: critical chain, 1: slack) given the
      // probed head/tail; returns the item, or -1 (with `owed` set when the
      // claimed slot is still in flight)
      auto claim = [&](int q) -> int {
        unsigned* head = &ctl->head[q].v;
        // one atomicAdd per claim (CAS retry loops serialise contending warps)
        const unsigned slot = atomicAdd(head, 1u);
        if (slot >= n_dynamic) return -1;
        const unsigned abs = (unsigned)q * (unsigned)p.ntasks + slot;
        // the pusher bumped the tail first and publishes the id a few
        // instructions later: wait briefly before parking the claim
        for (int spin = 0; spin < 64; ++spin) {
          if (ld_acquire(p.ready_flag + abs) == e1) {
            atomicAdd(&ctl->dyn_started, 1u);
            return __ldcg(p.ready_q + abs);
          }
          __nanosleep(32);
        }
        owed = (int)abs;
        return -1;
      };
      auto take_up = [&]() -> int {
        const unsigned s = atomicAdd(&ctl->static_head, 1u);
        if (s >= n_up) {
          up_done = true;
          return -1;
        }
        return __ldg(p.ready0 + s);
      };
      auto take_g = [&](int q) -> int {  // gated list q (1: inner rows, 2: leaf rows)
        if (q == 1 ? g_done1 : g_done2) return -1;
        if (!gate_open) {
          if (ld_acquire(&ctl->gate.v) < (unsigned)p.nup_gate) return -1;
          gate_open = true;
        }
        const unsigned n = q == 1 ? (unsigned)p.ngated1 : (unsigned)(p.ngated - p.ngated1);
        const unsigned s = atomicAdd(&ctl->g_head[q - 1].v, 1u);
        if (s >= n) {
          (q == 1 ? g_done1 : g_done2) = true;
          return -1;
        }
        return __ldg(p.gated + (q == 1 ? 0 : p.ngated1) + s);
      };
      auto take_near = [&]() -> int {
        const unsigned s = atomicAdd(&ctl->near_head, 1u);
        if (s >= n_near) {
          near_done = true;
          return -1;
        }
        return __ldg(p.ready0 + n_up + s);
      };
      unsigned backoff = 64;
      for (;;) {
        // probe both queues in one round trip
        unsigned h[kQueues], t[kQueues];
#pragma unroll
        for (int q = 0; q < kQueues; ++q) {
          h[q] = ld_relaxed(&ctl->head[q].v);
          t[q] = ld_relaxed(&ctl->tail[q].v);
        }
        if (owed >= 0) {
          if (ld_relaxed(p.ready_flag + owed) == e1) {
            ld_acquire(p.ready_flag + owed);
            item = __ldcg(p.ready_q + owed);
            owed = -1;
            atomicAdd(&ctl->dyn_started, 1u);
            break;
          }
        } else if (h[0] < t[0] && !(nprio && (p.flags & kFlagPrioNoChain)) && (item = claim(0)) >= 0) {
          break;
        }
        if (nprio) {
          // near-priority warps apply the leaf mix too: otherwise the leaf
          // coupling rows wait for the other warps and trail the near field
          // (with kFlagMixInner the coupling rows of inner clusters first:
          // they gate the downward chain)
          // (with kFlagUpMix the up-leaf items first: the upward pass gates
          // every coupling row, and on large operators the few other warps
          // drain it slowly)
          if (leaf_mix && near_run >= leaf_thr && (p.flags & kFlagUpMix) && !up_done && (item = take_up()) >= 0) {
            near_run = 0;
            break;
          }
          if (leaf_mix && near_run >= leaf_thr && owed < 0 && (p.flags & kFlagMixInner) &&
              ((h[1] < t[1] && (item = claim(1)) >= 0) || (item = take_g(1)) >= 0)) {
            near_run = 0;
            break;
          }
          if (leaf_mix && near_run >= leaf_thr && owed < 0 &&
              ((h[2] < t[2] && (item = claim(2)) >= 0) || (item = take_g(2)) >= 0)) {
            near_run = 0;
            break;
          }
          if (pend >= 0) {
            item = pend;
            pend = -1;
            ++near_run;
            break;
          }
          if (!near_done && near_ok && (item = take_near()) >= 0) {
            ++near_run;
            break;
          }
        }
        // class-0 static items (up-leaf) before any slack work
        if (!up_done && near_ok && (item = take_up()) >= 0) break;
        // coupling rows of inner clusters feed the downward chain level by level
        if ((p.flags & kFlagSlackFirst) && owed < 0 &&
            ((h[1] < t[1] && (item = claim(1)) >= 0) || (item = take_g(1)) >= 0)) break;
        if (leaf_mix && near_run >= leaf_thr && owed < 0 &&
            ((h[2] < t[2] && (item = claim(2)) >= 0) || (item = take_g(2)) >= 0)) {
          near_run = 0;
          break;
        }
        // the near item claimed ahead comes before the slack queue: near
        // items are issued longest first, and a long one must not wait
        if (pend >= 0) {
          item = pend;
          pend = -1;
          ++near_run;
          break;
        }
        // coupling rows of inner clusters: the chain needs them level by level
        if (owed < 0 && h[1] < t[1] && (item = claim(1)) >= 0) break;
        if ((item = take_g(1)) >= 0) break;
        if (owed < 0 && h[2] < t[2] && (item = claim(2)) >= 0) break;
        if ((item = take_g(2)) >= 0) break;
        if (!near_done && near_ok && (item = take_near()) >= 0) {
          ++near_run;
          break;
        }
        // every dynamic item has started (continuations skip the queues, so
        // an over-claimed slot may never be pushed): nothing more will come
        if (ld_relaxed(&ctl->dyn_started) >= n_dynamic && g_done1 && g_done2) {
          owed = -1;
          break;
        }
        // idle while the far-field chain catches up (its lower levels are
        // wide: every warp stays available, polling with backoff)
        __nanosleep(backoff);
        backoff = min(backoff * 2u, 1024u);
      }
    }
    // claim the next near item ahead, so that the next decision costs no
    // atomic round trip (its result is read after this item)
    unsigned ahead = 0xffffffffu;
    if (lane == 0 && item >= 0 && pend < 0 && (up_done || nprio) && !near_done && near_ok)
      ahead = atomicAdd(&ctl->near_head, 1u);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item < 0) break;
    unsigned long long t_start = 0;
    if (p.trace && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    // descriptor, inline segments and successor range in one round trip
    const DTask T = p.tasks[item];
    if ((p.pdl & 2) && !pdl_waited && T.kind != h2b::kNear) {
      // started under the upward sweep (programmatic dependent launch): near
      // items need only xp; anything else reads the sweep's x^
      asm volatile("griddepcontrol.wait;" ::: "memory");
      pdl_waited = true;
    }
    DSeg sin{0, 0, 0, 0, 0};
    if (lane < kInlineSegs) sin = p.seg_inline[(int64_t)item * kInlineSegs + lane];
    const int s0 = __ldg(p.succ0 + item), s1 = __ldg(p.succ0 + item + 1);
    unsigned long long t_desc = 0, t_gath = 0;
    if (p.trace && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_desc) : "r"(T.kind) : "memory");
    // successor list (two entries per lane), fetched now so that its latency
    // hides under the item
    int2 sd_first = make_int2(-1, 0), sd_second = make_int2(-1, 0);
    if (s0 + lane < s1) sd_first = __ldg(p.succ + s0 + lane);
    if (s0 + 32 + lane < s1) sd_second = __ldg(p.succ + s0 + 32 + lane);
    // Far-field items (the latency-critical chain) are staged whole into
    // shared memory by one TMA bulk copy, overlapping the source gather;
    // near-field items stream from global memory.
    int off = -1;
    if (T.kind != h2b::kNear && T.ld == T.m && T.ncols > 0 &&
        !(NRHS >= 8 && (p.flags & kFlagMrhsRingAll) && T.m <= 64)) {
      const double* g0 = p.mat + T.data;
      const uintptr_t a0 = (uintptr_t)g0 & ~(uintptr_t)15;
      const uintptr_t a1 = ((uintptr_t)(g0 + (size_t)T.m * T.ncols) + 15) & ~(uintptr_t)15;
      if (a1 - a0 <= (uintptr_t)stage_cap) {
        if (lane == 0) bulk_load(abuf, (const void*)a0, (unsigned)(a1 - a0), bar);
        off = (int)(((uintptr_t)g0 - a0) >> 3);
      }
    }
    if constexpr (NRHS >= 8) {
      if (off >= 0) {
        run_item_mma<NRHS, true, kMrhsMT>(p, T, sin, w, lane, abuf + off, bar, phase, t_gath);
        phase ^= 1u;
      } else if (T.ld == T.m && T.m <= 64 && T.ncols > 0 && !(p.flags & kFlagNoRing)) {  // all warps ring
        run_item_mma_ring<NRHS, kMrhsStage, kMrhsMT>(p, T, sin, w, ring_v, rpar, lane, t_gath);
      } else {
        run_item_mma<NRHS, false, kMrhsMT>(p, T, sin, w, lane, p.mat + T.data, bar, phase, t_gath);
      }
    } else if (off >= 0) {
      run_item<NRHS, true, 16>(p, T, sin, w, lane, abuf + off, bar, phase, t_gath);
      phase ^= 1u;
    } else if (NRHS == 1 && has_ring && T.ld == T.m && T.m > 16 && T.m <= 64 && T.ncols > 0 &&
               T.ncols <= kChunkBytes / 8) {
      run_item_ring1(p, T, sin, w, ring_v, rpar, lane, t_gath);
    } else if ((NRHS == 2 || NRHS == 4) && has_ring && T.ld == T.m && T.m > 16 && T.m <= 64 && T.ncols > 0 &&
               !(p.flags & kFlagNoRing)) {
      if constexpr (NRHS == 2 || NRHS == 4) run_item_ring_multi<NRHS>(p, T, sin, w, ring_v, rpar, lane, t_gath);
    } else if (stream_u == 4) {
      run_item<NRHS, false, 4>(p, T, sin, w, lane, p.mat + T.data, bar, phase, t_gath);
    } else {
      run_item<NRHS, false, 8>(p, T, sin, w, lane, p.mat + T.data, bar, phase, t_gath);
    }
    // publish: outputs visible GPU-wide, then count this item into each
    // successor.  Of the successors whose count this warp completes, it runs
    // the first one itself next and pushes the others.
    __syncwarp();
    if (p.ngated > 0 && T.kind <= h2b::kUpNode && lane == 0)
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&ctl->gate.v) : "memory");
    unsigned long long t_run = 0;
    if (p.trace && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_run));
    cont = -1;
    for (int k0 = s0; k0 < s1; k0 += 128) {
      // arrival counts of up to 4 x 32 successors in flight at once
      int dd[4], qq[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + 32 * u + lane;
        dd[u] = -1;
        qq[u] = 0;
        if (k < s1) {
          const int2 sd = (k0 == s0 && u == 0) ? sd_first
                          : (k0 == s0 && u == 1) ? sd_second : __ldg(p.succ + k);
          const unsigned ndep = (unsigned)sd.y & 0xffffffu;
          const unsigned long long old = (p.flags & kFlagReleaseArrivals) ? atom_add_release(p.arrived + sd.x, 1ull)
                                                                          : atom_add_acq_rel(p.arrived + sd.x, 1ull);
          if (old + 1ull == (unsigned long long)e1 * ndep) dd[u] = sd.x;
          qq[u] = sd.y >> 24;
        }
      }
      // of the successors this warp completed, run one itself next (chain
      // class first) and push the others: one fence, one tail atomic per queue
      unsigned any = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) any |= __ballot_sync(0xffffffffu, dd[u] >= 0);
      if (!any) continue;
      // release-only arrivals: the warp that completes a successor acquires
      // the other producers' outputs here (acquire pattern: the atomic's
      // read, then a fence), before running or publishing it
      if (p.flags & kFlagReleaseArrivals) fence_acq_rel();
      if (cont < 0) {
#pragma unroll
        for (int pass = 0; pass < 2; ++pass)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const unsigned cand = __ballot_sync(0xffffffffu, dd[u] >= 0 && (pass == 1 || qq[u] == 0));
            if (cont < 0 && cand) {
              const int first = __ffs(cand) - 1;
              cont = __shfl_sync(0xffffffffu, dd[u], first);
              if (lane == first) dd[u] = -1;
            }
          }
      }
      unsigned cnt[kQueues], mask[4][kQueues];
#pragma unroll
      for (int q = 0; q < kQueues; ++q) cnt[q] = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < kQueues; ++q) {
          mask[u][q] = __ballot_sync(0xffffffffu, dd[u] >= 0 && qq[u] == q);
          cnt[q] += __popc(mask[u][q]);
        }
      if (cnt[0] + cnt[1] + cnt[2] == 0) continue;
      unsigned base = 0;
      if (lane < kQueues && cnt[lane] > 0) base = atomicAdd(&ctl->tail[lane].v, cnt[lane]);
      unsigned b[kQueues];
#pragma unroll
      for (int q = 0; q < kQueues; ++q) b[q] = __shfl_sync(0xffffffffu, base, q);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (dd[u] >= 0) {
          const int q = qq[u];
          const unsigned slot = (unsigned)q * (unsigned)p.ntasks + b[q] + __popc(mask[u][q] & ((1u << lane) - 1u));
          p.ready_q[slot] = dd[u];
          st_release(p.ready_flag + slot, e1);
        }
#pragma unroll
        for (int q = 0; q < kQueues; ++q) b[q] += __popc(mask[u][q]);
      }
    }
    if (lane == 0 && ahead != 0xffffffffu) {
      if (ahead < n_near) pend = __ldg(p.ready0 + n_up + ahead);
      else near_done = true;
    }
    if (p.trace && lane == 0) {
      unsigned long long t_end, smid;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      asm volatile("mov.u32 %0, %%smid;" : "=r"(*(unsigned*)&smid));
      smid &= 0xffffffffull;
      unsigned long long* tr = p.trace + 8 * (int64_t)item;
      tr[0] = t_start;
      tr[1] = t_end;
      tr[2] = (smid << 32) | (unsigned)(blockIdx.x * nw + wib);
      tr[3] = (unsigned long long)(cont >= 0 ? cont + 1 : 0);
      tr[4] = t_run;
      tr[5] = t_desc;
      tr[6] = t_gath;
    }
    if (cont >= 0 && lane == 0) atomicAdd(&ctl->dyn_started, 1u);
    __syncwarp();
  }
  if (lane == 0) {
    const unsigned total = gridDim.x * (unsigned)nw;
    fence_acq_rel();
    if (atomicAdd(&ctl->exited, 1u) == total - 1) {
      // every warp has left the loop: reset the counters for the next launch
#pragma unroll
      for (int q = 0; q < kQueues; ++q) ctl->head[q].v = ctl->tail[q].v = 0;
      ctl->static_head = 0;
      ctl->near_head = 0;
      ctl->dyn_started = 0;
      ctl->exited = 0;
      ctl->gate.v = 0;
      ctl->g_head[0].v = ctl->g_head[1].v = 0;
      fence_acq_rel();
      atomicAdd(&ctl->epoch, 1u);
    }
  }
}

// Near-field stage of the multi-RHS near kernel: kNearCols columns of the
// item's matrix (<= 64 rows, column-major) and the same columns' sources
// (rows of xp, NRHS doubles each) -- both moved by TMA bulk copies into one
// stage, completing one mbarrier.
constexpr int kNearCols = 16;
template <int NRHS>
struct NearStage {
  static constexpr int kA = kNearCols * 64 * 8 + 32;          // matrix chunk (+ 16-byte rounding)
  static constexpr int kX = kNearCols * NRHS * 8;             // source rows
  static constexpr int kBytes = (kA + kX + 127) / 128 * 128;
};
template <int NRHS>
__host__ __device__ constexpr int near_warp_smem(int nst) {
  return (int)((sizeof(WarpSmem) + 127) / 128 * 128) + nst * NearStage<NRHS>::kBytes + 128;
}

// One near item (ld == m <= 64, x segments only) with NRHS = 8 or 16: per
// stage one bulk copy of the matrix chunk and one per source segment piece
// (a near segment is a contiguous range of xp: the nodes of a source leaf,
// node-major), NST stages in flight, DMMA tiles over the staged operands.
// The k-steps group columns exactly like run_item_mma(_ring): same bits.
template <int NRHS, int NST>
__device__ __forceinline__ void run_near_tma(const KParams& p, const DTask& T, const DSeg& sin, WarpSmem& w,
                                             unsigned char* stages, uint64_t* bars, unsigned& par, int lane,
                                             uint64_t pol) {
  using S = NearStage<NRHS>;
  constexpr int NT = NRHS / 8;
  constexpr int MT = 4;
  const int m = T.m;
  const int mtiles = (m + 15) >> 4;
  const int g = lane >> 2, t = lane & 3;
  const int nch = (T.ncols + kNearCols - 1) / kNearCols;
  const double* g0 = p.mat + T.data;
  int kseg = 0;  // lane 0: segment cursor (chunks are issued in column order)
  auto issue = [&](int j) {  // lane 0
    unsigned char* st = stages + (j % NST) * S::kBytes;
    uint64_t* bar = bars + (j % NST);
    const int col = j * kNearCols;
    const int cc = min(kNearCols, T.ncols - col);
    const double* src = g0 + (int64_t)col * m;
    const uintptr_t a0 = (uintptr_t)src & ~(uintptr_t)15;
    const uintptr_t a1 = ((uintptr_t)(src + (int64_t)cc * m) + 15) & ~(uintptr_t)15;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of this stage are done
    mbar_expect(bar, (unsigned)(a1 - a0) + (unsigned)(cc * NRHS * 8));
    bulk_copy_hint(st, (const void*)a0, (unsigned)(a1 - a0), bar, pol);
    double* xs = reinterpret_cast<double*>(st + S::kA);
    int c = col;
    while (c < col + cc) {
      while (w.seg_off[kseg + 1] <= c) ++kseg;
      const int hi = min(col + cc, w.seg_off[kseg + 1]);
      const int64_t e = (w.seg_src[kseg] + (c - w.seg_off[kseg])) * NRHS;
      bulk_copy(xs + (c - col) * NRHS, p.xp + e, (unsigned)((hi - c) * NRHS * 8), bar);
      c = hi;
    }
  };
  load_segtable(p, T, sin, w, lane);
  if (lane == 0)
    for (int j = 0; j < NST && j < nch; ++j) issue(j);

  double acc[MT][NT][4];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

  for (int jc = 0; jc < nch; ++jc) {
    const int s = jc % NST;
    const int col = jc * kNearCols;
    const int cc = min(kNearCols, T.ncols - col);
    mbar_wait(bars + s, (par >> s) & 1u);
    par ^= 1u << s;
    const unsigned char* st = stages + s * S::kBytes;
    const double* A = reinterpret_cast<const double*>(st) + ((((uintptr_t)(g0 + (int64_t)col * m)) & 15) >> 3);
    const double* xs = reinterpret_cast<const double*>(st + S::kA);
    for (int c = 0; c < cc; c += 4) {
      const bool okc = c + t < cc;
      double a[MT][2];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int r = 16 * i + g;
        const bool ok = okc && i < mtiles;
        a[i][0] = (ok && r < m) ? A[(c + t) * m + r] : 0.0;
        a[i][1] = (ok && r + 8 < m) ? A[(c + t) * m + r + 8] : 0.0;
      }
      double b[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = okc ? xs[(c + t) * NRHS + 8 * j + g] : 0.0;
#pragma unroll
      for (int i = 0; i < MT; ++i)
        if (i < mtiles)
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma_16x8x4(acc[i][j], a[i][0], a[i][1], b[j]);
    }
    __syncwarp();  // every lane is done with stage s
    if (lane == 0 && jc + NST < nch) issue(jc + NST);
  }
  mma_epilogue<NRHS, MT>(p, T, acc, lane, 0);
}

// The near field of a multi-RHS product (8 or 16 right-hand sides) on its
// own: near items have no inputs but x, so this lean kernel needs none of
// the dataflow kernel's scheduling -- warps claim items (longest first) from
// one counter and stream each through a TMA ring onto the DMMA tiles
// (run_item_mma_ring), writing the items' partial slots.  Small code and
// register footprint; the dataflow kernel then runs the rest of the product
// (Plan::ph_split).  STAGE: ring stage bytes (8 KB: 8 warps per SM; 4 KB:
// 16 warps per SM, the same bytes in flight).
template <int NRHS, int STAGE>
__global__ void __launch_bounds__(256, STAGE <= 4096 ? 2 : 1) h2b_near_kernel(KParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  WarpSmem& w = reinterpret_cast<WarpSmem*>(smem_raw)[wib];
  unsigned char* rb = smem_raw + (size_t)nw * sizeof(WarpSmem) + (size_t)wib * ring_bytes(STAGE);
  WarpRing ring{reinterpret_cast<double*>(rb), reinterpret_cast<uint64_t*>(rb + 2 * (STAGE + 32)),
                (STAGE + 32) / 8};
  if (lane == 0) {
    mbar_init(ring.bars);
    mbar_init(ring.bars + 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  unsigned rpar = 0;
  unsigned long long t_gath = 0;
  for (;;) {
    int item = -1;
    if (lane == 0) {
      const unsigned s = atomicAdd(&p.ctl->near_head, 1u);
      if (s < (unsigned)p.nready0) item = __ldg(p.ready0 + s);
    }
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item < 0) break;
    const DTask T = p.tasks[item];
    DSeg sin{0, 0, 0, 0, 0};
    if (lane < kInlineSegs) sin = p.seg_inline[(int64_t)item * kInlineSegs + lane];
    if (T.ld == T.m && T.m <= 64 && T.ncols > 0) {
      run_item_mma_ring<NRHS, STAGE>(p, T, sin, w, ring, rpar, lane, t_gath);
    } else {
      uint64_t* bar = reinterpret_cast<uint64_t*>(&w.bar);
      run_item_mma<NRHS, false>(p, T, sin, w, lane, p.mat + T.data, bar, 0u, t_gath);
    }
    __syncwarp();
  }
}

// The same work with both operands moved by TMA (run_near_tma): no source
// gathers through registers, so the L2 round trip of the sources is off the
// per-chunk critical path.  NST stages of (matrix chunk + sources) per warp.
template <int NRHS, int NST>
__global__ void __launch_bounds__(256, 1) h2b_near_tma_kernel(KParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char* mine = smem_raw + (size_t)wib * near_warp_smem<NRHS>(NST);
  WarpSmem& w = *reinterpret_cast<WarpSmem*>(mine);
  unsigned char* stages = mine + (sizeof(WarpSmem) + 127) / 128 * 128;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + NST * NearStage<NRHS>::kBytes);
  if (lane == 0) {
    for (int s = 0; s < NST; ++s) mbar_init(bars + s);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uint64_t pol = evict_first_policy();
  unsigned par = 0;
  unsigned long long t_gath = 0;
  for (;;) {
    int item = -1;
    if (lane == 0) {
      const unsigned s = atomicAdd(&p.ctl->near_head, 1u);
      if (s < (unsigned)p.nready0) item = __ldg(p.ready0 + s);
    }
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item < 0) break;
    const DTask T = p.tasks[item];
    DSeg sin{0, 0, 0, 0, 0};
    if (lane < kInlineSegs) sin = p.seg_inline[(int64_t)item * kInlineSegs + lane];
    if (T.ld == T.m && T.m <= 64 && T.ncols > 0) {
      run_near_tma<NRHS, NST>(p, T, sin, w, stages, bars, par, lane, pol);
    } else {
      uint64_t* bar = reinterpret_cast<uint64_t*>(&w.bar);
      run_item_mma<NRHS, false>(p, T, sin, w, lane, p.mat + T.data, bar, 0u, t_gath);
    }
    __syncwarp();
  }
}


// A sweep (Phase::mode 1): the far-field items of the bottom
// subtrees of the cluster tree -- the leaf forward transforms and the upward
// transfers below a subtree's root (h2.py:195-209), or the downward
// transfers below it and the leaf back-transforms with the near-field
// partial sums (h2.py:220-244).  One CTA runs a subtree: the items of a
// tree level (a "wave") spread over its warps, a block barrier between
// waves -- the links of the far-field chain inside a subtree cost a
// __syncthreads instead of an arrival count, a queue push and a claim.
// Every input from outside the subtree was written by an earlier launch.
// A warp stages its items' matrices through two shared-memory buffers by TMA
// bulk copies and prefetches its next item's matrix (same or next wave)
// while the current one runs.
constexpr int kSweepStage = 4096 + 32;  // one staged matrix (+ 16-byte alignment slack)
inline size_t sweep_smem_bytes(int nw) { return (size_t)nw * (sizeof(WarpSmem) + ring_bytes(4096)) + 128; }

__device__ __forceinline__ DTask load_task(const DTask* t) {
  // read-only path: the line was prefetched while earlier items ran
  union { DTask T; int4 q[4]; } u;
#pragma unroll
  for (int i = 0; i < 4; ++i) u.q[i] = __ldg(reinterpret_cast<const int4*>(t) + i);
  return u.T;
}
__device__ __forceinline__ void prefetch_l1(const void* q) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(q));
}
__device__ __forceinline__ void prefetch_l2(const void* q) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
}

// The generic sweep: units are claimed from one counter; a warp stages its
// items' matrices through two shared-memory buffers by TMA bulk copies and
// prefetches its next item's matrix (same or a later wave of the unit) while
// the current one runs.  Used when a unit's inputs do not fit shared memory
// (large subtrees, many right-hand sides); see the resident kernel below.
template <int NRHS>
__global__ void __launch_bounds__(256, NRHS >= 8 ? kMrhsSweepCtas : 2) h2b_sweep_kernel(KParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  // (H2B_PDL) the next launch may start now: its near field needs nothing from this sweep
  if (p.pdl & 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  WarpSmem& w = reinterpret_cast<WarpSmem*>(smem_raw)[wib];
  unsigned char* rb = smem_raw + (size_t)nw * sizeof(WarpSmem) + (size_t)wib * ring_bytes(4096);
  double* buf[2] = {reinterpret_cast<double*>(rb), reinterpret_cast<double*>(rb + kSweepStage)};
  uint64_t* bars = reinterpret_cast<uint64_t*>(rb + 2 * kSweepStage);
  uint64_t* wbar = reinterpret_cast<uint64_t*>(&w.bar);
  int* next_unit = reinterpret_cast<int*>(smem_raw + (size_t)nw * (sizeof(WarpSmem) + ring_bytes(4096)));
  if (lane == 0) {
    mbar_init(bars);
    mbar_init(bars + 1);
    mbar_init(wbar);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  Ctl* ctl = p.ctl;
  // the next unit is claimed while the current one runs; the last CTA to
  // leave resets the counter for the next launch
  if (threadIdx.x == 0) next_unit[0] = (int)atomicAdd(&ctl->static_head, 1u);
  __syncthreads();
  unsigned par = 0;   // parities of the two staging mbarriers (bit s)
  int cur = 0;        // staging buffer of the next item
  // bytes of an item's matrix rounded out to 16-byte boundaries, or 0 when
  // it is not one contiguous block
  auto span = [&](const DTask& T, uintptr_t& a0) -> unsigned {
    if (T.ld != T.m || T.ncols <= 0) return 0u;
    const double* g0 = p.mat + T.data;
    a0 = (uintptr_t)g0 & ~(uintptr_t)15;
    const uintptr_t a1 = ((uintptr_t)(g0 + (size_t)T.m * T.ncols) + 15) & ~(uintptr_t)15;
    return (unsigned)(a1 - a0);
  };
  unsigned long long t_gath = 0;
  for (int k = 0;; ++k) {
    const int u = next_unit[k & 1];
    if (u >= p.nunits) break;
    if (threadIdx.x == 0) next_unit[(k + 1) & 1] = (int)atomicAdd(&ctl->static_head, 1u);
    const int wv0 = __ldg(p.unit0 + u), wv1 = __ldg(p.unit0 + u + 1);
    // this warp's items in order: (wave, item), item = wave begin + warp, + nw, ...
    auto first_from = [&](int wv, int& item) -> int {  // first wave >= wv holding an item of this warp
      for (; wv < wv1; ++wv) {
        item = __ldg(p.wave0 + wv) + wib;
        if (item < __ldg(p.wave0 + wv + 1)) return wv;
      }
      item = -1;
      return wv1;
    };
    auto advance = [&](int wv, int item, int& nitem) -> int {
      nitem = item + nw;
      if (nitem < __ldg(p.wave0 + wv + 1)) return wv;
      return first_from(wv + 1, nitem);
    };
    int item, nx, nx2;
    int wv_i = first_from(wv0, item);
    int wv_n = wv1, wv_n2 = wv1;
    nx = nx2 = -1;
    if (item >= 0) wv_n = advance(wv_i, item, nx);
    if (nx >= 0) wv_n2 = advance(wv_n, nx, nx2);
    // prefetched matrix of `item`: staging mode (0: none yet) and offset
    int pf_mode = 0, pf_off = 0;
    if (nx >= 0) {
      prefetch_l1(p.tasks + nx);
      prefetch_l1(p.seg_inline + (int64_t)nx * kInlineSegs);
    }
    for (int wv = wv0; wv < wv1; ++wv) {
      while (item >= 0 && wv_i == wv) {
        unsigned long long t_start = 0;
        if (p.trace && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
        const DTask T = load_task(p.tasks + item);
        DSeg sin{0, 0, 0, 0, 0};
        if (lane < kInlineSegs) sin = p.seg_inline[(int64_t)item * kInlineSegs + lane];
        // this item's matrix: prefetched, staged now (one buffer, or both
        // when it is larger), or streamed from global memory
        int mode = pf_mode, off = pf_off;  // 1: staged in buf[cur], 2: across both buffers
        if (mode == 0) {
          uintptr_t a0 = 0;
          const unsigned bytes = span(T, a0);
          if (bytes > 0 && bytes <= 2u * kSweepStage) {
            mode = bytes <= (unsigned)kSweepStage ? 1 : 2;
            if (mode == 2) cur = 0;  // nothing is in flight: both buffers are free
            if (lane == 0) bulk_load(buf[cur], (const void*)a0, bytes, bars + cur);
            off = (int)(((uintptr_t)(p.mat + T.data) - a0) >> 3);
          }
        }
        // the warp's next item: its matrix into the other buffer while this
        // one runs, and the descriptor after that towards L1
        pf_mode = 0;
        if (nx >= 0) {
          const DTask N = load_task(p.tasks + nx);
          // the next item's inputs that earlier launches left in DRAM, towards
          // L2 while this item runs: its bias slots (near-field partial sums,
          // coupling sums), the finals' permutation entries, its range of x.
          // Otherwise the item pays them as dependent misses, one after the
          // other (bias, sources, permutation).
          if (p.sweep_prefetch) {
            const int rl = (N.m * NRHS * 8 + 127) / 128 + 1;
            if ((p.sweep_prefetch & 2) && N.bias >= 0 && lane < rl) {
              const int ns = min(N.bias_nslots, 32);
              for (int s2 = 0; s2 < ns; ++s2)
                prefetch_l2(p.coef + (N.bias + (int64_t)s2 * N.bias_stride) * NRHS + lane * 16);
            }
            if ((p.sweep_prefetch & 4) && N.kind == h2b::kFinal && lane < (N.m * 8 + 127) / 128 + 1) prefetch_l2(p.perm + N.out + lane * 16);
            if ((p.sweep_prefetch & 1) && lane < kInlineSegs && lane < N.seg1 - N.seg0 && N.seg1 - N.seg0 <= kInlineSegs) {
              const DSeg ns = p.seg_inline[(int64_t)nx * kInlineSegs + lane];
              if (ns.kind == h2b::kSegX)
                for (int o = 0; o < ns.ncols * NRHS + 15; o += 16) prefetch_l2(p.xp + ns.src * NRHS + o);
            }
          }
          if (mode == 1) {
            uintptr_t n0 = 0;
            const unsigned nb = span(N, n0);
            if (nb > 0 && nb <= (unsigned)kSweepStage) {
              if (lane == 0) bulk_load(buf[cur ^ 1], (const void*)n0, nb, bars + (cur ^ 1));
              pf_mode = 1;
              pf_off = (int)(((uintptr_t)(p.mat + N.data) - n0) >> 3);
            }
          }
          if (nx2 >= 0) {
            prefetch_l1(p.tasks + nx2);
            prefetch_l1(p.seg_inline + (int64_t)nx2 * kInlineSegs);
          }
        }
        const unsigned ph = (par >> cur) & 1u;
        unsigned long long t_desc = 0;
        if (p.trace && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_desc)::"memory");
        if constexpr (NRHS >= 8) {
          if (mode) run_item_mma<NRHS, true, kMrhsMT>(p, T, sin, w, lane, buf[cur] + off, bars + cur, ph, t_gath);
          else run_item_mma<NRHS, false, kMrhsMT>(p, T, sin, w, lane, p.mat + T.data, wbar, 0u, t_gath);
        } else {
          if (mode) run_item<NRHS, true, 16>(p, T, sin, w, lane, buf[cur] + off, bars + cur, ph, t_gath);
          else run_item<NRHS, false, 8>(p, T, sin, w, lane, p.mat + T.data, wbar, 0u, t_gath);
        }
        if (mode) par ^= 1u << cur;
        if (mode == 1) cur ^= 1;
        __syncwarp();
        if (p.trace && lane == 0) {
          unsigned long long t_end, smid;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
          asm volatile("mov.u32 %0, %%smid;" : "=r"(*(unsigned*)&smid));
          smid &= 0xffffffffull;
          unsigned long long* tr = p.trace + 8 * (int64_t)item;
          tr[0] = t_start;
          tr[1] = t_end;
          tr[2] = (smid << 32) | (unsigned)(blockIdx.x * nw + wib);
          tr[3] = w.dbg[0];
          tr[4] = w.dbg[2];
          tr[5] = t_desc;
          tr[6] = t_gath;
          tr[7] = w.dbg[1];
        }
        item = nx;
        wv_i = wv_n;
        nx = nx2;
        wv_n = wv_n2;
        nx2 = -1;
        wv_n2 = wv1;
        if (nx >= 0) wv_n2 = advance(wv_n, nx, nx2);
      }
      __syncthreads();  // the wave's outputs are visible to the CTA's next wave
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(&ctl->exited, 1u) == gridDim.x - 1) {
      ctl->static_head = 0;
      ctl->exited = 0;
      __threadfence();
    }
  }
}

// ---- Resident sweep.  The planner lays a unit's inputs out
// as a few contiguous ranges (Phase::u_range): its matrices in the pool, the
// coefficient slots of its clusters, the near-field partial slots and the
// permutation entries of its leaves (downward) or its range of x (upward),
// and its item descriptors.  The CTA copies all of them into shared memory
// with one batch of TMA bulk copies (one mbarrier), then runs the unit's
// waves entirely from shared memory -- a wave costs a block barrier and
// shared-memory latencies, not a chain of cold DRAM misses per item -- and
// writes x^ (upward; the dataflow launch reads it) or y (finals) to global
// memory.  With two or three CTAs per SM one unit's copies overlap another's
// waves, so the sweep is bound by HBM bandwidth.
constexpr int kSweepXs = 128;  // per-warp source scratch (columns)
struct SweepGeom {
  size_t off_v, off_dt, off_ds, off_xs, off_ctl, total;
};
__host__ __device__ inline SweepGeom sweep_geom(int nrhs, int nw, int cap_mat, int cap_vec, int cap_items) {
  auto up = [](size_t v) { return (v + 127) / 128 * 128; };
  SweepGeom g;
  g.off_v = up((size_t)(cap_mat + 2) * 8);
  g.off_dt = g.off_v + up((size_t)(cap_vec + 16) * 8 * nrhs);
  g.off_ds = g.off_dt + up((size_t)cap_items * sizeof(DTask));
  g.off_xs = g.off_ds + up((size_t)cap_items * kInlineSegs * sizeof(DSeg));
  g.off_ctl = g.off_xs + up((size_t)nw * kSweepXs * 8 * nrhs);
  g.total = g.off_ctl + 128 + 256;
  return g;
}

template <int NRHS>
__global__ void __launch_bounds__(256) h2b_sweep_resident_kernel(KParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  if (p.pdl & 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const SweepGeom G = sweep_geom(NRHS, nw, p.cap_mat, p.cap_vec, p.cap_items);
  double* Msm = reinterpret_cast<double*>(smem_raw);
  double* Vsm = reinterpret_cast<double*>(smem_raw + G.off_v);
  const DTask* DT = reinterpret_cast<const DTask*>(smem_raw + G.off_dt);
  const DSeg* DS = reinterpret_cast<const DSeg*>(smem_raw + G.off_ds);
  double* xs = reinterpret_cast<double*>(smem_raw + G.off_xs) + (size_t)wib * kSweepXs * NRHS;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + G.off_ctl);
  // the unit's record (Phase::u_rec) and the next unit's, fetched while this one runs
  int64_t* rec = reinterpret_cast<int64_t*>(smem_raw + G.off_ctl + 128);  // [2][16]
  int* next_unit = reinterpret_cast<int*>(smem_raw + G.off_ctl + 16);
  Ctl* ctl = p.ctl;
  // first unit: the CTA's index; further units from a counter (starting
  // behind the grid), the last CTA to leave resets it
  if (threadIdx.x == 0) {
    mbar_init(bar);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    next_unit[0] = (int)blockIdx.x;
  }
  if (threadIdx.x < 16 && (int)blockIdx.x < p.nunits) rec[threadIdx.x] = __ldg(p.u_range + 16 * (int64_t)blockIdx.x + threadIdx.x);
  __syncthreads();
  unsigned parity = 0;
  for (int k = 0;; ++k) {
    const int u = next_unit[k & 1];
    if (u >= p.nunits) break;
    const int64_t* R = rec + 16 * (k & 1);
    const int k0 = (int)(R[8] & 0xffffffff), nit = (int)(R[8] >> 32);
    const int nwv = (int)R[9];
    const int32_t* wend = reinterpret_cast<const int32_t*>(R + 10);
    // ranges, rounded out to 16-byte boundaries (even element offsets)
    const int64_t m0 = R[0] & ~(int64_t)1, m1 = (R[0] + R[1] + 1) & ~(int64_t)1;
    const int64_t c0 = (R[2] * NRHS) & ~(int64_t)1, c1 = ((R[2] + R[3]) * NRHS + 1) & ~(int64_t)1;
    const int64_t b0 = (R[4] * NRHS) & ~(int64_t)1, b1 = ((R[4] + R[5]) * NRHS + 1) & ~(int64_t)1;
    const int64_t x0 = R[6], xn = R[7];
    // the V area: [C | B | X or perm]
    double* Csm = Vsm;
    double* Bsm = Csm + (c1 - c0) + 2;
    double* Xsm = Bsm + (b1 - b0) + 2;
    const bool up_sweep = (R[9] >> 32) != 0;   // planner: 1 in the high word for an upward unit
    const int64_t xa0 = up_sweep ? (x0 * NRHS) & ~(int64_t)1 : x0 & ~(int64_t)1;
    // diagnostics: unit timeline in the trace slots of its first item
    unsigned long long* tr = p.trace ? p.trace + 8 * (int64_t)k0 : nullptr;
    auto stamp = [&](int j) {
      if (tr && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
        tr[j] = t;
      }
    };
    stamp(0);
    if (threadIdx.x == 0) {
      const int64_t xa1 = up_sweep ? ((x0 + xn) * NRHS + 1) & ~(int64_t)1 : (x0 + xn + 1) & ~(int64_t)1;
      const unsigned bm = (unsigned)((m1 - m0) * 8), bc = (unsigned)((c1 - c0) * 8), bb = (unsigned)((b1 - b0) * 8);
      const unsigned bx = (unsigned)((xa1 - xa0) * 8);
      const unsigned bt = (unsigned)(nit * sizeof(DTask)), bs = (unsigned)(nit * kInlineSegs * sizeof(DSeg));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(bar, bm + bc + bb + bx + bt + bs);
      if (bm) bulk_copy(Msm, p.mat + m0, bm, bar);
      if (bc) bulk_copy(Csm, p.coef + c0, bc, bar);
      if (bb) bulk_copy(Bsm, p.coef + b0, bb, bar);
      if (bx) bulk_copy(Xsm, up_sweep ? (const void*)(p.xp + xa0) : (const void*)(p.perm + xa0), bx, bar);
      bulk_copy(const_cast<DTask*>(DT), p.tasks + k0, bt, bar);
      bulk_copy(const_cast<DSeg*>(DS), p.seg_inline + (int64_t)k0 * kInlineSegs, bs, bar);
      // claim the next unit and fetch its record while this one runs
      const int nu = (int)(atomicAdd(&ctl->static_head, 1u) + gridDim.x);
      next_unit[(k + 1) & 1] = nu;
      if (nu < p.nunits) {
        int64_t* Rn = rec + 16 * ((k + 1) & 1);
#pragma unroll
        for (int j = 0; j < 16; ++j) Rn[j] = __ldg(p.u_range + 16 * (int64_t)nu + j);
      }
    }
    stamp(3);
    mbar_wait(bar, parity);
    parity ^= 1u;
    stamp(4);
    // element (scaled by NRHS) -> pointer: shared memory inside the unit's
    // ranges, global memory (L2) outside
    auto coef_ptr = [&](int64_t e, int64_t span) -> const double* {  // e: scaled offset, span: scaled extent read from it
      if (e >= c0 && e + span <= c1) return Csm + (e - c0);
      if (e >= b0 && e + span <= b1) return Bsm + (e - b0);
      return nullptr;
    };
    int t0 = 0;
    for (int wv = 0; wv < nwv; ++wv) {
      const int t1 = wend[wv];
      for (int it = t0 + wib; it < t1; it += nw) {
        const DTask& T = DT[it];
        const int m = T.m, ld = T.ld, ncols = T.ncols;
        const int nseg = T.seg1 - T.seg0;
        const double* A = Msm + (T.data - m0);
        // lanes: rows rr (and rr + 32 when m > 32); for m <= 16 the columns
        // are split over 32 / m' lane groups and reduced at the end
        int mp = 32;
        if (m <= 16) { mp = 1; while (mp < m) mp <<= 1; }
        const int Gn = 32 / mp, g = lane / mp, rr = lane - g * mp;
        double acc0[NRHS], acc1[NRHS];
#pragma unroll
        for (int r = 0; r < NRHS; ++r) acc0[r] = acc1[r] = 0.0;
        const bool v0 = rr < m, v1 = (mp == 32) && (rr + 32 < m);
        for (int col = 0; col < ncols; col += kSweepXs) {
          const int cc = min(kSweepXs, ncols - col);
          // sources of columns [col, col + cc): slot sums, through the segments
          for (int j = lane; j < cc * NRHS; j += 32) {
            const int c = col + j / NRHS, r = j - (j / NRHS) * NRHS;
            int sbase = 0, sj = 0;
            DSeg S = nseg <= kInlineSegs ? DS[it * kInlineSegs] : p.segs[T.seg0];
            while (sbase + S.ncols <= c) {
              sbase += S.ncols;
              ++sj;
              S = nseg <= kInlineSegs ? DS[it * kInlineSegs + sj] : p.segs[T.seg0 + sj];
            }
            const int64_t e = (S.src + (c - sbase)) * NRHS + r;
            double v = 0.0;
            if (S.kind == h2b::kSegX) {
              v = (up_sweep && S.src >= x0 && S.src + S.ncols <= x0 + xn) ? Xsm[e - xa0] : __ldg(p.xp + e);
            } else {
              const int64_t st = (int64_t)S.stride * NRHS;
              const double* q = coef_ptr(e, (int64_t)(S.nslots - 1) * st + 1);
              if (q) {
                for (int s2 = 0; s2 < S.nslots; ++s2) v += q[(int64_t)s2 * st];
              } else {
                // global (L2): eight slots in flight at a time, added in slot order
                const double* gq = p.coef + e;
                int s2 = 0;
                for (; s2 + 8 <= S.nslots; s2 += 8) {
                  double t8[8];
#pragma unroll
                  for (int i = 0; i < 8; ++i) t8[i] = __ldcg(gq + (int64_t)(s2 + i) * st);
#pragma unroll
                  for (int i = 0; i < 8; ++i) v += t8[i];
                }
                double t8[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) t8[i] = (s2 + i < S.nslots) ? __ldcg(gq + (int64_t)(s2 + i) * st) : 0.0;
#pragma unroll
                for (int i = 0; i < 8; ++i) v += t8[i];
              }
            }
            xs[j] = v;
          }
          __syncwarp();
          // four independent partial sums per row (columns c, c+Gn, c+2Gn,
          // c+3Gn): the loads of a step are in flight together and the FMA
          // chains are a quarter as long
          const double* Ar = A + (int64_t)col * ld + (v0 ? rr : 0);
          const int step = Gn * ld;
          double q0[4][NRHS], q1[4][NRHS];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int r = 0; r < NRHS; ++r) q0[i][r] = q1[i][r] = 0.0;
          int c = g;
          const double* Ap = Ar + (int64_t)g * ld;
          for (; c + 3 * Gn < cc; c += 4 * Gn, Ap += 4 * step) {
            double a0[4], a1[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              a0[i] = Ap[i * step];
              a1[i] = v1 ? Ap[i * step + 32] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int r = 0; r < NRHS; ++r) {
                const double xv = xs[(c + i * Gn) * NRHS + r];
                q0[i][r] = fma(a0[i], xv, q0[i][r]);
                q1[i][r] = fma(a1[i], xv, q1[i][r]);
              }
          }
          for (; c < cc; c += Gn, Ap += step) {
            const double a0 = Ap[0];
            const double a1 = v1 ? Ap[32] : 0.0;
#pragma unroll
            for (int r = 0; r < NRHS; ++r) {
              const double xv = xs[c * NRHS + r];
              q0[0][r] = fma(a0, xv, q0[0][r]);
              q1[0][r] = fma(a1, xv, q1[0][r]);
            }
          }
#pragma unroll
          for (int r = 0; r < NRHS; ++r) {
            acc0[r] += (q0[0][r] + q0[1][r]) + (q0[2][r] + q0[3][r]);
            acc1[r] += (q1[0][r] + q1[1][r]) + (q1[2][r] + q1[3][r]);
          }
          __syncwarp();
        }
        if (!v0) {
#pragma unroll
          for (int r = 0; r < NRHS; ++r) acc0[r] = 0.0;
        }
        if (Gn > 1) {
#pragma unroll
          for (int r = 0; r < NRHS; ++r)
            for (int o = mp; o < 32; o <<= 1) acc0[r] += __shfl_xor_sync(0xffffffffu, acc0[r], o);
        }
        // bias slots (the finals' near-field partial sums), in slot order
        if (T.bias >= 0) {
          for (int s2 = 0; s2 < T.bias_nslots; ++s2) {
            const int64_t e = (T.bias + (int64_t)s2 * T.bias_stride) * NRHS;
            const double* q = coef_ptr(e, (int64_t)m * NRHS);
#pragma unroll
            for (int r = 0; r < NRHS; ++r) {
              if (v0) acc0[r] += q ? q[(int64_t)rr * NRHS + r] : __ldcg(p.coef + e + (int64_t)rr * NRHS + r);
              if (v1) acc1[r] += q ? q[(int64_t)(rr + 32) * NRHS + r] : __ldcg(p.coef + e + (int64_t)(rr + 32) * NRHS + r);
            }
          }
        }
        // outputs: y (finals), or the coefficient slot -- in shared memory for
        // the unit's later waves, and in global memory when a later launch
        // reads it (x^) or it lies outside the unit's range
        if (g == 0) {
          if (T.kind == h2b::kFinal) {
            const int64_t* pm = reinterpret_cast<const int64_t*>(Xsm) + (T.out - xa0);
            const bool in = !up_sweep && T.out >= x0 && T.out + m <= x0 + xn;
            if (v0) {
              const int64_t node = in ? pm[rr] : __ldg(p.perm + T.out + rr);
#pragma unroll
              for (int r = 0; r < NRHS; ++r) p.y[node * NRHS + r] = acc0[r];
            }
            if (v1) {
              const int64_t node = in ? pm[rr + 32] : __ldg(p.perm + T.out + rr + 32);
#pragma unroll
              for (int r = 0; r < NRHS; ++r) p.y[node * NRHS + r] = acc1[r];
            }
          } else {
            const int64_t e = T.out * NRHS;
            double* q = const_cast<double*>(coef_ptr(e, (int64_t)m * NRHS));
            const bool glob = q == nullptr || T.kind <= h2b::kUpNode;
#pragma unroll
            for (int r = 0; r < NRHS; ++r) {
              if (v0) {
                if (q) q[(int64_t)rr * NRHS + r] = acc0[r];
                if (glob) p.coef[e + (int64_t)rr * NRHS + r] = acc0[r];
              }
              if (v1) {
                if (q) q[(int64_t)(rr + 32) * NRHS + r] = acc1[r];
                if (glob) p.coef[e + (int64_t)(rr + 32) * NRHS + r] = acc1[r];
              }
            }
          }
        }
        __syncwarp();
      }
      __syncthreads();  // the wave's outputs are visible to the CTA's next wave
      t0 = t1;
      if (wv < 2) stamp(5 + wv);
      if (wv == nwv - 2) stamp(7);
    }
    stamp(1);
    if (tr && threadIdx.x == 0) tr[2] = ((unsigned long long)nwv << 32) | blockIdx.x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(&ctl->exited, 1u) == gridDim.x - 1) {
      ctl->static_head = 0;
      ctl->exited = 0;
      __threadfence();
    }
  }
}

}  // namespace

namespace h2b_detail {
int set_error(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace h2b_detail

// One kernel launch worth of device state (a Phase of the plan).
struct PhaseDev {
  int64_t ntasks = 0;
  int64_t nnodes = 0;
  DTask* d_tasks = nullptr;
  DSeg* d_segs = nullptr;
  DSeg* d_seg_inline = nullptr;
  int32_t* d_succ0 = nullptr;
  int2* d_succ = nullptr;
  int32_t* d_ready0 = nullptr;
  int32_t nready0 = 0;
  int32_t nready0_hi = 0;
  int32_t* d_gated = nullptr;
  int32_t ngated = 0, ngated1 = 0, nup = 0;
  unsigned long long* d_arrived = nullptr;
  int32_t* d_ready_q = nullptr;
  unsigned* d_ready_flag = nullptr;
  Ctl* d_ctl = nullptr;
  unsigned long long* d_trace = nullptr;
  int mode = 0, group = 0;        // Phase::mode, Phase::group
  int32_t* d_unit0 = nullptr;     // sweeps
  int32_t* d_wave0 = nullptr;
  int32_t nunits = 0;
  int64_t bytes = 0;              // matrix bytes its items stream
  int64_t* d_u_range = nullptr;   // resident sweeps
  bool resident = false;
  int cap_mat = 0, cap_vec = 0, cap_items = 0;
};

// Host threads for the optional staged copies of h2b_matvec
// (H2B_COPY_THREADS > 0): the callers' vectors are pageable numpy arrays
// (apply_operator, compute_demag), which the driver copies through its own
// staging at ~18 GB/s (0.89 ms for the 8.3 MB pair of config 3 against
// 0.32 ms from pinned memory).  With this option chunks are copied by a few
// threads into / out of a pinned buffer and moved by DMA as they become
// ready, so the memcpy and the DMA overlap.  Measured no better than the
// driver's path on the B200 box, hence off by default.
class CopyPool {
 public:
  explicit CopyPool(int nthreads) {
    for (int t = 0; t < nthreads; ++t) workers_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  // fn(i) for i in [0, n): the caller takes part; returns when all are done
  void parallel_for(int n, const std::function<void(int)>& fn) {
    auto job = std::make_shared<Job>();
    job->fn = &fn;
    job->n = n;
    job->pending = n;
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = job;
      ++gen_;
    }
    cv_.notify_all();
    run(*job);
    std::unique_lock<std::mutex> lk(job->mu);
    job->done.wait(lk, [&] { return job->pending == 0; });
  }

 private:
  // one parallel_for: a worker that wakes up late holds an exhausted job
  struct Job {
    const std::function<void(int)>* fn = nullptr;
    int n = 0;
    std::atomic<int> next{0};
    std::mutex mu;
    std::condition_variable done;
    int pending = 0;
  };
  static void run(Job& j) {
    for (;;) {
      const int i = j.next.fetch_add(1);
      if (i >= j.n) return;
      (*j.fn)(i);
      std::lock_guard<std::mutex> lk(j.mu);
      if (--j.pending == 0) j.done.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::shared_ptr<Job> job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        job = job_;
      }
      run(*job);
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::shared_ptr<Job> job_;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

struct h2b_op {
  int device = 0;
  int64_t n = 0;
  int64_t coef_len = 0;
  int max_nrhs = 16;
  int wpc = 8;
  int grid[5] = {0, 0, 0, 0, 0};  // per NRHS template 1,2,4,8,16
  int sweep_grid[5] = {0, 0, 0, 0, 0};
  int sweep_resident = 1;   // H2B_SWEEP_RESIDENT=0: always the generic sweep kernel (A/B switch)
  int smem_optin = 0, nsm = 0;
  double* d_mat = nullptr;
  double* d_coef = nullptr;
  int64_t* d_perm = nullptr;
  double* d_xp = nullptr;  // x in tree order
  int flags = 0;
  int ring_warps = 0;  // NRHS < 8: TMA-ring warps per CTA (sched_flags bits 4-7)
  int sched = 0;       // effective sched_flags (defaults applied)
  int ring_stage = kRingStageBytes;  // NRHS < 8: ring stage payload (sched_flags bits 18-19)
  int mrhs_wpc = 8;                  // 8/16 RHS dataflow launches: warps per CTA (H2B_MRHS_WARPS, <= 12)
  int mrhs_stage = kMrhsStage;       // ... and their ring stage payload (6 KB above 10 warps: shared memory)
  int pdl_now = 0;                   // set per launch by launch_group: 1 this sweep triggers its dependent, 2 this dataflow launch is the dependent
  int pdl = 0;                       // the dataflow launch starts under the upward sweep (programmatic dependent launch)
  int sweep_prefetch = 0;            // generic sweep: L2 prefetch of the next item's static inputs (H2B_SWEEP_PREFETCH mask)
  std::vector<PhaseDev> ph;
  // single GPU, 8/16 right-hand sides: near field (lean kernel), then the rest
  std::vector<PhaseDev> ph_split;
  int near_stage = 8192;    // lean near kernel ring stage (H2B_NEAR_STAGE=4096: 16 warps per SM)
  int near_grid = 0;
  int near_impl = 1;        // 1: both operands by TMA (h2b_near_tma_kernel), 0: ring + register gathers
  int near_nst = 2;         // TMA stages per warp (2: 8 warps per CTA, 3: 6 warps)
  int near_warps = 8;
  int split_only = 0;       // diagnostics (H2B_SPLIT_ONLY=near|rest): time one part; y is then wrong
  int trace_split = 0;      // diagnostics (H2B_TRACE_SPLIT=1): trace the split product's dataflow part
  // multi-GPU
  int rank = 0, world = 1;
  int64_t exch_off = 0, exch_count = 0;
  std::vector<int64_t> rank_lo, rank_hi;  // tree-position rows of every rank
  int64_t rows_max = 0;                   // max rows of a rank
  int64_t* d_rank_lo = nullptr;           // [world] on the device
  double* d_rows = nullptr;               // host path: gathered rows (world * rows_max * nrhs)
  size_t rows_cap = 0;
  ncclComm_t comm = nullptr;
  // host path buffers
  double* d_x = nullptr;
  double* d_y = nullptr;
  size_t xy_cap = 0;
  cudaStream_t hstream = nullptr;
  // staged host copies (h2b_matvec): pinned buffers, chunk events, copy threads
  double* pin_x = nullptr;
  double* pin_y = nullptr;
  size_t pin_cap = 0;
  std::vector<cudaEvent_t> chunk_ev;
  std::unique_ptr<CopyPool> pool;
  int copy_threads = -1;  // -1: not decided yet; 0: plain cudaMemcpyAsync from the caller's memory
  size_t copy_chunk = (size_t)1 << 20;
  // One product in flight per operator: the scheduler state (queue heads,
  // arrival counters, epoch) and the coefficient workspace are per operator.
  // Every launch waits for the previous one's completion event, whatever
  // stream either ran on; `mu` serialises the host side.
  cudaEvent_t done = nullptr;
  std::mutex mu;
  std::vector<cudaEvent_t>* tev = nullptr;  // h2b_launch_times: events of the product being timed
  int tev_n = 0;
  h2b_stats stats{};
};

struct h2b_plan {
  h2b::Plan plan;
  h2b_stats stats{};
};

namespace {

#define H2B_NCCL(call)                                                                   \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess) return fail(H2B_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

// Near-field plus coupling bytes of the operator (the bulk of
// storage_bytes()), per rank: decides the streaming defaults before planning.
// Runs before build_plan validates the descriptor, so it only reads what it
// has checked itself (a malformed descriptor gets 0 here and H2B_EINVAL from
// build_plan).
int64_t desc_stream_bytes_per_rank(const h2b_desc* d, const h2b_options* o) {
  if (!d || !d->cl_start || !d->cl_end || !d->k_row || !d->k_col || d->nclusters < 1) return 0;
  const int64_t nc = d->nclusters;
  auto ok = [nc](int64_t c) { return c >= 0 && c < nc; };
  int64_t b = 0;
  if (d->nnear > 0 && d->nr_row && d->nr_col)
    for (int64_t i = 0; i < d->nnear; ++i) {
      const int64_t r = d->nr_row[i], c = d->nr_col[i];
      if (ok(r) && ok(c)) b += (d->cl_end[r] - d->cl_start[r]) * (d->cl_end[c] - d->cl_start[c]);
    }
  if (d->ncoupling > 0 && d->cp_row && d->cp_col)
    for (int64_t i = 0; i < d->ncoupling; ++i) {
      const int64_t r = d->cp_row[i], c = d->cp_col[i];
      if (ok(r) && ok(c)) b += d->k_row[r] * d->k_col[c];
    }
  const int world = (o && o->world_size > 1) ? o->world_size : 1;
  return 8 * b / world;
}

bool streaming_defaults(const h2b_desc* d, const h2b_options* o) {
  return !(o && (o->sched_flags & H2B_SCHED_EXPLICIT)) && desc_stream_bytes_per_rank(d, o) >= H2B_STREAM_DEFAULT_BYTES;
}

h2b::PlanOptions to_plan_options(const h2b_desc* d, const h2b_options* o) {
  h2b::PlanOptions po;
  // the staged product (sweeps over the bottom subtrees around one dataflow
  // launch) by default: config 1 60 -> 52 us, config 2 0.209 -> 0.177 ms,
  // config 3 2.366 -> 2.295 ms, 2 / 4 right-hand sides -8..-15 %
  po.staged = true;
  // the level-skipping chain where the product is chain-bound: operators
  // (or rank shards) below 4 GiB of near-field and coupling bytes
  // (config 1 -6 %, config 2 -3.5 %, config 3 at 8 ranks -7 %; config 3 on
  // one GPU, near-field bound, +2.7 %: off)
  po.skip_levels = desc_stream_bytes_per_rank(d, o) < H2B_SKIP_DEFAULT_BYTES;
  // streaming operators: 8 KB chain pieces (a ring warp stages both ring
  // stages at once), halving the latency-bound up-leaf items
  // and 256 KB near-field pieces (a ring warp keeps streaming across the
  // whole item: fewer per-item round trips, and fewer partial-sum slots for
  // the finals to add -- at 16 RHS a slot is 8 KB; config 3 with 128 / 192 /
  // 256 / 384 KB: 2.264 / 2.251 / 2.238 / 2.92 ms -- 384 KB exceeds the 512
  // gathered columns of a ring item -- 8 RHS 3.017 / 2.952 / 2.916 / 2.877,
  // 16 RHS 4.086 / 3.947 / 3.858 / 3.777 ms)
  if (streaming_defaults(d, o)) {
    po.far_task_bytes = 8192;
    po.task_bytes = 262144;
  }
  if (o) {
    if (o->task_bytes > 0) po.task_bytes = o->task_bytes;
    if (o->far_task_bytes > 0) po.far_task_bytes = o->far_task_bytes;
    if (o->band_depth > 0) po.band_depth = o->band_depth;
    if (o->sched_flags & H2B_SCHED_FINAL_SLACK) po.final_class = 2;
    if (o->near_phase0_pct < 0) po.near_phase0_pct = 0;
    else if (o->near_phase0_pct > 0) po.near_phase0_pct = std::min(100, o->near_phase0_pct);
    po.rank = o->rank;
    po.world_size = o->world_size > 0 ? o->world_size : 1;
    if (o->plan_flags & H2B_PLAN_SKIP_LEVELS) po.skip_levels = true;
    if (o->plan_flags & H2B_PLAN_NO_SKIP) po.skip_levels = false;
    if ((o->plan_flags >> 4) & 0xf) po.coupling_task_bytes = (int64_t)1024 << ((o->plan_flags >> 4) & 0xf);
    if (o->plan_flags & H2B_PLAN_GATE) po.gate_coupling = true;
    if (o->plan_flags & H2B_PLAN_NO_GATE) po.gate_coupling = false;
    if (o->plan_flags & H2B_PLAN_STAGED) po.staged = true;
    if (o->plan_flags & H2B_PLAN_NO_STAGED) po.staged = false;
    if ((o->plan_flags >> 12) & 0xf) po.sweep_nodes = (int64_t)64 << ((o->plan_flags >> 12) & 0xf);
  }
  {
    const char* sg = std::getenv("H2B_STAGED");  // A/B switch for tools and benches
    if (sg && sg[0] == '1') po.staged = true;
    if (sg && sg[0] == '0') po.staged = false;
  }
  return po;
}

void fill_stats(const h2b::Plan& P, h2b_stats* s) {
  std::memset(s, 0, sizeof(*s));
  s->n = P.n;
  s->stream_bytes = P.stream_bytes;
  s->pool_bytes = 8 * P.mat_len;
  s->coef_doubles = P.coef_len;
  for (const auto& F : P.ph) {
    s->ntasks += F.ntasks();
    s->nsegs += F.nsegs();
    s->ndeps += (int64_t)F.deps.size();
    for (int k = 0; k < 5; ++k) s->tasks_by_kind[k] += F.tasks_by_kind[k];
  }
  for (int k = 0; k < 5; ++k) s->bytes_by_kind[k] = P.bytes_by_kind[k];
  s->rank = P.rank;
  s->world_size = P.world_size;
  s->local_bytes = P.local_bytes;
  s->extra_bytes = P.extra_bytes;
  s->launches = (int32_t)P.ph.size();
  s->resident_mask = 0;
}

int nrhs_index(int nrhs) {
  switch (nrhs) {
    case 1: return 0;
    case 2: return 1;
    case 4: return 2;
    case 8: return 3;
    case 16: return 4;
    default: return -1;
  }
}

template <int NRHS>
int occupancy_grid(int wpc, int ring_warps, int ring_stage, int ctas_per_sm, int* grid) {
  // NRHS >= 8: wpc and ring_stage are the multi-RHS launch's (h2b_op::mrhs_wpc, mrhs_stage)
  const size_t sm = NRHS >= 8 ? smem_bytes(wpc, wpc, ring_stage) : smem_bytes(wpc, ring_warps, ring_stage);
  H2B_CUDA(cudaFuncSetAttribute(h2b_dataflow_kernel<NRHS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int per_sm = 0;
  H2B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, h2b_dataflow_kernel<NRHS>, wpc * 32, sm));
  int dev = 0, nsm = 0;
  H2B_CUDA(cudaGetDevice(&dev));
  H2B_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  if (per_sm < 1) return fail(H2B_EINVAL, "per-warp shared memory does not fit: lower warps_per_cta");
  if (ctas_per_sm > 0 && ctas_per_sm < per_sm) per_sm = ctas_per_sm;
  *grid = per_sm * nsm;
  return H2B_OK;
}

template <int NRHS>
int sweep_grid(int wpc, int* grid) {
  const size_t sm = sweep_smem_bytes(wpc);
  H2B_CUDA(cudaFuncSetAttribute(h2b_sweep_kernel<NRHS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int per_sm = 0, dev = 0, nsm = 0;
  H2B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, h2b_sweep_kernel<NRHS>, wpc * 32, sm));
  H2B_CUDA(cudaGetDevice(&dev));
  H2B_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  if (per_sm < 1) return fail(H2B_EINVAL, "sweep kernel does not fit an SM: lower warps_per_cta");
  *grid = per_sm * nsm;
  return H2B_OK;
}

// xp = x[perm] (h2.py:192-193)
template <int NRHS>
int launch_permute(h2b_op* op, const double* x, cudaStream_t st) {
  const int64_t total = op->n * NRHS;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  h2b_permute_kernel<NRHS><<<blocks, 256, 0, st>>>(x, op->d_perm, op->d_xp, op->n);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(H2B_ECUDA, std::string("permute kernel launch: ") + cudaGetErrorString(e));
  return H2B_OK;
}

template <int NRHS>
KParams phase_params(h2b_op* op, const PhaseDev& F, double* y) {
  KParams p{};
  p.tasks = F.d_tasks;
  p.segs = F.d_segs;
  p.seg_inline = F.d_seg_inline;
  p.succ0 = F.d_succ0;
  p.succ = F.d_succ;
  p.ready0 = F.d_ready0;
  p.nready0 = F.nready0;
  p.nready0_hi = F.nready0_hi;
  p.gated = F.d_gated;
  p.ngated = F.ngated;
  p.ngated1 = F.ngated1;
  p.nup_gate = F.nup;
  p.arrived = F.d_arrived;
  p.ready_q = F.d_ready_q;
  p.ready_flag = F.d_ready_flag;
  p.ctl = F.d_ctl;
  p.trace = F.d_trace;
  p.ntasks = (int32_t)F.ntasks;
  p.nnodes = (int32_t)F.nnodes;
  p.mat = op->d_mat;
  p.coef = op->d_coef;
  p.perm = op->d_perm;
  p.xp = op->d_xp;
  p.y = y;
  p.flags = op->flags;
  p.ring_warps = op->ring_warps;
  p.ring_stage = op->ring_stage;
  p.mrhs_stage = op->mrhs_stage;
  p.unit0 = F.d_unit0;
  p.wave0 = F.d_wave0;
  p.nunits = F.nunits;
  p.u_range = F.d_u_range;
  p.cap_mat = F.cap_mat;
  p.cap_vec = F.cap_vec;
  p.cap_items = F.cap_items;
  p.sweep_prefetch = op->sweep_prefetch;
  p.pdl = op->pdl_now;
  return p;
}

// One dataflow launch (Phase::mode 0).
template <int NRHS>
int launch_phase_dev(h2b_op* op, const PhaseDev& F, double* y, cudaStream_t st) {
  if (F.ntasks == 0) return H2B_OK;
  const KParams p = phase_params<NRHS>(op, F, y);
  const int gi = nrhs_index(NRHS);
  const int wpc = NRHS >= 8 ? op->mrhs_wpc : op->wpc;
  const size_t smem = NRHS >= 8 ? smem_bytes(wpc, wpc, op->mrhs_stage)
                                : smem_bytes(op->wpc, op->ring_warps, op->ring_stage);
  const cudaError_t stale = cudaGetLastError();  // clear errors of unrelated earlier calls
  // the attribute is per function and shared by every operator of the process
  H2B_CUDA(cudaFuncSetAttribute(h2b_dataflow_kernel<NRHS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (op->pdl_now == 2) {
    // programmatic dependent launch: CTAs may become resident while the
    // preceding sweep still runs; the kernel waits for it where it must
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)op->grid[gi]);
    cfg.blockDim = dim3((unsigned)(wpc * 32));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    H2B_CUDA(cudaLaunchKernelEx(&cfg, h2b_dataflow_kernel<NRHS>, p));
  } else {
    h2b_dataflow_kernel<NRHS><<<op->grid[gi], wpc * 32, smem, st>>>(p);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return fail(H2B_ECUDA, std::string("kernel launch (nrhs=") + std::to_string(NRHS) + ", grid=" +
                               std::to_string(op->grid[gi]) + ", block=" + std::to_string(wpc * 32) +
                               ", smem=" + std::to_string(smem) +
                               "): " + cudaGetErrorString(e) + " (stale: " + cudaGetErrorString(stale) + ")");
  return H2B_OK;
}

// One sweep launch (Phase::mode 1): CTAs claim units from a counter.  The
// resident kernel when every unit's inputs are contiguous ranges that fit a
// CTA's shared memory at this NRHS (at least two CTAs per SM preferred),
// else the generic one.
template <int NRHS>
int launch_sweep(h2b_op* op, const PhaseDev& F, double* y, cudaStream_t st) {
  if (F.ntasks == 0 || F.nunits == 0) return H2B_OK;
  const KParams p = phase_params<NRHS>(op, F, y);
  if (F.resident && op->sweep_resident) {
    const size_t smem = sweep_geom(NRHS, op->wpc, F.cap_mat, F.cap_vec, F.cap_items).total;
    if (smem <= (size_t)op->smem_optin) {
      H2B_CUDA(cudaFuncSetAttribute(h2b_sweep_resident_kernel<NRHS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
      int per_sm = 0;
      H2B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, h2b_sweep_resident_kernel<NRHS>, op->wpc * 32,
                                                             smem));
      if (per_sm >= 1) {
        const int grid = std::min<int>(per_sm * op->nsm, F.nunits);
        h2b_sweep_resident_kernel<NRHS><<<grid, op->wpc * 32, smem, st>>>(p);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess)
          return fail(H2B_ECUDA, std::string("resident sweep kernel launch: ") + cudaGetErrorString(e));
        return H2B_OK;
      }
    }
  }
  const size_t smem = sweep_smem_bytes(op->wpc);
  H2B_CUDA(cudaFuncSetAttribute(h2b_sweep_kernel<NRHS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int gi = nrhs_index(NRHS);
  const int grid = std::min<int>(op->sweep_grid[gi], F.nunits);
  h2b_sweep_kernel<NRHS><<<grid, op->wpc * 32, smem, st>>>(p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(H2B_ECUDA, std::string("sweep kernel launch: ") + cudaGetErrorString(e));
  return H2B_OK;
}

template <int NRHS, int STAGE>
int launch_near(h2b_op* op, const PhaseDev& F, cudaStream_t st) {
  if (F.ntasks == 0) return H2B_OK;
  KParams p = phase_params<NRHS>(op, F, nullptr);
  const size_t smem = (size_t)op->wpc * sizeof(WarpSmem) + (size_t)op->wpc * ring_bytes(STAGE);
  H2B_CUDA(cudaMemsetAsync(&F.d_ctl->near_head, 0, sizeof(unsigned), st));
  H2B_CUDA(cudaFuncSetAttribute(h2b_near_kernel<NRHS, STAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  h2b_near_kernel<NRHS, STAGE><<<op->near_grid, op->wpc * 32, smem, st>>>(p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(H2B_ECUDA, std::string("near kernel launch: ") + cudaGetErrorString(e));
  return H2B_OK;
}

template <int NRHS, int NST>
int launch_near_tma(h2b_op* op, const PhaseDev& F, cudaStream_t st) {
  if (F.ntasks == 0) return H2B_OK;
  KParams p = phase_params<NRHS>(op, F, nullptr);
  const size_t smem = (size_t)op->near_warps * near_warp_smem<NRHS>(NST);
  H2B_CUDA(cudaMemsetAsync(&F.d_ctl->near_head, 0, sizeof(unsigned), st));
  H2B_CUDA(cudaFuncSetAttribute(h2b_near_tma_kernel<NRHS, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  int per_sm = 0, dev = 0, nsm = 0;
  H2B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, h2b_near_tma_kernel<NRHS, NST>,
                                                         op->near_warps * 32, smem));
  H2B_CUDA(cudaGetDevice(&dev));
  H2B_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  if (per_sm < 1) return fail(H2B_EINVAL, "near TMA kernel does not fit an SM");
  h2b_near_tma_kernel<NRHS, NST><<<per_sm * nsm, op->near_warps * 32, smem, st>>>(p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(H2B_ECUDA, std::string("near TMA kernel launch: ") + cudaGetErrorString(e));
  return H2B_OK;
}

// One launch of the plan, by its mode.
template <int NRHS>
int launch_one(h2b_op* op, const PhaseDev& F, double* y, cudaStream_t st) {
  if (F.mode == 1) return op->split_only == 1 ? H2B_OK : launch_sweep<NRHS>(op, F, y, st);
  if constexpr (NRHS >= 8) {
    // the near field of a split multi-RHS product: the lean near kernel
    if (F.mode == 2) {
      if (op->split_only == 2) return H2B_OK;
      return op->near_impl == 1 ? (op->near_nst == 3 ? launch_near_tma<NRHS, 3>(op, F, st)
                                                     : launch_near_tma<NRHS, 2>(op, F, st))
             : op->near_stage == 4096 ? launch_near<NRHS, 4096>(op, F, st) : launch_near<NRHS, 8192>(op, F, st);
    }
  }
  if (op->split_only == 1) return H2B_OK;
  return launch_phase_dev<NRHS>(op, F, y, st);
}

// The launches of one group (0: before the x^ exchange -- xp = x[perm]
// first -- 1: after it).  8/16 right-hand sides on one GPU use the split
// list (the near field in the lean kernel).
template <int NRHS>
int launch_group(h2b_op* op, int group, const double* x, double* y, cudaStream_t st) {
  const std::vector<PhaseDev>& list = (NRHS >= 8 && !op->ph_split.empty()) ? op->ph_split : op->ph;
  int rc = H2B_OK;
  // (h2b_launch_times: an event before every launch and after the last)
  auto mark = [&]() {
    if (op->tev && op->tev_n < (int)op->tev->size()) cudaEventRecord((*op->tev)[op->tev_n++], st);
  };
  if (group == 0) {
    mark();
    if ((rc = launch_permute<NRHS>(op, x, st)) != H2B_OK) return rc;
  }
  // (H2B_PDL) an upward sweep directly followed by the dataflow launch of the
  // same group: the pair is launched as primary and programmatic dependent
  // (multi-GPU: group 0 is [upward sweep][dataflow launch of phase 0] -- the same pair)
  const bool pdl_ok = op->pdl && NRHS <= 4 && !op->tev && op->split_only == 0;
  for (size_t k = 0; k < list.size(); ++k) {
    const PhaseDev& F = list[k];
    if (F.group != group) continue;
    op->pdl_now = 0;
    if (pdl_ok && F.mode == 1 && F.ntasks > 0 && k + 1 < list.size() && list[k + 1].group == group &&
        list[k + 1].mode == 0 && list[k + 1].ntasks > 0)
      op->pdl_now = 1;
    else if (pdl_ok && F.mode == 0 && k > 0 && list[k - 1].group == group && list[k - 1].mode == 1 &&
             list[k - 1].ntasks > 0 && F.ntasks > 0)
      op->pdl_now = 2;
    mark();
    rc = launch_one<NRHS>(op, F, y, st);
    op->pdl_now = 0;
    if (rc != H2B_OK) return rc;
  }
  mark();
  return H2B_OK;
}

// The whole product: both groups, with the x^ all-gather between them.
template <int NRHS>
int launch(h2b_op* op, const double* x, double* y, cudaStream_t st) {
  int rc = launch_group<NRHS>(op, 0, x, y, st);
  if (rc != H2B_OK || op->world <= 1) return rc;
  if (!op->comm) return fail(H2B_EINVAL, "multi-GPU operator without an NCCL communicator");
  double* base = op->d_coef + op->exch_off * NRHS;
  const size_t cnt = (size_t)op->exch_count * NRHS;
  if (cnt > 0) H2B_NCCL(ncclAllGather(base + (size_t)op->rank * cnt, base, cnt, ncclDouble, op->comm, st));
  return launch_group<NRHS>(op, 1, x, y, st);
}

template <typename T>
int upload(T** dst, const T* src, size_t count) {
  if (count == 0) count = 1;
  H2B_CUDA(cudaMalloc((void**)dst, sizeof(T) * count));
  if (src) H2B_CUDA(cudaMemcpy(*dst, src, sizeof(T) * count, cudaMemcpyHostToDevice));
  return H2B_OK;
}

void free_phase(PhaseDev& F) {
  cudaFree(F.d_tasks);
  cudaFree(F.d_segs);
  cudaFree(F.d_seg_inline);
  cudaFree(F.d_succ0);
  cudaFree(F.d_succ);
  cudaFree(F.d_ready0);
  cudaFree(F.d_gated);
  cudaFree(F.d_arrived);
  cudaFree(F.d_ready_q);
  cudaFree(F.d_ready_flag);
  cudaFree(F.d_ctl);
  cudaFree(F.d_trace);
  cudaFree(F.d_unit0);
  cudaFree(F.d_wave0);
  cudaFree(F.d_u_range);
}

void free_op(h2b_op* op) {
  if (!op) return;
  for (auto& F : op->ph) free_phase(F);
  for (auto& F : op->ph_split) free_phase(F);
  if (op->comm) ncclCommDestroy(op->comm);
  cudaFree(op->d_mat);
  cudaFree(op->d_coef);
  cudaFree(op->d_perm);
  cudaFree(op->d_x);
  cudaFree(op->d_y);
  cudaFree(op->d_xp);
  cudaFree(op->d_rank_lo);
  cudaFree(op->d_rows);
  if (op->hstream) cudaStreamDestroy(op->hstream);
  if (op->done) cudaEventDestroy(op->done);
  op->pool.reset();
  for (cudaEvent_t e : op->chunk_ev) cudaEventDestroy(e);
  if (op->pin_x) cudaFreeHost(op->pin_x);
  if (op->pin_y) cudaFreeHost(op->pin_y);
  delete op;
}

int upload_phase(const h2b::Phase& P, PhaseDev* F) {
  int rc;
  F->ntasks = P.ntasks();
  F->nnodes = P.nnodes;
  F->mode = P.mode;
  F->group = P.group;
  for (int64_t i = 0; i < P.ntasks(); ++i) F->bytes += 8 * (int64_t)P.t_m[i] * P.t_ncols[i];
  if (P.mode == 1) {
    if ((rc = upload(&F->d_unit0, P.unit0.data(), P.unit0.size()))) return rc;
    if ((rc = upload(&F->d_wave0, P.wave0.data(), P.wave0.size()))) return rc;
    F->nunits = (int32_t)P.unit0.size() - 1;
    if ((rc = upload(&F->d_u_range, P.u_rec.data(), P.u_rec.size()))) return rc;
    F->resident = P.resident && P.res_mat_max < (1 << 20) && P.res_vec_max < (1 << 20);
    F->cap_mat = (int)P.res_mat_max;
    F->cap_vec = (int)P.res_vec_max;
    F->cap_items = P.res_items_max;
  }
  std::vector<DTask> tasks(P.ntasks());
  for (int64_t i = 0; i < P.ntasks(); ++i) {
    DTask& t = tasks[i];
    t.data = P.t_data[i];
    t.out = P.t_out[i];
    t.bias = P.t_bias[i];
    t.m = P.t_m[i];
    t.ld = P.t_ld[i];
    t.ncols = P.t_ncols[i];
    t.kind = P.t_kind[i];
    t.seg0 = P.t_seg0[i];
    t.seg1 = P.t_seg0[i + 1];
    t.pad0_ = t.pad1_ = 0;
    t.bias_nslots = P.t_bias_nslots[i];
    t.bias_stride = P.t_bias_stride[i];
  }
  std::vector<DSeg> segs(P.nsegs());
  for (int64_t i = 0; i < P.nsegs(); ++i) {
    segs[i].src = P.s_src[i];
    segs[i].ncols = P.s_ncols[i];
    segs[i].kind = P.s_kind[i];
    segs[i].nslots = P.s_nslots[i];
    segs[i].stride = P.s_stride[i];
  }
  if ((rc = upload(&F->d_tasks, tasks.data(), tasks.size()))) return rc;
  if ((rc = upload(&F->d_segs, segs.data(), segs.size()))) return rc;
  {
    std::vector<DSeg> inl((size_t)std::max<int64_t>(1, P.ntasks()) * kInlineSegs, DSeg{0, 0, 0, 0, 0});
    for (int64_t i = 0; i < P.ntasks(); ++i) {
      const int32_t a = P.t_seg0[i], b = P.t_seg0[i + 1];
      if (b - a <= kInlineSegs)
        for (int32_t k = a; k < b; ++k) inl[(size_t)i * kInlineSegs + (k - a)] = segs[k];
    }
    if ((rc = upload(&F->d_seg_inline, inl.data(), inl.size()))) return rc;
  }
  if ((rc = upload(&F->d_succ0, P.succ0.data(), P.succ0.size()))) return rc;
  {
    std::vector<int2> sd(P.succ.size());
    for (size_t k = 0; k < sd.size(); ++k) {
      const int32_t d = P.succ[k];
      // low 24 bits: dependency count; bits 24+: the successor's queue class
      sd[k] = make_int2(d, (P.t_dep0[d + 1] - P.t_dep0[d]) | ((int)P.t_qclass[d] << 24));
    }
    if ((rc = upload(&F->d_succ, sd.data(), sd.size()))) return rc;
  }
  if ((rc = upload(&F->d_ready0, P.ready0.data(), P.ready0.size()))) return rc;
  F->nready0 = (int32_t)P.ready0.size();
  F->nready0_hi = P.n_ready0_hi;
  if ((rc = upload(&F->d_gated, P.gated.data(), P.gated.size()))) return rc;
  F->ngated = (int32_t)P.gated.size();
  F->ngated1 = P.n_gated1;
  F->nup = P.n_up;
  // (a sweep has no scheduler state: one entry each)
  const size_t T1 = P.mode == 1 ? 1 : (size_t)std::max<int64_t>(1, P.ntasks());
  if ((rc = upload<unsigned long long>(&F->d_arrived, nullptr, T1))) return rc;
  if ((rc = upload<int32_t>(&F->d_ready_q, nullptr, kQueues * T1))) return rc;
  if ((rc = upload<unsigned>(&F->d_ready_flag, nullptr, kQueues * T1))) return rc;
  if ((rc = upload<Ctl>(&F->d_ctl, nullptr, 1))) return rc;
  H2B_CUDA(cudaMemset(F->d_arrived, 0, sizeof(unsigned long long) * T1));
  H2B_CUDA(cudaMemset(F->d_ready_flag, 0, sizeof(unsigned) * kQueues * T1));
  H2B_CUDA(cudaMemset(F->d_ctl, 0, sizeof(Ctl)));
  return H2B_OK;
}

int host_threads() {
  const unsigned h = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(16u, h ? h : 1u));
}

// The pool straight from the descriptor's matrices to the device, packed
// by host threads into two pinned staging buffers that alternate with the
// copies: no host copy of the whole pool (config 5: ~29 GB).
int upload_pool(const h2b::Plan& P, double* d_mat) {
  constexpr size_t kStage = size_t(64) << 20;  // doubles per staging buffer (512 MB)
  double* stage[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaStream_t st = nullptr;
  int rc = H2B_OK;
  auto cleanup = [&]() {
    if (st) cudaStreamSynchronize(st);
    for (int k = 0; k < 2; ++k) {
      if (stage[k]) cudaFreeHost(stage[k]);
      if (ev[k]) cudaEventDestroy(ev[k]);
    }
    if (st) cudaStreamDestroy(st);
  };
  auto cuda = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && rc == H2B_OK) rc = fail(H2B_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return e == cudaSuccess;
  };
  const size_t cap = std::min<size_t>(kStage, std::max<int64_t>(1, P.mat_len));
  if (!cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream") ||
      !cuda(cudaMallocHost((void**)&stage[0], sizeof(double) * cap), "cudaMallocHost") ||
      !cuda(cudaMallocHost((void**)&stage[1], sizeof(double) * cap), "cudaMallocHost") ||
      !cuda(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming), "event") ||
      !cuda(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming), "event")) {
    cleanup();
    return rc;
  }
  const int threads = host_threads();
  size_t g = 0, k = 0;
  const size_t G = P.groups.size();
  while (g < G && rc == H2B_OK) {
    while (g < G && P.groups[g].base < 0) ++g;
    if (g >= G) break;
    // groups [g, g1) fill at most one staging buffer (a larger group alone)
    const int64_t b0 = P.groups[g].base;
    size_t g1 = g;
    int64_t end = b0;
    while (g1 < G) {
      const auto& q = P.groups[g1];
      if (q.base >= 0) {
        if (q.base + q.size() - b0 > (int64_t)cap && g1 > g) break;
        end = q.base + q.size();
      }
      ++g1;
    }
    if (end - b0 > (int64_t)cap) {  // one group above 512 MB: pack it through host memory
      std::vector<double> tmp((size_t)(end - b0));
      h2b::pack_groups(P, g, g1, tmp.data(), threads);
      cuda(cudaStreamSynchronize(st), "sync");
      cuda(cudaMemcpy(d_mat + b0, tmp.data(), sizeof(double) * tmp.size(), cudaMemcpyHostToDevice), "upload");
    } else {
      cuda(cudaEventSynchronize(ev[k]), "sync");   // the copy that last used this buffer
      h2b::pack_groups(P, g, g1, stage[k], threads);
      cuda(cudaMemcpyAsync(d_mat + b0, stage[k], sizeof(double) * (size_t)(end - b0), cudaMemcpyHostToDevice, st),
           "upload");
      cuda(cudaEventRecord(ev[k], st), "event");
      k ^= 1;
    }
    g = g1;
  }
  cleanup();
  return rc;
}

int create_impl(const h2b_desc* d, const h2b_options* o, h2b_op** out) {
  if (!out) return fail(H2B_EINVAL, "null output pointer");
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
    cudaGetLastError();
    return fail(H2B_ENODEV, "no CUDA device available");
  }
  h2b::Plan P;
  std::string err;
  h2b::PlanOptions po = to_plan_options(d, o);
  // 8/16 right-hand sides on one GPU: the near field in the lean kernel
  // (H2B_NEAR_SPLIT=0: the near field inside the dataflow kernel, round 1)
  const int max_nrhs_req = (o && o->max_nrhs > 0) ? o->max_nrhs : 16;
  const char* ns_env = std::getenv("H2B_NEAR_SPLIT");
  po.near_split = po.world_size <= 1 && max_nrhs_req >= 8 && !(ns_env && ns_env[0] == '0');
  {
    // the split product's bottom subtrees as sweeps too (the generic sweep kernel fits two
    // CTAs per SM at 8/16 RHS): config 3, 8 RHS 3.398 -> 3.014 ms, 16 RHS 4.247 -> 4.089 ms,
    // the same bits.  H2B_SPLIT_SWEEPS=0: every far-field item in the dataflow launch.
    const char* sw = std::getenv("H2B_SPLIT_SWEEPS");
    po.split_sweeps = po.staged && !(sw && sw[0] == '0');
  }
  int rc = h2b::build_plan(d, po, &P, &err);
  if (rc != H2B_OK) return fail(rc, err);
  for (const auto& F : P.ph) {
    if (F.ntasks() >= INT32_MAX / kQueues) return fail(H2B_EINVAL, "too many work items");
    if (F.mode != 1 && F.nnodes != F.ntasks())
      return fail(H2B_EINVAL, "band_depth > 1 (fused runs) is a planning option only: the kernel runs "
                              "single items (fused runs measured slower on B200, DESIGN.md)");
  }

  std::unique_ptr<h2b_op, void (*)(h2b_op*)> op(new h2b_op(), free_op);
  H2B_CUDA(cudaGetDevice(&op->device));
  op->n = P.n;
  op->coef_len = P.coef_len;
  op->max_nrhs = (o && o->max_nrhs > 0) ? o->max_nrhs : 16;
  if (nrhs_index(op->max_nrhs) < 0) return fail(H2B_EINVAL, "max_nrhs must be 1, 2, 4, 8 or 16");
  op->wpc = (o && o->warps_per_cta > 0) ? o->warps_per_cta : 8;
  if (op->wpc > 8) return fail(H2B_EINVAL, "warps_per_cta must be <= 8");
  const int cps = o ? o->ctas_per_sm : 0;
  int sf = o ? o->sched_flags : 0;
  if (!(sf & H2B_SCHED_EXPLICIT) && !streaming_defaults(d, o) && ((sf >> 20) & 0xf) == 0)
    sf |= H2B_SCHED_LEAF_MIX(2);   // plain scheduling: config 2 0.2085 -> 0.2026 ms with the skipping chain
  if (streaming_defaults(d, o)) {
    // streaming defaults (measured on config 3)
    if (((sf >> 4) & 0xf) == 0) sf |= H2B_SCHED_RING_WARPS(8) | H2B_SCHED_RING_STAGE(2);
    if (((sf >> 26) & 0xf) == 0) sf |= H2B_SCHED_NEAR_PRIO(6);
    if (((sf >> 20) & 0xf) == 0) sf |= H2B_SCHED_LEAF_MIX(4);
    sf |= H2B_SCHED_STREAM_EVICT_FIRST;
  }
  op->sched = sf;
  op->flags = ((sf & H2B_SCHED_NEAR_FIRST) ? 0 : kFlagSlackFirst) | (int)((unsigned)sf & 0xfff3ff04u);
  {
    // 8/16 RHS: every item with <= 64 rows through the TMA ring, sources by
    // TMA where contiguous (config 3, 16 RHS: 5.09 -> 4.52 ms; 8 RHS 3.63 -> 3.51)
    const char* ra = std::getenv("H2B_MRHS_RING_ALL");
    if (!(ra && ra[0] == '0')) op->flags |= kFlagMrhsRingAll;
    const char* um = std::getenv("H2B_UP_MIX");
    if (um && um[0] == '1') op->flags |= kFlagUpMix;
    // ... and the TMA-moved sources of few-row items inside the ring stage (twice the columns per stage)
    const char* ss = std::getenv("H2B_MRHS_SRC_IN_STAGE");
    if (!(ss && ss[0] == '0')) op->flags |= kFlagMrhsSrcInStage;
    // ... on H2B_MRHS_WARPS warps per SM (one CTA; 12 warps: 168 registers each, 6 KB ring stages)
    const char* mw = std::getenv("H2B_MRHS_WARPS");
    op->mrhs_wpc = mw ? std::max(1, std::min(kMrhsThreads / 32, std::atoi(mw))) : kMrhsThreads / 32;
    op->mrhs_stage = op->mrhs_wpc > 12 ? 4096 : op->mrhs_wpc > 10 ? 6144 : kMrhsStage;
  }
  op->ring_warps = std::min((sf >> 4) & 0xf, op->wpc);
  {
    const int sel = (sf >> 18) & 3;
    op->ring_stage = sel == 1 ? 6144 : sel == 2 ? 4096 : kRingStageBytes;
    {
      // Programmatic dependent launch of the dataflow kernel under the upward sweep: its
      // near-priority warps stream near-field items (which need only xp) while the sweep
      // -- latency-bound, HBM mostly idle -- still runs; every other item waits for the
      // sweep (griddepcontrol.wait).  On for streaming operators: config 3 2.240 -> 2.213 ms,
      // config 5 4.636 -> 4.576 ms, the same bits; off for small ones, where the product is
      // the far-field chain and the early near field only slows the sweep (config 2
      // 0.179 -> 0.220 ms).  H2B_PDL=0 / 1 forces it.
      const char* pd = std::getenv("H2B_PDL");
      op->pdl = pd ? (pd[0] == '1') : (desc_stream_bytes_per_rank(d, o) >= H2B_STREAM_DEFAULT_BYTES ? 1 : 0);
      const char* e = std::getenv("H2B_SWEEP_PREFETCH");  // A/B switch, read at create (tools/sweep.py --env)
      // bit 0: x ranges, 1: bias slots, 2: permutation entries.  Off by default: measured on
      // config 3 the up sweep gets faster (0.110 -> 0.093 ms) but the product does not
      // (2.263 ms off, 2.279 / 2.264 / 2.266 / 2.275 ms with masks 1 / 2 / 4 / 3)
      op->sweep_prefetch = e ? std::atoi(e) : 0;
    }
  }
  op->rank = P.rank;
  op->world = P.world_size;
  op->exch_off = P.exch_off;
  op->exch_count = P.exch_count;
  op->rank_lo = P.rank_lo;
  op->rank_hi = P.rank_hi;
  for (size_t r = 0; r < P.rank_lo.size(); ++r) op->rows_max = std::max(op->rows_max, P.rank_hi[r] - P.rank_lo[r]);

  // the pool plus 48 bytes: bulk copies round a matrix's end up to 16 bytes
  if ((rc = upload<double>(&op->d_mat, nullptr, (size_t)P.mat_len + 6))) return rc;
  H2B_CUDA(cudaMemset(op->d_mat + P.mat_len, 0, sizeof(double) * 6));
  if ((rc = upload_pool(P, op->d_mat))) return rc;
  op->ph.resize(P.ph.size());
  for (size_t k = 0; k < P.ph.size(); ++k)
    if ((rc = upload_phase(P.ph[k], &op->ph[k]))) return rc;
  op->ph_split.resize(P.ph_split.size());
  for (size_t k = 0; k < P.ph_split.size(); ++k)
    if ((rc = upload_phase(P.ph_split[k], &op->ph_split[k]))) return rc;
  // (+2 entries: the resident sweeps' bulk copies round ranges out to 16 bytes)
  if ((rc = upload<int64_t>(&op->d_perm, nullptr, P.perm.size() + 2))) return rc;
  H2B_CUDA(cudaMemset(op->d_perm, 0, sizeof(int64_t) * (P.perm.size() + 2)));
  H2B_CUDA(cudaMemcpy(op->d_perm, P.perm.data(), sizeof(int64_t) * P.perm.size(), cudaMemcpyHostToDevice));
  if ((rc = upload(&op->d_rank_lo, P.rank_lo.data(), P.rank_lo.size()))) return rc;
  if ((rc = upload<double>(&op->d_coef, nullptr, (size_t)std::max<int64_t>(1, P.coef_len) * op->max_nrhs + 2))) return rc;
  if ((rc = upload<double>(&op->d_xp, nullptr, (size_t)P.n * op->max_nrhs + 2))) return rc;
  H2B_CUDA(cudaMemset(op->d_xp, 0, sizeof(double) * ((size_t)P.n * op->max_nrhs + 2)));
  H2B_CUDA(cudaMemset(op->d_coef, 0, sizeof(double) * std::max<int64_t>(1, P.coef_len) * op->max_nrhs));

  if ((rc = occupancy_grid<1>(op->wpc, op->ring_warps, op->ring_stage, cps, &op->grid[0]))) return rc;
  if ((rc = occupancy_grid<2>(op->wpc, op->ring_warps, op->ring_stage, cps, &op->grid[1]))) return rc;
  if ((rc = occupancy_grid<4>(op->wpc, op->ring_warps, op->ring_stage, cps, &op->grid[2]))) return rc;
  if ((rc = occupancy_grid<8>(op->mrhs_wpc, op->mrhs_wpc, op->mrhs_stage, cps, &op->grid[3]))) return rc;
  if ((rc = occupancy_grid<16>(op->mrhs_wpc, op->mrhs_wpc, op->mrhs_stage, cps, &op->grid[4]))) return rc;
  H2B_CUDA(cudaDeviceGetAttribute(&op->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, op->device));
  H2B_CUDA(cudaDeviceGetAttribute(&op->nsm, cudaDevAttrMultiProcessorCount, op->device));
  {
    const char* sr = std::getenv("H2B_SWEEP_RESIDENT");
    op->sweep_resident = !(sr && sr[0] == '0');
  }
  if ((rc = sweep_grid<1>(op->wpc, &op->sweep_grid[0]))) return rc;
  if ((rc = sweep_grid<2>(op->wpc, &op->sweep_grid[1]))) return rc;
  if ((rc = sweep_grid<4>(op->wpc, &op->sweep_grid[2]))) return rc;
  if ((rc = sweep_grid<8>(op->wpc, &op->sweep_grid[3]))) return rc;
  if ((rc = sweep_grid<16>(op->wpc, &op->sweep_grid[4]))) return rc;
  if (!op->ph_split.empty()) {
    const char* st_env = std::getenv("H2B_NEAR_STAGE");
    op->near_stage = (st_env && std::atoi(st_env) == 4096) ? 4096 : 8192;
    const char* im_env = std::getenv("H2B_NEAR_IMPL");
    op->near_impl = (im_env && std::string(im_env) == "ring") ? 0 : 1;
    const char* ns_env2 = std::getenv("H2B_NEAR_NST");
    op->near_nst = (ns_env2 && std::atoi(ns_env2) == 3) ? 3 : 2;
    op->near_warps = op->near_nst == 3 ? 6 : 8;
    const char* so = std::getenv("H2B_SPLIT_ONLY");
    op->split_only = !so ? 0 : std::string(so) == "near" ? 1 : std::string(so) == "rest" ? 2 : 0;
    const char* ts = std::getenv("H2B_TRACE_SPLIT");
    op->trace_split = ts && ts[0] == '1';
    const size_t sm = (size_t)op->wpc * sizeof(WarpSmem) + (size_t)op->wpc * ring_bytes(op->near_stage);
    int per_sm = 0, dev = 0, nsm = 0;
    if (op->near_stage == 4096) {
      H2B_CUDA(cudaFuncSetAttribute(h2b_near_kernel<16, 4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      H2B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, h2b_near_kernel<16, 4096>, op->wpc * 32, sm));
    } else {
      H2B_CUDA(cudaFuncSetAttribute(h2b_near_kernel<16, 8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      H2B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, h2b_near_kernel<16, 8192>, op->wpc * 32, sm));
    }
    H2B_CUDA(cudaGetDevice(&dev));
    H2B_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    if (per_sm < 1) return fail(H2B_EINVAL, "near kernel does not fit an SM");
    op->near_grid = per_sm * nsm;
  }
  if (op->world > 1 && o && o->nccl_unique_id) {
    ncclUniqueId id;
    std::memcpy(&id, o->nccl_unique_id, sizeof(id));
    H2B_NCCL(ncclCommInitRank(&op->comm, op->world, id, op->rank));
  }
  H2B_CUDA(cudaEventCreateWithFlags(&op->done, cudaEventDisableTiming));
  H2B_CUDA(cudaDeviceSynchronize());

  fill_stats(P, &op->stats);
  op->stats.grid = op->grid[0];
  op->stats.warps_per_cta = op->wpc;
  op->stats.sched_flags = op->sched;
  op->stats.ring_warps = op->ring_warps;
  for (int i = 0; i < 5 && op->sweep_resident; ++i) {
    bool all = false;
    for (const auto& F : ((1 << i) >= 8 && !op->ph_split.empty()) ? op->ph_split : op->ph) {
      if (F.mode != 1 || F.nunits == 0) continue;
      all = F.resident && sweep_geom(1 << i, op->wpc, F.cap_mat, F.cap_vec, F.cap_items).total <= (size_t)op->smem_optin;
      if (!all) break;
    }
    if (all) op->stats.resident_mask |= 1 << i;
  }
  *out = op.release();
  return H2B_OK;
}

int check_nrhs(const h2b_op* op, int nrhs) {
  if (nrhs_index(nrhs) < 0 || nrhs > op->max_nrhs)
    return fail(H2B_EINVAL, "nrhs must be 1, 2, 4, 8 or 16 and <= max_nrhs");
  return H2B_OK;
}

// Scheduler state back to its just-created values (all phases): arrival
// counters, ready flags, queue heads and the epoch.  Caller holds op->mu.
int reset_locked(h2b_op* op) {
  H2B_CUDA(cudaSetDevice(op->device));
  H2B_CUDA(cudaDeviceSynchronize());
  for (auto* list : {&op->ph, &op->ph_split})
  for (auto& F : *list) {
    const size_t T1 = F.mode == 1 ? 1 : (size_t)std::max<int64_t>(1, F.ntasks);
    H2B_CUDA(cudaMemset(F.d_arrived, 0, sizeof(unsigned long long) * T1));
    H2B_CUDA(cudaMemset(F.d_ready_flag, 0, sizeof(unsigned) * kQueues * T1));
    H2B_CUDA(cudaMemset(F.d_ctl, 0, sizeof(Ctl)));
  }
  H2B_CUDA(cudaDeviceSynchronize());
  return H2B_OK;
}

// Caller holds op->mu.  `phase` < 0: the whole product (all phases and the
// exchange); else that phase only.
int matvec_locked(h2b_op* op, int phase, const double* x, double* y, int nrhs, void* stream) {
  if (!x || !y) return fail(H2B_EINVAL, "null vector");
  if (check_nrhs(op, nrhs)) return H2B_EINVAL;
  H2B_CUDA(cudaSetDevice(op->device));
  cudaStream_t st = (cudaStream_t)stream;
  H2B_CUDA(cudaStreamWaitEvent(st, op->done, 0));   // the previous product of this operator
  int rc;
  if (phase < 0) {
    switch (nrhs) {
      case 1: rc = launch<1>(op, x, y, st); break;
      case 2: rc = launch<2>(op, x, y, st); break;
      case 4: rc = launch<4>(op, x, y, st); break;
      case 8: rc = launch<8>(op, x, y, st); break;
      default: rc = launch<16>(op, x, y, st); break;
    }
  } else {
    switch (nrhs) {
      case 1: rc = launch_group<1>(op, phase, x, y, st); break;
      case 2: rc = launch_group<2>(op, phase, x, y, st); break;
      case 4: rc = launch_group<4>(op, phase, x, y, st); break;
      case 8: rc = launch_group<8>(op, phase, x, y, st); break;
      default: rc = launch_group<16>(op, phase, x, y, st); break;
    }
  }
  if (rc != H2B_OK) {
    // a launch that failed part-way may have left a phase's counters
    // mid-product: restore the created state (keeps the first error message)
    const std::string msg = h2b_last_error();
    reset_locked(op);
    return fail(rc, msg);
  }
  H2B_CUDA(cudaEventRecord(op->done, st));
  return H2B_OK;
}

int matvec_dev_impl(h2b_op* op, const double* x, double* y, int nrhs, void* stream) {
  if (!op) return fail(H2B_EINVAL, "null operator");
  std::lock_guard<std::mutex> lk(op->mu);
  return matvec_locked(op, -1, x, y, nrhs, stream);
}

void fill_view(const h2b::Plan& P, const h2b::Phase& F, h2b_plan_view* v) {
  v->ntasks = F.ntasks();
  v->nsegs = F.nsegs();
  v->ndeps = (int64_t)F.deps.size();
  v->mat_len = (int64_t)P.mat.size();
  v->coef_len = P.coef_len;
  v->mat = P.mat.data();
  v->t_data = F.t_data.data();
  v->t_out = F.t_out.data();
  v->t_bias = F.t_bias.data();
  v->t_m = F.t_m.data();
  v->t_ld = F.t_ld.data();
  v->t_ncols = F.t_ncols.data();
  v->t_kind = F.t_kind.data();
  v->t_seg0 = F.t_seg0.data();
  v->t_dep0 = F.t_dep0.data();
  v->t_mlen = F.t_mlen.data();
  v->gated = F.gated.data();
  v->ngated = (int64_t)F.gated.size();
  v->n_gated1 = F.n_gated1;
  v->n_up = F.n_up;
  v->t_bias_nslots = F.t_bias_nslots.data();
  v->t_bias_stride = F.t_bias_stride.data();
  v->s_src = F.s_src.data();
  v->s_ncols = F.s_ncols.data();
  v->s_kind = F.s_kind.data();
  v->s_nslots = F.s_nslots.data();
  v->s_stride = F.s_stride.data();
  v->deps = F.deps.data();
  v->mode = F.mode;
  v->group = F.group;
  v->split = 0;
  v->resident = F.resident ? 1 : 0;
  v->u_range = F.u_range.data();
  v->res_mat_max = F.res_mat_max;
  v->res_vec_max = F.res_vec_max;
  v->res_items_max = F.res_items_max;
  v->nunits = F.mode == 1 ? (int64_t)F.unit0.size() - 1 : 0;
  v->nwaves = F.mode == 1 ? (int64_t)F.wave0.size() - 1 : 0;
  v->unit0 = F.unit0.data();
  v->wave0 = F.wave0.data();
}

}  // namespace

extern "C" {

int h2b_abi_version(void) { return H2B_ABI_VERSION; }

const char* h2b_last_error(void) { return g_err.c_str(); }

int h2b_plan_create(const h2b_desc* d, const h2b_options* opt, h2b_plan** out) {
  if (!out) return fail(H2B_EINVAL, "null output pointer");
  *out = nullptr;
  try {
    std::unique_ptr<h2b_plan> p(new h2b_plan());
    std::string err;
    h2b::PlanOptions po = to_plan_options(d, opt);
    po.near_split = po.world_size <= 1 && opt && (opt->plan_flags & H2B_PLAN_NEAR_SPLIT);
    int rc = h2b::build_plan(d, po, &p->plan, &err);
    if (rc != H2B_OK) return fail(rc, err);
    h2b::pack_pool(&p->plan, host_threads());
    fill_stats(p->plan, &p->stats);
    *out = p.release();
    return H2B_OK;
  } catch (const std::bad_alloc&) {
    return fail(H2B_ENOMEM, "host allocation failed while planning");
  }
}

int h2b_plan_view_get(const h2b_plan* p, h2b_plan_view* v) { return h2b_plan_phase_view(p, 0, v); }

int h2b_plan_phases(const h2b_plan* p) { return p ? (int)(p->plan.ph.size() + p->plan.ph_split.size()) : -1; }

int h2b_plan_phase_view(const h2b_plan* p, int phase, h2b_plan_view* v) {
  const int n0 = p ? (int)p->plan.ph.size() : 0;
  if (!p || !v || phase < 0 || phase >= n0 + (int)p->plan.ph_split.size()) return fail(H2B_EINVAL, "bad plan or phase");
  fill_view(p->plan, phase < n0 ? p->plan.ph[phase] : p->plan.ph_split[phase - n0], v);
  v->split = phase < n0 ? 0 : 1;
  return H2B_OK;
}

int h2b_plan_partition(const h2b_plan* p, int64_t* rank_lo_hi, int64_t* exchange) {
  if (!p || !rank_lo_hi || !exchange) return fail(H2B_EINVAL, "null argument");
  const h2b::Plan& P = p->plan;
  for (size_t r = 0; r < P.rank_lo.size(); ++r) {
    rank_lo_hi[2 * r] = P.rank_lo[r];
    rank_lo_hi[2 * r + 1] = P.rank_hi[r];
  }
  exchange[0] = P.exch_off;
  exchange[1] = P.exch_count;
  return H2B_OK;
}

int h2b_plan_stats(const h2b_plan* p, h2b_stats* out) {
  if (!p || !out) return fail(H2B_EINVAL, "null argument");
  *out = p->stats;
  return H2B_OK;
}

void h2b_plan_destroy(h2b_plan* p) { delete p; }

int h2b_create(const h2b_desc* d, const h2b_options* opt, h2b_op** out) {
  try {
    return create_impl(d, opt, out);
  } catch (const std::bad_alloc&) {
    return fail(H2B_ENOMEM, "host allocation failed while creating the operator");
  }
}

int h2b_matvec_dev(h2b_op* op, const double* x_dev, double* y_dev, int nrhs, void* stream) {
  return matvec_dev_impl(op, x_dev, y_dev, nrhs, stream);
}

int h2b_matvec_phase(h2b_op* op, int phase, const double* x_dev, double* y_dev, int nrhs, void* stream) {
  if (!op || phase < 0 || phase > (op->world > 1 ? 1 : 0)) return fail(H2B_EINVAL, "bad operator or phase");
  std::lock_guard<std::mutex> lk(op->mu);
  return matvec_locked(op, phase, x_dev, y_dev, nrhs, stream);
}

int h2b_reset(h2b_op* op) {
  if (!op) return fail(H2B_EINVAL, "null operator");
  std::lock_guard<std::mutex> lk(op->mu);
  return reset_locked(op);
}

int h2b_exchange_region(h2b_op* op, int nrhs, double** base, int64_t* count_per_rank) {
  if (!op || !base || !count_per_rank) return fail(H2B_EINVAL, "null argument");
  *base = op->d_coef + op->exch_off * nrhs;
  *count_per_rank = op->exch_count * nrhs;
  return H2B_OK;
}

int h2b_exchange_copy(h2b_op* dst, const h2b_op* src, int nrhs, void* stream) {
  if (!dst || !src || dst->exch_count != src->exch_count || dst->exch_off != src->exch_off)
    return fail(H2B_EINVAL, "operators do not share an exchange layout");
  const size_t cnt = (size_t)src->exch_count * nrhs;
  const size_t off = (size_t)src->exch_off * nrhs + (size_t)src->rank * cnt;
  if (cnt)
    H2B_CUDA(cudaMemcpyAsync(dst->d_coef + off, src->d_coef + off, sizeof(double) * cnt, cudaMemcpyDefault,
                             (cudaStream_t)stream));
  return H2B_OK;
}

int h2b_matvec(h2b_op* op, const double* x_host, double* y_host, int64_t n, int nrhs) {
  if (!op) return fail(H2B_EINVAL, "null operator");
  if (n != op->n) return fail(H2B_EINVAL, "vector must have shape (" + std::to_string(op->n) + ",)");
  if (!x_host || !y_host) return fail(H2B_EINVAL, "null vector");
  std::lock_guard<std::mutex> lk(op->mu);
  H2B_CUDA(cudaSetDevice(op->device));
  const size_t bytes = sizeof(double) * (size_t)n * (size_t)std::max(1, nrhs);
  if (op->xy_cap < bytes) {
    cudaFree(op->d_x);
    cudaFree(op->d_y);
    op->d_x = op->d_y = nullptr;
    op->xy_cap = 0;
    H2B_CUDA(cudaMalloc(&op->d_x, bytes));
    H2B_CUDA(cudaMalloc(&op->d_y, bytes));
    op->xy_cap = bytes;
  }
  // one stream: copy in, product, copy out, then a single synchronisation
  // (a blocking stream: ordered with the legacy default stream, like before)
  if (!op->hstream) H2B_CUDA(cudaStreamCreate(&op->hstream));
  cudaStream_t st = op->hstream;
  // Host copies: staged through pinned memory by the copy threads (see
  // CopyPool) for vectors of at least 1 MB, else straight from the caller's.
  if (op->copy_threads < 0) {
    const char* e = std::getenv("H2B_COPY_THREADS");
    const int hw = (int)std::thread::hardware_concurrency();
    // Off by default: on the 16-vCPU B200 box the threads' memcpy does not beat the
    // driver's own staging (config 3, h2_matvec from pageable arrays: 2.90 ms plain,
    // 2.87 / 2.86 ms with 4 / 8 threads and 1 MB chunks, 3.1-3.6 ms with 256 KB
    // chunks; profiles/r02_config3_e2e_staged_copies.jsonl)
    (void)hw;
    op->copy_threads = e ? std::max(0, std::min(16, std::atoi(e))) : 0;
    const char* ck = std::getenv("H2B_COPY_CHUNK_KB");
    op->copy_chunk = (size_t)std::max(64, ck ? std::atoi(ck) : 1024) << 10;
  }
  const size_t kChunk = op->copy_chunk;  // bytes per staged chunk
  // vectors already in page-locked memory go straight to the DMA engine
  auto pinned = [](const void* q) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, q) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  };
  const bool big = op->copy_threads > 0 && bytes >= ((size_t)1 << 20);
  const bool staged_x = big && !pinned(x_host);
  const bool staged = big && !pinned(y_host);   // the output side
  const int nchunks = (staged || staged_x) ? (int)((bytes + kChunk - 1) / kChunk) : 0;
  if (staged || staged_x) {
    if (op->pin_cap < bytes) {
      if (op->pin_x) cudaFreeHost(op->pin_x);
      if (op->pin_y) cudaFreeHost(op->pin_y);
      op->pin_x = op->pin_y = nullptr;
      op->pin_cap = 0;
      H2B_CUDA(cudaHostAlloc((void**)&op->pin_x, bytes, cudaHostAllocDefault));
      H2B_CUDA(cudaHostAlloc((void**)&op->pin_y, bytes, cudaHostAllocDefault));
      op->pin_cap = bytes;
    }
    while ((int)op->chunk_ev.size() < nchunks) {
      cudaEvent_t ev;
      H2B_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      op->chunk_ev.push_back(ev);
    }
    if (!op->pool) op->pool.reset(new CopyPool(op->copy_threads - 1));
  }
  if (staged_x) {
    // x: each chunk is copied into pinned memory and handed to the DMA engine
    // by the thread that copied it (chunks are disjoint; their order is free)
    std::atomic<int> bad{0};
    const char* xs = reinterpret_cast<const char*>(x_host);
    char* xp = reinterpret_cast<char*>(op->pin_x);
    char* xd = reinterpret_cast<char*>(op->d_x);
    const int dev = op->device;
    op->pool->parallel_for(nchunks, [&](int i) {
      const size_t o = (size_t)i * kChunk, len = std::min(kChunk, bytes - o);
      std::memcpy(xp + o, xs + o, len);
      if (cudaSetDevice(dev) != cudaSuccess ||
          cudaMemcpyAsync(xd + o, xp + o, len, cudaMemcpyHostToDevice, st) != cudaSuccess)
        bad.store(1);
    });
    if (bad.load()) return fail(H2B_ECUDA, "staged host-to-device copy failed");
  } else {
    H2B_CUDA(cudaMemcpyAsync(op->d_x, x_host, bytes, cudaMemcpyHostToDevice, st));
  }
  int rc = matvec_locked(op, -1, op->d_x, op->d_y, nrhs, st);
  if (rc != H2B_OK) return rc;
  // multi-GPU: every rank wrote its own rows; an all-gather of the owned
  // rows (packed in tree order, padded to the largest rank) assembles the
  // full y everywhere
  if (op->world > 1) {
    if (!op->comm) return fail(H2B_EINVAL, "multi-GPU operator without an NCCL communicator");
    const int nr = std::max(1, nrhs);
    const size_t per = (size_t)op->rows_max * nr;
    if (op->rows_cap < per * op->world) {
      cudaFree(op->d_rows);
      op->d_rows = nullptr;
      op->rows_cap = 0;
      H2B_CUDA(cudaMalloc(&op->d_rows, sizeof(double) * per * op->world));
      op->rows_cap = per * op->world;
    }
    const int64_t lo = op->rank_lo[op->rank], cnt = op->rank_hi[op->rank] - lo;
    double* mine = op->d_rows + per * op->rank;
    h2b_pack_rows_kernel<<<(int)std::min<int64_t>(1184, (cnt * nr + 255) / 256 + 1), 256, 0, st>>>(
        op->d_y, op->d_perm, lo, cnt, nr, mine);
    H2B_NCCL(ncclAllGather(mine, op->d_rows, per, ncclDouble, op->comm, st));
    h2b_unpack_rows_kernel<<<(int)std::min<int64_t>(1184, (n * nr + 255) / 256 + 1), 256, 0, st>>>(
        op->d_rows, op->d_perm, op->d_rank_lo, op->world, n, op->rows_max, nr, op->d_y);
    H2B_CUDA(cudaGetLastError());
  }
  if (staged) {
    // y: DMA chunk by chunk into pinned memory, an event behind each; the
    // copy threads move a chunk to the caller's array as soon as it landed
    char* yp = reinterpret_cast<char*>(op->pin_y);
    const char* yd = reinterpret_cast<const char*>(op->d_y);
    for (int i = 0; i < nchunks; ++i) {
      const size_t o = (size_t)i * kChunk, len = std::min(kChunk, bytes - o);
      H2B_CUDA(cudaMemcpyAsync(yp + o, yd + o, len, cudaMemcpyDeviceToHost, st));
      H2B_CUDA(cudaEventRecord(op->chunk_ev[i], st));
    }
    std::atomic<int> bad{0};
    char* ys = reinterpret_cast<char*>(y_host);
    op->pool->parallel_for(nchunks, [&](int i) {
      const size_t o = (size_t)i * kChunk, len = std::min(kChunk, bytes - o);
      if (cudaEventSynchronize(op->chunk_ev[i]) != cudaSuccess) {
        bad.store(1);
        return;
      }
      std::memcpy(ys + o, yp + o, len);
    });
    if (bad.load()) {
      cudaStreamSynchronize(st);
      return fail(H2B_ECUDA, "staged device-to-host copy failed");
    }
    return H2B_OK;
  }
  H2B_CUDA(cudaMemcpyAsync(y_host, op->d_y, bytes, cudaMemcpyDeviceToHost, st));
  H2B_CUDA(cudaStreamSynchronize(st));
  return H2B_OK;
}

int64_t h2b_stream_bytes(const h2b_op* op) { return op ? op->stats.stream_bytes : -1; }

// The phase the trace covers: the single-GPU product's, or (H2B_TRACE_SPLIT=1
// at create, 8/16 right-hand sides) the dataflow part of the split product.
static PhaseDev& traced_phase(const h2b_op* op) {
  h2b_op* o = const_cast<h2b_op*>(op);
  std::vector<PhaseDev>& list = (o->trace_split && !o->ph_split.empty()) ? o->ph_split : o->ph;
  // H2B_TRACE_PHASE=k: launch k of the list; default: its first dataflow launch
  const char* tp = std::getenv("H2B_TRACE_PHASE");
  if (tp && std::atoi(tp) >= 0 && std::atoi(tp) < (int)list.size()) return list[std::atoi(tp)];
  for (auto& F : list)
    if (F.mode == 0) return F;
  return list[0];
}

int h2b_trace_enable(h2b_op* op, int on) {
  if (!op) return fail(H2B_EINVAL, "null operator");
  H2B_CUDA(cudaSetDevice(op->device));
  PhaseDev& F = traced_phase(op);
  const size_t cnt = 8 * (size_t)std::max<int64_t>(1, F.ntasks);
  if (on && !F.d_trace) {
    H2B_CUDA(cudaMalloc(&F.d_trace, sizeof(unsigned long long) * cnt));
    H2B_CUDA(cudaMemset(F.d_trace, 0, sizeof(unsigned long long) * cnt));
  } else if (!on && F.d_trace) {
    cudaFree(F.d_trace);
    F.d_trace = nullptr;
  }
  return H2B_OK;
}

int h2b_trace_read(const h2b_op* op, uint64_t* out, int64_t nitems) {
  if (!op || !out || nitems != traced_phase(op).ntasks || !traced_phase(op).d_trace)
    return fail(H2B_EINVAL, "trace not enabled or wrong size");
  H2B_CUDA(cudaMemcpy(out, traced_phase(op).d_trace, sizeof(uint64_t) * 8 * nitems, cudaMemcpyDeviceToHost));
  return H2B_OK;
}

int h2b_item_kinds(const h2b_op* op, int32_t* out, int64_t nitems) {
  if (!op || !out || nitems != traced_phase(op).ntasks) return fail(H2B_EINVAL, "wrong size");
  std::vector<DTask> t(nitems);
  H2B_CUDA(cudaMemcpy(t.data(), traced_phase(op).d_tasks, sizeof(DTask) * nitems, cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < nitems; ++i) out[i] = t[i].kind;
  return H2B_OK;
}

int h2b_launch_count(const h2b_op* op, int nrhs) {
  if (!op || nrhs_index(nrhs) < 0) return -1;
  const auto& list = (nrhs >= 8 && !op->ph_split.empty()) ? op->ph_split : op->ph;
  return 1 + (int)list.size();
}

int h2b_launch_info(const h2b_op* op, int nrhs, int launch, int32_t* kind, int64_t* items, int64_t* bytes) {
  const int n = h2b_launch_count(op, nrhs);
  if (n < 0 || launch < 0 || launch >= n || !kind || !items || !bytes) return fail(H2B_EINVAL, "bad launch index");
  if (launch == 0) {
    *kind = -1;
    *items = op->n;
    *bytes = 0;
    return H2B_OK;
  }
  const auto& list = (nrhs >= 8 && !op->ph_split.empty()) ? op->ph_split : op->ph;
  const PhaseDev& F = list[launch - 1];
  *kind = F.mode;
  *items = F.ntasks;
  *bytes = F.bytes;
  return H2B_OK;
}

int h2b_launch_times(h2b_op* op, const double* x_dev, double* y_dev, int nrhs, int steps, void* stream,
                     double* ms_per_launch) {
  if (!op || !ms_per_launch || steps < 1) return fail(H2B_EINVAL, "bad argument");
  if (op->world > 1) return fail(H2B_EINVAL, "h2b_launch_times: single-GPU operators only");
  const int n = h2b_launch_count(op, nrhs);
  if (n < 0) return fail(H2B_EINVAL, "nrhs must be 1, 2, 4, 8 or 16");
  std::lock_guard<std::mutex> lk(op->mu);
  H2B_CUDA(cudaSetDevice(op->device));
  std::vector<cudaEvent_t> ev((size_t)n + 1, nullptr);
  for (auto& e : ev) H2B_CUDA(cudaEventCreate(&e));
  std::vector<double> acc((size_t)n, 0.0);
  int rc = H2B_OK;
  for (int s = 0; s < steps && rc == H2B_OK; ++s) {
    op->tev = &ev;
    op->tev_n = 0;
    rc = matvec_locked(op, -1, x_dev, y_dev, nrhs, stream);
    op->tev = nullptr;
    if (rc != H2B_OK) break;
    if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) { rc = fail(H2B_ECUDA, "synchronize"); break; }
    for (int k = 0; k < n; ++k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
      acc[k] += ms;
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  if (rc != H2B_OK) return rc;
  for (int k = 0; k < n; ++k) ms_per_launch[k] = acc[k] / steps;
  return H2B_OK;
}

int h2b_stats_get(const h2b_op* op, h2b_stats* out) {
  if (!op || !out) return fail(H2B_EINVAL, "null argument");
  *out = op->stats;
  return H2B_OK;
}

void h2b_destroy(h2b_op* op) {
  if (!op) return;
  cudaSetDevice(op->device);
  cudaDeviceSynchronize();
  free_op(op);
}

int h2b_nccl_unique_id(void* out128) {
  if (!out128) return fail(H2B_EINVAL, "null argument");
  ncclUniqueId id;
  H2B_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
  return H2B_OK;
}

}  // extern "C"
