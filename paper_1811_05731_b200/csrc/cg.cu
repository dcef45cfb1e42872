// cg.cu — the FEM solves either side of the boundary operator on the GPU
// (SURVEY §8f row 3): Jacobi-preconditioned conjugate gradients with
// optional deflation of the constant mode, restating the reference's
// cg_solve (solver.py:44-98) as used by solve_u1 / solve_u2 (fem.py:79-121).
//
// One cooperative persistent kernel runs the whole solve: every CTA owns a
// contiguous range of rows, three grid-wide barriers per iteration separate
// the sparse product, the vector updates and the direction update.  Scalars
// (p'Ap, r'z, sum z, sum r, r'r) are per-CTA partial sums that EVERY CTA then
// reduces in the same fixed order after the barrier, so all CTAs hold
// bit-identical scalars without another barrier, and the result does not
// depend on scheduling (deterministic, no float atomics).
//
// Differences from the reference are floating-point rounding only: the dot
// products are summed in a different order than numpy's, and r'z of the
// deflated z is formed as r'z0 - mean(z0) sum(r) (the same value in exact
// arithmetic).  Iterates therefore agree to the solve tolerance, not bit for
// bit.  The sparse product is HBM-bound (12 bytes per stored entry plus the
// vectors); four lanes per row.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "../../include/h2b.h"

namespace cgk = cooperative_groups;

namespace h2b_detail {
int set_error(int code, const std::string& msg);
}

namespace {

int gfail(int code, const std::string& m) { return h2b_detail::set_error(code, m); }

#define CG_CUDA(call)                                                                       \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) return gfail(H2B_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr int kThreads = 256;
constexpr int kLanesPerRow = 4;
constexpr size_t kRpSmemPerSm = 200 * 1024;  // row-pointer cache budget per SM
constexpr int kParts = 5;  // partial sums per CTA: p'Ap | r'z0, sum z0, sum r, r'r

struct CGParams {
  int64_t n;
  const int64_t* __restrict__ rp;
  const int32_t* __restrict__ ci;
  const double* __restrict__ va;
  const double* __restrict__ inv;  // 1 / diag(A)
  const double* __restrict__ b;
  double* x;
  double* r;
  double* z;  // preconditioned residual before deflation (z0)
  double* p;
  double* ap;
  double* part;  // [gridDim.x * kParts]
  double* out;   // [4]: iterations, final relative residual, status, ||b||
  double tol;
  int64_t max_iter;
  int deflate;
  int rp_smem;  // the CTA's row pointers cached in dynamic shared memory (32-bit, relative)
};

// Block sum of v (all threads get it); scratch: kThreads/32 doubles.
__device__ double block_sum(double v, double* scratch) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) scratch[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += scratch[i];  // fixed order
  return s;
}

// Sum of part[k] over all CTAs in CTA order (the same in every CTA).
__device__ double grid_total(const double* part, int k, double* scratch) {
  double v = 0.0;
  // each thread a strided subset, then a fixed-order block sum: identical in
  // every CTA because the split depends only on blockDim and gridDim
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) v += __ldcg(part + (int64_t)i * kParts + k);
  return block_sum(v, scratch);
}

__device__ void rows_of_block(int64_t n, int64_t* lo, int64_t* hi) {
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  *lo = (int64_t)blockIdx.x * per;
  *hi = min(n, *lo + per);
}

// U: rows per lane group per pass of the sparse product; MINB: co-resident
// CTAs per SM the register allocation is bounded for.
// NT: threads per CTA; PF: passes ahead whose entries are prefetched to L2
// (needs the row pointers in shared memory).
template <int U, int MINB, int NT = kThreads, int PF = 0>
__global__ void __launch_bounds__(NT, MINB) cg_kernel(CGParams P) {
  cgk::grid_group grid = cgk::this_grid();
  __shared__ double scratch[NT / 32];
  extern __shared__ int32_t rps[];  // rp[lo..hi] - rp[lo] when P.rp_smem
  int64_t lo, hi;
  rows_of_block(P.n, &lo, &hi);
  const int tid = threadIdx.x;
  const int64_t n = P.n;
  // The matrix is fixed for the solve: with the row pointers in shared
  // memory a pass of the sparse product has two dependent global round trips
  // (entries, then the gathers of p) instead of three.
  const int64_t ebase = lo < hi ? P.rp[lo] : 0;
  if (P.rp_smem)
    for (int64_t i = lo + tid; i <= hi; i += blockDim.x) rps[i - lo] = (int32_t)(P.rp[i] - ebase);

  // ---- setup: ||b||, deflated b, x = 0, r = b, z0 = inv r
  double s_bb = 0.0, s_b = 0.0;
  for (int64_t i = lo + tid; i < hi; i += blockDim.x) {
    const double bi = P.b[i];
    s_bb += bi * bi;
    s_b += bi;
  }
  s_bb = block_sum(s_bb, scratch);
  s_b = block_sum(s_b, scratch);
  if (tid == 0) {
    P.part[blockIdx.x * kParts + 0] = s_bb;
    P.part[blockIdx.x * kParts + 1] = s_b;
  }
  grid.sync();
  const double bnorm = sqrt(grid_total(P.part, 0, scratch));
  const double bmean = P.deflate ? grid_total(P.part, 1, scratch) / (double)n : 0.0;
  if (bnorm == 0.0) {
    for (int64_t i = lo + tid; i < hi; i += blockDim.x) P.x[i] = 0.0;
    if (blockIdx.x == 0 && tid == 0) {
      P.out[0] = 0.0;
      P.out[1] = 0.0;
      P.out[2] = 0.0;
      P.out[3] = 0.0;
    }
    return;
  }
  grid.sync();  // every CTA has read the setup partials
  double s_rz = 0.0, s_z = 0.0, s_r = 0.0, s_rr = 0.0;
  for (int64_t i = lo + tid; i < hi; i += blockDim.x) {
    const double ri = P.b[i] - bmean;
    const double zi = P.inv[i] * ri;
    P.x[i] = 0.0;
    P.r[i] = ri;
    P.z[i] = zi;
    s_rz += ri * zi;
    s_z += zi;
    s_r += ri;
    s_rr += ri * ri;
  }
  s_rz = block_sum(s_rz, scratch);
  s_z = block_sum(s_z, scratch);
  s_r = block_sum(s_r, scratch);
  s_rr = block_sum(s_rr, scratch);
  if (tid == 0) {
    double* q = P.part + blockIdx.x * kParts;
    q[1] = s_rz;
    q[2] = s_z;
    q[3] = s_r;
    q[4] = s_rr;
  }
  grid.sync();
  double zmean = P.deflate ? grid_total(P.part, 2, scratch) / (double)n : 0.0;
  double rz = grid_total(P.part, 1, scratch) - zmean * grid_total(P.part, 3, scratch);
  double res = sqrt(grid_total(P.part, 4, scratch)) / bnorm;
  for (int64_t i = lo + tid; i < hi; i += blockDim.x) P.p[i] = P.z[i] - zmean;  // p = z
  int64_t it = 0;
  double status = 0.0;
  grid.sync();

  const int sub = tid / kLanesPerRow, sl = tid % kLanesPerRow;
  const int rows_per_pass = NT / kLanesPerRow;
  while (res > P.tol && it < P.max_iter) {
    // ---- A: ap = A p on this CTA's rows, partial p'Ap
    // U rows per lane group per pass, all their loads issued together
    // (the row pointers, then up to 4 entries per lane of each row, then
    // the gathers): the sparse product is latency-bound otherwise.  The
    // per-lane and per-row summation order is that of a row-at-a-time loop.
    double s_pap = 0.0;
    for (int64_t r0 = lo; r0 < hi; r0 += (int64_t)rows_per_pass * U) {
      int64_t e0[U], e1[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t ik = r0 + k * rows_per_pass + sub;
        if (P.rp_smem) {
          e0[k] = ik < hi ? ebase + rps[ik - lo] : 0;
          e1[k] = ik < hi ? ebase + rps[ik - lo + 1] : 0;
        } else {
          e0[k] = ik < hi ? __ldg(P.rp + ik) : 0;
          e1[k] = ik < hi ? __ldg(P.rp + ik + 1) : 0;
        }
      }
      double v[U];
      int c[U][4];
      double a[U][4];
#pragma unroll
      for (int k = 0; k < U; ++k)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t eu = e0[k] + sl + u * kLanesPerRow;
          c[k][u] = eu < e1[k] ? __ldg(P.ci + eu) : -1;
          a[k][u] = eu < e1[k] ? __ldg(P.va + eu) : 0.0;
        }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        double q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) q[u] = c[k][u] >= 0 ? __ldcg(P.p + c[k][u]) : 0.0;
        v[k] = 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) v[k] += a[k][u] * q[u];
      }
      // rows longer than 4 entries per lane
#pragma unroll
      for (int k = 0; k < U; ++k)
        for (int64_t e = e0[k] + sl + 4 * kLanesPerRow; e < e1[k]; e += 4 * kLanesPerRow) {
          int cc[4];
          double aa[4], q[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int64_t eu = e + u * kLanesPerRow;
            cc[u] = eu < e1[k] ? __ldg(P.ci + eu) : -1;
            aa[u] = eu < e1[k] ? __ldg(P.va + eu) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) q[u] = cc[u] >= 0 ? __ldcg(P.p + cc[u]) : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u) v[k] += aa[u] * q[u];
        }
#pragma unroll
      for (int k = 0; k < U; ++k) {
#pragma unroll
        for (int o = kLanesPerRow / 2; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o, kLanesPerRow);
        const int64_t ik = r0 + k * rows_per_pass + sub;
        if (ik < hi && sl == 0) {
          P.ap[ik] = v[k];
          s_pap += v[k] * P.p[ik];
        }
      }
      // L2 prefetch of the entries PF passes ahead (one 128-byte line of va
      // or ci per thread): their loads then wait on L2, not HBM
      if (PF > 0 && P.rp_smem) {
        const int64_t pass = (int64_t)rows_per_pass * U;
        const int64_t a = r0 + PF * pass;
        if (a < hi) {
          const int64_t b = min(hi, a + pass);
          const int64_t f0 = ebase + rps[a - lo], f1 = ebase + rps[b - lo];
          const char* va0 = (const char*)(P.va + f0);
          const char* ci0 = (const char*)(P.ci + f0);
          const int64_t nva = ((const char*)(P.va + f1) - va0 + 127) >> 7;
          const int64_t nci = ((const char*)(P.ci + f1) - ci0 + 127) >> 7;
          for (int64_t j = tid; j < nva + nci; j += NT) {
            const char* addr = j < nva ? va0 + (j << 7) : ci0 + ((j - nva) << 7);
            asm volatile("prefetch.global.L2 [%0];" ::"l"(addr));
          }
        }
      }
    }
    s_pap = block_sum(s_pap, scratch);
    if (tid == 0) P.part[blockIdx.x * kParts + 0] = s_pap;
    grid.sync();
    // ---- B: alpha; x += alpha p, r -= alpha ap, z0 = inv r; partials
    const double pap = grid_total(P.part, 0, scratch);
    if (!(pap > 0.0)) {
      status = 1.0;  // negative curvature (solver.py:85-86)
      break;
    }
    const double alpha = rz / pap;
    s_rz = s_z = s_r = s_rr = 0.0;
    for (int64_t i = lo + tid; i < hi; i += blockDim.x) {
      const double pi = P.p[i];
      P.x[i] += alpha * pi;
      const double ri = P.r[i] - alpha * P.ap[i];
      P.r[i] = ri;
      const double zi = P.inv[i] * ri;
      P.z[i] = zi;
      s_rz += ri * zi;
      s_z += zi;
      s_r += ri;
      s_rr += ri * ri;
    }
    s_rz = block_sum(s_rz, scratch);
    s_z = block_sum(s_z, scratch);
    s_r = block_sum(s_r, scratch);
    s_rr = block_sum(s_rr, scratch);
    if (tid == 0) {
      double* q = P.part + blockIdx.x * kParts;
      q[1] = s_rz;
      q[2] = s_z;
      q[3] = s_r;
      q[4] = s_rr;
    }
    grid.sync();
    // ---- C: beta; p = (z0 - mean) + beta p
    zmean = P.deflate ? grid_total(P.part, 2, scratch) / (double)n : 0.0;
    const double rz_new = grid_total(P.part, 1, scratch) - zmean * grid_total(P.part, 3, scratch);
    const double beta = rz_new / rz;
    for (int64_t i = lo + tid; i < hi; i += blockDim.x) P.p[i] = (P.z[i] - zmean) + beta * P.p[i];
    rz = rz_new;
    ++it;
    res = sqrt(grid_total(P.part, 4, scratch)) / bnorm;
    grid.sync();
  }
  // deflated solution: zero mean (solver.py:96-97)
  if (P.deflate && status == 0.0) {
    double s_x = 0.0;
    for (int64_t i = lo + tid; i < hi; i += blockDim.x) s_x += P.x[i];
    s_x = block_sum(s_x, scratch);
    if (tid == 0) P.part[blockIdx.x * kParts + 0] = s_x;
    grid.sync();
    const double xmean = grid_total(P.part, 0, scratch) / (double)n;
    for (int64_t i = lo + tid; i < hi; i += blockDim.x) P.x[i] -= xmean;
  }
  if (blockIdx.x == 0 && tid == 0) {
    P.out[0] = (double)it;
    P.out[1] = res;
    P.out[2] = status;
    P.out[3] = bnorm;
  }
}

__global__ void inv_diag_kernel(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                const double* __restrict__ va, double* inv, int* zero) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double d = 0.0;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e)
      if (ci[e] == i) d += va[e];
    if (d == 0.0) atomicExch(zero, 1);
    inv[i] = 1.0 / d;
  }
}

}  // namespace

struct h2b_cg {
  int device = 0;
  int64_t n = 0, nnz = 0;
  int64_t* rp = nullptr;
  int32_t* ci = nullptr;
  double* va = nullptr;
  double* inv = nullptr;
  double *x = nullptr, *r = nullptr, *z = nullptr, *p = nullptr, *ap = nullptr, *part = nullptr, *out = nullptr;
  double* hb = nullptr;  // host path: device b
  int grid = 0;
  const void* kernel = nullptr;
  int threads = kThreads;
  size_t smem = 0;  // dynamic shared memory: the CTA's row pointers, or 0
};

namespace {
void cg_free(h2b_cg* c) {
  if (!c) return;
  cudaFree(c->rp);
  cudaFree(c->ci);
  cudaFree(c->va);
  cudaFree(c->inv);
  cudaFree(c->x);
  cudaFree(c->r);
  cudaFree(c->z);
  cudaFree(c->p);
  cudaFree(c->ap);
  cudaFree(c->part);
  cudaFree(c->out);
  cudaFree(c->hb);
  delete c;
}

int cg_create_impl(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val, h2b_cg* c) {
  c->n = n;
  c->nnz = row_ptr[n];
  CG_CUDA(cudaGetDevice(&c->device));
  CG_CUDA(cudaMalloc(&c->rp, sizeof(int64_t) * (n + 1)));
  CG_CUDA(cudaMalloc(&c->ci, sizeof(int32_t) * std::max<int64_t>(1, c->nnz)));
  CG_CUDA(cudaMalloc(&c->va, sizeof(double) * std::max<int64_t>(1, c->nnz)));
  CG_CUDA(cudaMemcpy(c->rp, row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
  CG_CUDA(cudaMemcpy(c->ci, col, sizeof(int32_t) * c->nnz, cudaMemcpyHostToDevice));
  CG_CUDA(cudaMemcpy(c->va, val, sizeof(double) * c->nnz, cudaMemcpyHostToDevice));
  for (double** v : {&c->inv, &c->x, &c->r, &c->z, &c->p, &c->ap, &c->hb})
    CG_CUDA(cudaMalloc(v, sizeof(double) * std::max<int64_t>(1, n)));
  // Kernel variant: rows per lane group and CTAs per SM (H2B_CG_VARIANT;
  // tools/cg_bench.py compares them; <U, CTAs per SM[, threads]>).  913k-node cube, us per iteration with
  // / without the row pointers in shared memory: <2,4> 76 / 80, <1,4> 77 /
  // 86, <2,3> 80 / 86, <4,2> (128 registers) 88 / 91.
  static const struct {
    const void* fn;
    int minb;
    int threads;
  } variants[] = {{(const void*)cg_kernel<2, 4>, 4, kThreads},      {(const void*)cg_kernel<4, 2>, 2, kThreads},
                  {(const void*)cg_kernel<2, 3>, 3, kThreads},      {(const void*)cg_kernel<1, 4>, 4, kThreads},
                  {(const void*)cg_kernel<2, 2, 512, 2>, 2, 512},   {(const void*)cg_kernel<2, 1, 1024>, 1, 1024},
                  {(const void*)cg_kernel<2, 2, 512>, 2, 512}};
  int nsm0 = 0;
  CG_CUDA(cudaDeviceGetAttribute(&nsm0, cudaDevAttrMultiProcessorCount, c->device));
  // default: 512 threads at 2 CTAs per SM (half the CTAs at each grid
  // barrier) with the entries two passes ahead prefetched to L2, while its
  // row pointers fit 100 KB of shared memory, else 256 at 4.  us per
  // iteration: 913 k nodes 72-74 vs 76-77 without the prefetch, 69.5-71 with
  // (1 / 3 / 4 passes ahead: 71 / 73.4 / 77); 118 k 18.6 vs 19.0; 2.1 M 150.6
  // vs 155.3 without the prefetch; 4.17 M 295-296 vs 296 (317 when its row
  // pointers were limited to 48 KB and read from global memory)
  // (profiles/r01_cg_variants_512.log, r01_cg_prefetch.log, r01_cg_rp_smem_200k.log).
  int v = sizeof(int32_t) * (size_t)((n + 2 * nsm0 - 1) / (2 * nsm0) + 1) <= kRpSmemPerSm / 2 ? 4 : 0;
  if (const char* e = getenv("H2B_CG_VARIANT")) v = std::min(std::max(atoi(e), 0), 6);
  const int nt = variants[v].threads;
  c->threads = nt;
  c->kernel = variants[v].fn;
  int per_sm = 0, nsm = 0;
  CG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
  // co-resident CTAs for the grid barrier: the variant's count per SM (the
  // gathers of the sparse product need the memory-level parallelism; every
  // CTA reads all partial sums after a barrier, so more CTAs cost L2 traffic)
  const int want = variants[v].minb;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)want * nsm, (n + nt - 1) / nt));
  const int64_t per_cta = (n + grid - 1) / grid;
  size_t smem = sizeof(int32_t) * (per_cta + 1);
  const char* no_smem = getenv("H2B_CG_RP_SMEM");
  // up to ~200 KB of row pointers per SM (beyond 48 KB per CTA by opt-in)
  if (smem > kRpSmemPerSm / (size_t)want || (no_smem && atoi(no_smem) == 0)) smem = 0;
  if (smem > 48 * 1024)
    CG_CUDA(cudaFuncSetAttribute(c->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, c->kernel, nt, smem));
  if (per_sm < want && smem) {
    smem = 0;
    CG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, c->kernel, nt, 0));
  }
  if (per_sm < 1) return gfail(H2B_ECUDA, "cg kernel does not fit on an SM");
  c->grid = (int)std::min<int64_t>(grid, (int64_t)per_sm * nsm);
  if (c->grid < grid) smem = 0;  // rows per CTA changed; use the global row pointers
  c->smem = smem;
  CG_CUDA(cudaMalloc(&c->part, sizeof(double) * kParts * c->grid));
  CG_CUDA(cudaMalloc(&c->out, sizeof(double) * 4));
  int* d_zero = nullptr;
  CG_CUDA(cudaMalloc(&d_zero, sizeof(int)));
  cudaError_t e = cudaMemset(d_zero, 0, sizeof(int));
  if (e == cudaSuccess) {
    inv_diag_kernel<<<std::max<int64_t>(1, std::min<int64_t>(1184, (n + 255) / 256)), 256>>>(n, c->rp, c->ci, c->va,
                                                                                              c->inv, d_zero);
    e = cudaGetLastError();
  }
  int zero = 0;
  if (e == cudaSuccess) e = cudaMemcpy(&zero, d_zero, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(d_zero);
  if (e != cudaSuccess) return gfail(H2B_ECUDA, std::string("inv_diag: ") + cudaGetErrorString(e));
  if (zero) return gfail(H2B_EINVAL, "Jacobi preconditioner requires a zero-free diagonal");
  return H2B_OK;
}
}  // namespace

extern "C" {

int h2b_cg_create(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val, h2b_cg** out) {
  if (!out || n < 1 || !row_ptr || !col || !val) return gfail(H2B_EINVAL, "h2b_cg_create: invalid argument");
  if (row_ptr[0] != 0) return gfail(H2B_EINVAL, "h2b_cg_create: row_ptr[0] must be 0");
  for (int64_t i = 0; i < n; ++i)
    if (row_ptr[i + 1] < row_ptr[i]) return gfail(H2B_EINVAL, "h2b_cg_create: row_ptr must be nondecreasing");
  for (int64_t e = 0; e < row_ptr[n]; ++e)
    if (col[e] < 0 || col[e] >= n) return gfail(H2B_EINVAL, "h2b_cg_create: column index out of range");
  h2b_cg* c = new h2b_cg();
  const int rc = cg_create_impl(n, row_ptr, col, val, c);
  if (rc != H2B_OK) {
    cg_free(c);
    return rc;
  }
  *out = c;
  return H2B_OK;
}

int h2b_cg_solve_dev(h2b_cg* c, const double* b_dev, double* x_dev, double tol, int deflate, int64_t max_iter,
                     int64_t* iterations, double* residual, void* stream) {
  if (!c || !b_dev || !x_dev) return gfail(H2B_EINVAL, "h2b_cg_solve_dev: invalid argument");
  CG_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  CGParams P;
  P.n = c->n;
  P.rp = c->rp;
  P.ci = c->ci;
  P.va = c->va;
  P.inv = c->inv;
  P.b = b_dev;
  P.x = x_dev;
  P.r = c->r;
  P.z = c->z;
  P.p = c->p;
  P.ap = c->ap;
  P.part = c->part;
  P.out = c->out;
  P.tol = tol;
  P.max_iter = max_iter > 0 ? max_iter : 10 * c->n;  // solver.py:62-63
  P.deflate = deflate ? 1 : 0;
  P.rp_smem = c->smem ? 1 : 0;
  void* args[] = {&P};
  CG_CUDA(cudaLaunchCooperativeKernel(c->kernel, dim3(c->grid), dim3(c->threads), args, c->smem, st));
  double out[4];
  CG_CUDA(cudaMemcpyAsync(out, c->out, sizeof(out), cudaMemcpyDeviceToHost, st));
  CG_CUDA(cudaStreamSynchronize(st));
  if (iterations) *iterations = (int64_t)out[0];
  if (residual) *residual = out[1];
  if (out[2] != 0.0) return gfail(H2B_ECONV, "negative curvature encountered in CG");
  return H2B_OK;
}

int h2b_cg_solve(h2b_cg* c, const double* b_host, double* x_host, double tol, int deflate, int64_t max_iter,
                 int64_t* iterations, double* residual) {
  if (!c || !b_host || !x_host) return gfail(H2B_EINVAL, "h2b_cg_solve: invalid argument");
  CG_CUDA(cudaSetDevice(c->device));
  CG_CUDA(cudaMemcpy(c->hb, b_host, sizeof(double) * c->n, cudaMemcpyHostToDevice));
  int rc = h2b_cg_solve_dev(c, c->hb, c->x, tol, deflate, max_iter, iterations, residual, nullptr);
  if (rc != H2B_OK) return rc;
  CG_CUDA(cudaMemcpy(x_host, c->x, sizeof(double) * c->n, cudaMemcpyDeviceToHost));
  return H2B_OK;
}

void h2b_cg_destroy(h2b_cg* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  cg_free(c);
}

}  // extern "C"
