// colloc.cu — collocation entries of the double-layer operator M = K + D on
// the GPU (the 72%-of-build-time host loop of the
// reference, bem.py:99-153 `_panel_rows` called per row by
// CollocationAssembler.block / row_for_point, bem.py:207-235).
//
// One warp per "row job" (a collocation point and a list of column nodes);
// lanes own columns and gather over the node's incident triangles in
// increasing triangle id, the same summation order as the reference's
// np.add.at scatter.  The closed form (solid angle + edge log terms, with the
// coplanarity guard) is evaluated in fp64.  Used by the operator builder
// (paper_1811_05731_b200/assembly), never by the matvec.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/h2b.h"

namespace {

int cfail(int code, const std::string& m);

constexpr int kPanelDoubles = 34;  // v0 v1 v2 (9) n (3) grads (9) gm (9) cop (1) slen (3)

__device__ double panel_value(const double* __restrict__ P, double x0, double x1, double x2, int i) {
  const double a0 = P[0] - x0, a1 = P[1] - x1, a2 = P[2] - x2;
  const double b0 = P[3] - x0, b1 = P[4] - x1, b2 = P[5] - x2;
  const double c0 = P[6] - x0, c1 = P[7] - x1, c2 = P[8] - x2;
  const double ra = sqrt(a0 * a0 + a1 * a1 + a2 * a2);
  const double rb = sqrt(b0 * b0 + b1 * b1 + b2 * b2);
  const double rc = sqrt(c0 * c0 + c1 * c1 + c2 * c2);
  const double n0 = P[9], n1 = P[10], n2 = P[11];
  const double zeta = n0 * a0 + n1 * a1 + n2 * a2;
  const double rmax = fmax(fmax(ra, rb), rc);
  if (fabs(zeta) <= 1e-12 * fmax(rmax, P[30])) return 0.0;  // coplanar guard (bem.py:131-132, 152)
  // signed solid angle (Van Oosterom-Strackee), bem.py:121-128
  const double bxc0 = b1 * c2 - b2 * c1, bxc1 = b2 * c0 - b0 * c2, bxc2 = b0 * c1 - b1 * c0;
  const double det = a0 * bxc0 + a1 * bxc1 + a2 * bxc2;
  const double den = ra * rb * rc + (a0 * b0 + a1 * b1 + a2 * b2) * rc + (b0 * c0 + b1 * c1 + b2 * c2) * ra +
                     (c0 * a0 + c1 * a1 + c2 * a2) * rb;
  const double omega = 2.0 * atan2(det, den);
  // barycentric coordinate of the in-plane projection, bem.py:134-136
  const double p0 = x0 + zeta * n0, p1 = x1 + zeta * n1, p2 = x2 + zeta * n2;
  const double* V = P + 3 * i;
  const double* g = P + 12 + 3 * i;
  const double lam = 1.0 + (g[0] * (p0 - V[0]) + g[1] * (p1 - V[1]) + g[2] * (p2 - V[2]));
  // edge integrals of 1/r, bem.py:138-148
  const double rp[3] = {ra + rb, rb + rc, rc + ra};
  const double* gm = P + 21 + 3 * i;
  double s = 0.0;
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    const double num = rp[e] + P[31 + e];
    const double dnm = rp[e] - P[31 + e];
    const double pe = dnm > 0.0 ? log(num / dnm) : 0.0;
    s += gm[e] * pe;
  }
  return -(lam * omega - zeta * s) / (4.0 * 3.14159265358979323846);
}

__global__ void __launch_bounds__(256) colloc_rows_kernel(
    const double* __restrict__ panels, const int64_t* __restrict__ inc_ptr, const int64_t* __restrict__ inc_tri,
    const int8_t* __restrict__ inc_loc, const double* __restrict__ diag, int64_t njobs,
    const double* __restrict__ points, const int64_t* __restrict__ col_begin, const int32_t* __restrict__ col_count,
    const int64_t* __restrict__ diag_node, const int64_t* __restrict__ out_off, const int64_t* __restrict__ colidx,
    double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t job = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (job >= njobs) return;
  const double x0 = points[3 * job], x1 = points[3 * job + 1], x2 = points[3 * job + 2];
  const int64_t cb = col_begin[job];
  const int cnt = col_count[job];
  const int64_t dn = diag_node[job];
  const int64_t oo = out_off[job];
  for (int c = lane; c < cnt; c += 32) {
    const int64_t v = colidx[cb + c];
    double acc = 0.0;
    for (int64_t k = inc_ptr[v]; k < inc_ptr[v + 1]; ++k)
      acc += panel_value(panels + kPanelDoubles * inc_tri[k], x0, x1, x2, inc_loc[k]);
    if (v == dn) acc += diag[v];  // M = K + D on the diagonal (bem.py:232-234)
    out[oo + c] = acc;
  }
}

#define CC(call)                                                                           \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) return cfail(H2B_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

}  // namespace

struct h2b_colloc {
  int64_t n = 0, ntri = 0;
  double* d_panels = nullptr;
  int64_t* d_inc_ptr = nullptr;
  int64_t* d_inc_tri = nullptr;
  int8_t* d_inc_loc = nullptr;
  double* d_diag = nullptr;
};

namespace h2b_detail {
int set_error(int code, const std::string& msg);  // defined in h2b.cu
}

namespace {
int cfail(int code, const std::string& m) { return h2b_detail::set_error(code, m); }

template <typename T>
int up(T** d, const T* h, size_t n) {
  CC(cudaMalloc((void**)d, sizeof(T) * std::max<size_t>(1, n)));
  if (n) CC(cudaMemcpy(*d, h, sizeof(T) * n, cudaMemcpyHostToDevice));
  return H2B_OK;
}

void colloc_free(h2b_colloc* c) {
  if (!c) return;
  cudaFree(c->d_panels);
  cudaFree(c->d_inc_ptr);
  cudaFree(c->d_inc_tri);
  cudaFree(c->d_inc_loc);
  cudaFree(c->d_diag);
  delete c;
}
}  // namespace

extern "C" {

int h2b_colloc_create(int64_t n, int64_t ntri, const double* panels, const int64_t* inc_ptr,
                      const int64_t* inc_tri, const int8_t* inc_loc, const double* diag, h2b_colloc** out) {
  if (!out || n < 1 || ntri < 1 || !panels || !inc_ptr || !inc_tri || !inc_loc || !diag)
    return cfail(H2B_EINVAL, "h2b_colloc_create: invalid argument");
  *out = nullptr;
  h2b_colloc* c = new h2b_colloc();
  c->n = n;
  c->ntri = ntri;
  const int64_t nnz = inc_ptr[n];
  int rc;
  if ((rc = up(&c->d_panels, panels, (size_t)ntri * kPanelDoubles)) || (rc = up(&c->d_inc_ptr, inc_ptr, (size_t)n + 1)) ||
      (rc = up(&c->d_inc_tri, inc_tri, (size_t)nnz)) || (rc = up(&c->d_inc_loc, inc_loc, (size_t)nnz)) ||
      (rc = up(&c->d_diag, diag, (size_t)n))) {
    colloc_free(c);
    return rc;
  }
  *out = c;
  return H2B_OK;
}

int h2b_colloc_eval(h2b_colloc* c, int64_t njobs, const double* points, const int64_t* col_begin,
                    const int32_t* col_count, const int64_t* diag_node, const int64_t* out_off, int64_t ncolidx,
                    const int64_t* colidx, int64_t out_len, double* out) {
  if (!c || njobs < 0 || !out) return cfail(H2B_EINVAL, "h2b_colloc_eval: invalid argument");
  if (njobs == 0) return H2B_OK;
  double* d_pts = nullptr;
  int64_t *d_cb = nullptr, *d_dn = nullptr, *d_oo = nullptr, *d_ci = nullptr;
  int32_t* d_cc = nullptr;
  double* d_out = nullptr;
  int rc = H2B_OK;
  do {
    if ((rc = up(&d_pts, points, (size_t)njobs * 3)) || (rc = up(&d_cb, col_begin, (size_t)njobs)) ||
        (rc = up(&d_cc, col_count, (size_t)njobs)) || (rc = up(&d_dn, diag_node, (size_t)njobs)) ||
        (rc = up(&d_oo, out_off, (size_t)njobs)) || (rc = up(&d_ci, colidx, (size_t)ncolidx)))
      break;
    cudaError_t e = cudaMalloc(&d_out, sizeof(double) * std::max<int64_t>(1, out_len));
    if (e != cudaSuccess) { rc = cfail(H2B_ECUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e)); break; }
    const int wpb = 8;
    const int64_t blocks = (njobs + wpb - 1) / wpb;
    colloc_rows_kernel<<<(unsigned)blocks, wpb * 32>>>(c->d_panels, c->d_inc_ptr, c->d_inc_tri, c->d_inc_loc,
                                                       c->d_diag, njobs, d_pts, d_cb, d_cc, d_dn, d_oo, d_ci, d_out);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(out, d_out, sizeof(double) * out_len, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) { rc = cfail(H2B_ECUDA, std::string("colloc kernel: ") + cudaGetErrorString(e)); break; }
  } while (0);
  cudaFree(d_pts); cudaFree(d_cb); cudaFree(d_cc); cudaFree(d_dn); cudaFree(d_oo); cudaFree(d_ci); cudaFree(d_out);
  return rc;
}

void h2b_colloc_destroy(h2b_colloc* c) { colloc_free(c); }

}  // extern "C"
