// plan.cpp — builds the work-item queue for one H² operator (host only).
//
// Semantics follow the reference matvec h2_matvec (h2.py:186-244) exactly:
//   forward   x^_leaf = W_t^T x|_t ; x^_p = sum_c F_c^T x^_c   (h2.py:195-209)
//   coupling  y^_t   += S_b x^_s                               (h2.py:211-218)
//   backward  coeff_c = E_c coeff_p + y^_c ; y|_t += V_t coeff  (h2.py:220-235)
//   near      y|_t   += N_ts x|_s                              (h2.py:237-240)
// The backward recursion's "coeff" of a cluster is materialised as the
// vector y^_c (own coupling rows plus the transferred parent coefficient),
// so coupling and the downward pass fuse into one item per cluster.
#include "plan.h"

#include <algorithm>
#include <functional>
#include <queue>
#include <unordered_map>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <thread>

namespace h2b {
namespace {

struct Vec {
  int64_t off = -1;   // coefficient-pool offset of slot 0
  int32_t len = 0;    // entries per slot
  int32_t nslots = 0; // partial sums to add
  std::vector<int32_t> producers;  // provisional task ids
  bool exists() const { return off >= 0 && len > 0; }
};

struct SegSpec {
  int32_t kind;           // SegKind
  int64_t src;            // tree position (x) or pool offset (coef)
  int32_t ncols;
  const Vec* vec;         // coef source (nullptr for x)
  const double* a;        // source matrix block
  bool transpose;         // false: a is (ncols x m) row-major == (m x ncols) col-major
                          // true : a is (m x ncols) row-major with row stride a_ld
  int64_t a_ld;
};

struct Piece {
  int64_t col0 = 0, ncols = 0;
  // (segment index, first column inside it, columns)
  std::vector<std::array<int64_t, 3>> parts;
};

struct TaskTmp {
  int64_t data;      // pool offset (set once the groups have their bases)
  int32_t group;     // pool group
  int64_t goff;      // offset inside the group
  int64_t out, bias;
  int32_t m, ld, ncols, kind, bias_nslots, bias_stride;
  int32_t stage;
  int32_t qclass = 0;
  int32_t cl = 0;                // cluster (row cluster for down/near/final)
  bool transfer = false;         // down item holding the parent-transfer segment (the chain link)
  std::vector<int32_t> seg_idx;  // into seg tables
  std::vector<int32_t> deps;     // provisional ids
};

class Builder {
 public:
  Builder(const h2b_desc* d, const PlanOptions& o, Plan* p) : d_(d), opt_(o), plan_(p) {}

  int run(std::string* err);

 private:
  const h2b_desc* d_;
  PlanOptions opt_;
  Plan* plan_;

  std::vector<int32_t> parent_, depth_, height_;
  std::vector<int32_t> order_;              // clusters in preorder
  std::vector<int32_t> leaves_;             // preorder == position order
  // staged plans: root of the bottom subtree containing each cluster, or -1
  // for the clusters above the subtrees ("top")
  std::vector<int32_t> broot_;
  std::vector<std::vector<int32_t>> units_;  // clusters of every bottom subtree (preorder), roots in tree order
  bool top(int32_t c) const { return broot_.empty() || broot_[c] < 0; }
  void mark_bottom_subtrees();
  // a sweep phase from provisional task ids: units by bottom subtree (tree
  // order), waves by dependency depth inside the unit
  int finalize_sweep(Phase* F, const std::vector<int32_t>& ids, std::string* err);
  std::vector<Vec> xhat_, yhat_, nearv_;
  std::vector<TaskTmp> tasks_;
  int32_t cur_cl_ = 0;  // cluster of the group being emitted
  int32_t cur_region_ = 0;  // Group::region / unit of the group being emitted
  int64_t cur_unit_ = 0;
  // finish one phase from provisional task ids (any order); deps outside
  // `in_phase` are dropped (satisfied before the phase starts)
  int finalize(Phase* F, std::vector<int32_t> ids, const std::vector<char>& in_phase, std::string* err);
  // segment tables (final)
  std::vector<int64_t> s_src_;
  std::vector<int32_t> s_ncols_, s_kind_, s_nslots_, s_stride_;

  int64_t size(int32_t c) const { return d_->cl_end[c] - d_->cl_start[c]; }
  bool is_leaf(int32_t c) const { return d_->cl_child[2 * c] < 0; }

  int validate(std::string* err);
  // a (r x q) row-major times b (q x c) row-major -> owned (r x c) row-major
  const double* product(const double* a, const double* b, int64_t r, int64_t q, int64_t c) {
    auto buf = std::make_unique<std::vector<double>>((size_t)(r * c), 0.0);
    double* o = buf->data();
    for (int64_t i = 0; i < r; ++i)
      for (int64_t k = 0; k < q; ++k) {
        const double v = a[i * q + k];
        for (int64_t j = 0; j < c; ++j) o[i * c + j] += v * b[k * c + j];
      }
    plan_->extra_bytes += 8 * r * c;
    plan_->owned.push_back(std::move(buf));
    return plan_->owned.back()->data();
  }
  // pool offsets of the groups used by the selected tasks (in group order)
  void assign_bases(const std::vector<char>& sel);
  void alloc_vec(Vec* v, int32_t len, int32_t nslots) {
    v->len = len;
    v->nslots = nslots;
    v->off = plan_->coef_len;
    plan_->coef_len += (int64_t)len * nslots;
  }
  // Packs the group's matrix, splits it into pieces, emits tasks.
  void emit_group(int32_t kind, int32_t stage, int32_t m_total, std::vector<SegSpec>& segs,
                  Vec* outv, int64_t y_pos, const Vec* bias, bool allow_split, int32_t qclass = 0,
                  bool seg0_hi = false, bool append = false);
  void collect_leaves(int32_t c, std::vector<int32_t>* out) const {
    if (is_leaf(c)) { out->push_back(c); return; }
    collect_leaves((int32_t)d_->cl_child[2 * c], out);
    collect_leaves((int32_t)d_->cl_child[2 * c + 1], out);
  }
};

int Builder::validate(std::string* err) {
  const h2b_desc* d = d_;
  if (!d) { *err = "null descriptor"; return H2B_EINVAL; }
  if (d->n < 1) { *err = "n must be >= 1"; return H2B_EINVAL; }
  if (d->nclusters < 1 || d->nclusters > INT32_MAX / 2) { *err = "bad nclusters"; return H2B_EINVAL; }
  if (!d->perm || !d->cl_start || !d->cl_end || !d->cl_child || !d->k_row || !d->k_col) {
    *err = "null tree array"; return H2B_EINVAL;
  }
  const int64_t n = d->n, nc = d->nclusters;
  {
    std::vector<uint8_t> seen(n, 0);
    for (int64_t i = 0; i < n; ++i) {
      int64_t v = d->perm[i];
      if (v < 0 || v >= n || seen[v]) { *err = "perm is not a permutation of range(n)"; return H2B_EINVAL; }
      seen[v] = 1;
    }
  }
  if (d->cl_start[0] != 0 || d->cl_end[0] != n) { *err = "cluster 0 must be the root [0, n)"; return H2B_EINVAL; }
  parent_.assign(nc, -2);
  depth_.assign(nc, 0);
  height_.assign(nc, 0);
  parent_[0] = -1;
  // preorder walk with explicit stack; checks that children partition parents
  std::vector<int32_t> order;
  order.reserve(nc);
  std::vector<int32_t> stack{0};
  while (!stack.empty()) {
    int32_t c = stack.back();
    stack.pop_back();
    order.push_back(c);
    if (d->cl_start[c] < 0 || d->cl_end[c] > n || d->cl_start[c] >= d->cl_end[c]) {
      *err = "cluster " + std::to_string(c) + " has an empty or out-of-range index range";
      return H2B_EINVAL;
    }
    if (d->k_row[c] < 0 || d->k_col[c] < 0 || d->k_row[c] > INT32_MAX / 64 || d->k_col[c] > INT32_MAX / 64) {
      *err = "negative or huge rank"; return H2B_EINVAL;
    }
    int64_t a = d->cl_child[2 * c], b = d->cl_child[2 * c + 1];
    if (a < 0 && b < 0) {
      if (d->cl_end[c] - d->cl_start[c] > INT32_MAX / 64) { *err = "leaf too large"; return H2B_EINVAL; }
      continue;
    }
    if (a < 0 || b < 0 || a >= nc || b >= nc) { *err = "cluster " + std::to_string(c) + " must have 0 or 2 valid children"; return H2B_EINVAL; }
    if (parent_[a] != -2 || parent_[b] != -2 || a == 0 || b == 0) { *err = "cluster tree is not a tree"; return H2B_EINVAL; }
    if (d->cl_start[a] != d->cl_start[c] || d->cl_end[a] != d->cl_start[b] || d->cl_end[b] != d->cl_end[c]) {
      *err = "children of cluster " + std::to_string(c) + " do not partition its range"; return H2B_EINVAL;
    }
    parent_[a] = c; parent_[b] = c;
    depth_[a] = depth_[c] + 1; depth_[b] = depth_[c] + 1;
    stack.push_back((int32_t)b);
    stack.push_back((int32_t)a);
  }
  if ((int64_t)order.size() != nc) { *err = "clusters unreachable from the root"; return H2B_EINVAL; }
  for (auto it = order.rbegin(); it != order.rend(); ++it) {
    int32_t c = *it;
    if (!is_leaf(c)) {
      int32_t a = (int32_t)d->cl_child[2 * c], b = (int32_t)d->cl_child[2 * c + 1];
      height_[c] = 1 + std::max(height_[a], height_[b]);
    }
  }
  for (int32_t c : order) if (is_leaf(c)) leaves_.push_back(c);
  order_ = order;
  // bases / transfers
  for (int64_t c = 0; c < nc; ++c) {
    if (is_leaf((int32_t)c)) {
      if ((d->k_row[c] > 0 && (!d->row_basis || !d->row_basis[c])) ||
          (d->k_col[c] > 0 && (!d->col_basis || !d->col_basis[c]))) {
        *err = "missing leaf basis for cluster " + std::to_string(c); return H2B_EINVAL;
      }
    }
    if (c != 0) {
      int32_t p = parent_[c];
      if ((d->k_row[c] * d->k_row[p] > 0 && (!d->row_transfer || !d->row_transfer[c])) ||
          (d->k_col[c] * d->k_col[p] > 0 && (!d->col_transfer || !d->col_transfer[c]))) {
        *err = "missing transfer matrix for cluster " + std::to_string(c); return H2B_EINVAL;
      }
    }
  }
  if (d->ncoupling < 0 || d->nnear < 0) { *err = "negative block count"; return H2B_EINVAL; }
  for (int64_t b = 0; b < d->ncoupling; ++b) {
    int64_t r = d->cp_row[b], s = d->cp_col[b];
    if (r < 0 || r >= nc || s < 0 || s >= nc) { *err = "coupling block cluster id out of range"; return H2B_EINVAL; }
    if (d->k_row[r] * d->k_col[s] > 0 && !d->cp_data[b]) { *err = "null coupling matrix"; return H2B_EINVAL; }
  }
  for (int64_t b = 0; b < d->nnear; ++b) {
    int64_t r = d->nr_row[b], s = d->nr_col[b];
    if (r < 0 || r >= nc || s < 0 || s >= nc) { *err = "near block cluster id out of range"; return H2B_EINVAL; }
    if (!d->nr_data[b]) { *err = "null near-field matrix"; return H2B_EINVAL; }
  }
  return H2B_OK;
}

void Builder::emit_group(int32_t kind, int32_t stage, int32_t m_total, std::vector<SegSpec>& segs,
                         Vec* outv, int64_t y_pos, const Vec* bias, bool allow_split, int32_t qclass,
                         bool seg0_hi, bool append) {
  Plan& P = *plan_;
  if (m_total <= 0) return;
  // 1. the group matrix (m_total x C, column-major, ld = m_total): recorded,
  // packed later (pack_groups) once it is known whether this rank uses it
  int64_t C = 0;
  for (auto& s : segs) C += s.ncols;
  const int32_t gid = (int32_t)P.groups.size();
  {
    Group g;
    g.m = m_total;
    g.ncols = C;
    g.region = cur_region_;
    g.unit = cur_unit_;
    for (auto& s : segs) g.segs.push_back({s.a, s.ncols, s.transpose, s.a_ld});
    P.groups.push_back(std::move(g));
  }
  P.bytes_by_kind[kind] += 8 * (int64_t)m_total * C;
  // 2. split columns into pieces of <= task_bytes (at segment boundaries when possible)
  std::vector<Piece> pieces;
  // Far-field items are latency-critical (the tree chain): small pieces, each
  // staged by one TMA bulk copy.  Near-field items are bandwidth work.
  // A heavy near-field row is cut into at most kMaxNearPieces items so that
  // its final item sums a bounded number of partial slots.
  // In a downward item the parent transfer (segment 0, seg0_hi) is the link
  // of the far-field chain: it gets a small piece of its own; the coupling
  // blocks after it are slack and streamed in large pieces.
  const bool bulk = kind == kNear || kind == kDown;
  // (coupling rows of inner clusters sit close to the chain: medium pieces)
  const int64_t leaf_cp = opt_.coupling_task_bytes > 0 ? opt_.coupling_task_bytes : opt_.task_bytes;
  const int64_t big = kind == kNear ? std::max<int64_t>(opt_.task_bytes, (8 * (int64_t)m_total * C + kMaxNearPieces - 1) /
                                                                             kMaxNearPieces)
                                    : (qclass == 1 ? std::min<int64_t>(opt_.task_bytes, 16384) : leaf_cp);
  const int64_t cap = bulk ? big : opt_.far_task_bytes;
  const int64_t maxc = allow_split ? std::max<int64_t>(1, cap / (8 * (int64_t)m_total)) : INT64_MAX;
  Piece cur;
  int64_t col = 0;
  for (int64_t si = 0; si < (int64_t)segs.size(); ++si) {
    int64_t nc = segs[si].ncols, c0 = 0;
    if (nc == 0) continue;
    const bool alone = seg0_hi && (si == 1);  // close the transfer-only piece
    if (cur.ncols > 0 && (alone || cur.ncols + nc > maxc || (int)cur.parts.size() >= kMaxSegs)) {
      pieces.push_back(cur); cur = Piece(); cur.col0 = col;
    }
    while (nc - c0 > 0) {
      int64_t take = std::min(nc - c0, maxc - cur.ncols);
      if (take <= 0 || (int)cur.parts.size() >= kMaxSegs) { pieces.push_back(cur); cur = Piece(); cur.col0 = col; continue; }
      if (cur.ncols == 0) cur.col0 = col;
      cur.parts.push_back({si, c0, take});
      cur.ncols += take; c0 += take; col += take;
    }
  }
  if (cur.ncols > 0 || pieces.empty()) pieces.push_back(cur);
  // 3. output vector (`append`: further slots right behind the ones it has)
  int32_t slot0 = 0;
  if (outv) {
    if (append && outv->exists() && outv->len == m_total &&
        outv->off + (int64_t)outv->len * outv->nslots == plan_->coef_len) {
      slot0 = outv->nslots;
      outv->nslots += (int32_t)pieces.size();
      plan_->coef_len += (int64_t)m_total * (int64_t)pieces.size();
    } else {
      alloc_vec(outv, m_total, (int32_t)pieces.size());
    }
  }
  // 4. tasks: one per (piece, row tile)
  for (size_t pi = 0; pi < pieces.size(); ++pi) {
    const Piece& pc = pieces[pi];
    // segment records of this piece (shared by its row tiles)
    std::vector<int32_t> seg_ids;
    std::vector<int32_t> deps;
    for (auto& part : pc.parts) {
      const SegSpec& s = segs[part[0]];
      seg_ids.push_back((int32_t)s_ncols_.size());
      s_ncols_.push_back((int32_t)part[2]);
      s_kind_.push_back(s.kind);
      if (s.kind == kSegX) {
        s_src_.push_back(s.src + part[1]);
        s_nslots_.push_back(1);
        s_stride_.push_back(0);
      } else {
        s_src_.push_back(s.vec->off + part[1]);
        s_nslots_.push_back(s.vec->nslots);
        s_stride_.push_back(s.vec->len);
        deps.insert(deps.end(), s.vec->producers.begin(), s.vec->producers.end());
      }
    }
    if (bias) deps.insert(deps.end(), bias->producers.begin(), bias->producers.end());
    std::sort(deps.begin(), deps.end());
    deps.erase(std::unique(deps.begin(), deps.end()), deps.end());
    for (int32_t r0 = 0; r0 < m_total; r0 += kMaxRows) {
      TaskTmp t;
      t.data = -1;
      t.group = gid;
      t.goff = pc.col0 * m_total + r0;
      t.m = std::min<int32_t>(kMaxRows, m_total - r0);
      t.ld = m_total;
      t.ncols = (int32_t)pc.ncols;
      t.kind = kind;
      t.stage = stage;
      t.out = outv ? outv->off + (int64_t)(slot0 + (int32_t)pi) * m_total + r0 : y_pos + r0;
      if (bias && bias->exists()) {
        t.bias = bias->off + r0;
        t.bias_nslots = bias->nslots;
        t.bias_stride = bias->len;
      } else {
        t.bias = -1; t.bias_nslots = 0; t.bias_stride = 0;
      }
      t.seg_idx = seg_ids;
      t.deps = deps;
      // scheduling class: the transfer pieces, the upward pass and the finals
      // form the far-field critical chain (class 0); coupling pieces of inner
      // clusters are needed as the chain descends (class 1); coupling pieces
      // of leaves and the near field only by the finals (class 2)
      t.qclass = qclass;
      t.cl = cur_cl_;
      if (seg0_hi) {
        for (auto& part : pc.parts) if (part[0] == 0) { t.qclass = 0; t.transfer = true; }
      }
      if (outv) outv->producers.push_back((int32_t)tasks_.size());
      tasks_.push_back(std::move(t));
    }
  }
}

int Builder::run(std::string* err) {
  int rc = validate(err);
  if (rc != H2B_OK) return rc;
  const h2b_desc* d = d_;
  Plan& P = *plan_;
  const int64_t nc = d->nclusters;
  P.n = d->n;
  P.perm.assign(d->perm, d->perm + d->n);
  P.rank = opt_.rank;
  P.world_size = opt_.world_size;
  if (opt_.staged) mark_bottom_subtrees();

  // Algorithmic byte count, H2Matrix.storage_bytes() (h2.py:77-83).
  int64_t entries = 0;
  for (int64_t c = 0; c < nc; ++c) {
    if (is_leaf((int32_t)c)) entries += size((int32_t)c) * (d->k_row[c] + d->k_col[c]);
    if (c != 0) {
      int32_t p = parent_[c];
      entries += d->k_row[c] * d->k_row[p] + d->k_col[c] * d->k_col[p];
    }
  }
  for (int64_t b = 0; b < d->ncoupling; ++b) entries += d->k_row[d->cp_row[b]] * d->k_col[d->cp_col[b]];
  for (int64_t b = 0; b < d->nnear; ++b) entries += size((int32_t)d->nr_row[b]) * size((int32_t)d->nr_col[b]);
  P.stream_bytes = 8 * entries;

  xhat_.assign(nc, Vec());
  yhat_.assign(nc, Vec());
  nearv_.assign(nc, Vec());

  // ---- forward (h2.py:195-209).  Staged plans emit the bottom subtrees one
  // after another (leaves, then inner clusters by height), so that a unit's
  // matrices and x^ vectors are contiguous; then the clusters above them.
  auto emit_up_leaf = [&](int32_t c) {   // x^_t = W_t^T x|_t (h2.py:199-200)
    int32_t k = (int32_t)d->k_col[c];
    if (k == 0) return;
    std::vector<SegSpec> segs{{kSegX, d->cl_start[c], (int32_t)size(c), nullptr, d->col_basis[c], false, 0}};
    cur_cl_ = c;
    emit_group(kUpLeaf, 0, k, segs, &xhat_[c], 0, nullptr, true);
  };
  auto emit_up_node = [&](int32_t p) {   // x^_p = sum_c F_c^T x^_c (h2.py:201-205)
    int32_t k = (int32_t)d->k_col[p];
    if (k == 0) return;
    std::vector<SegSpec> segs;
    // (staged plans: only above the bottom subtrees, whose levels are
    // separated by block barriers, not by scheduling links)
    const bool skip = opt_.skip_levels && height_[p] >= 2 && height_[p] % 2 == 0 && top(p);
    for (int j = 0; j < 2; ++j) {
      int32_t ch = (int32_t)d->cl_child[2 * p + j];
      if (skip && !is_leaf(ch)) {
        // x^_p += (F_g F_ch)^T x^_g over the grandchildren g (h2.py:201-205 expanded)
        const int64_t kc = d->k_col[ch];
        if (kc == 0) continue;
        for (int jj = 0; jj < 2; ++jj) {
          const int32_t g = (int32_t)d->cl_child[2 * ch + jj];
          if (!xhat_[g].exists()) continue;
          const int64_t kg = d->k_col[g];
          const double* fg = product(d->col_transfer[g], d->col_transfer[ch], kg, kc, k);
          segs.push_back({kSegCoef, 0, (int32_t)kg, &xhat_[g], fg, false, 0});
        }
        continue;
      }
      if (!xhat_[ch].exists()) continue;
      segs.push_back({kSegCoef, 0, (int32_t)d->k_col[ch], &xhat_[ch], d->col_transfer[ch], false, 0});
    }
    cur_cl_ = p;
    emit_group(kUpNode, height_[p], k, segs, &xhat_[p], 0, nullptr, true);
  };
  // the clusters of every bottom subtree (preorder), in tree order of the roots
  std::vector<std::vector<int32_t>>& units = units_;
  if (opt_.staged)
    for (int32_t c : order_) {
      if (broot_[c] == c) units.emplace_back();
      if (broot_[c] >= 0) units.back().push_back(c);
    }
  for (auto& sub : units) {
    cur_region_ = 1;
    cur_unit_ = d->cl_start[sub[0]];
    std::vector<int32_t> inner;
    for (int32_t c : sub) {
      if (is_leaf(c)) emit_up_leaf(c);
      else inner.push_back(c);
    }
    std::stable_sort(inner.begin(), inner.end(), [&](int32_t a, int32_t b) { return height_[a] < height_[b]; });
    for (int32_t p : inner) emit_up_node(p);
  }
  cur_region_ = 0;
  cur_unit_ = 0;
  for (int32_t c : leaves_) if (top(c)) emit_up_leaf(c);
  {
    std::vector<int32_t> inner;
    for (int32_t c = 0; c < nc; ++c) if (!is_leaf(c) && top(c)) inner.push_back(c);
    std::stable_sort(inner.begin(), inner.end(), [&](int32_t a, int32_t b) { return height_[a] < height_[b]; });
    for (int32_t p : inner) emit_up_node(p);
  }
  // ---- near field, grouped by target leaf (h2.py:237-240).  Blocks whose
  // row cluster is not a leaf are split into their leaf row ranges.
  {
    std::vector<std::vector<std::pair<int64_t, int64_t>>> by_leaf(nc);  // (block, row offset)
    for (int64_t b = 0; b < d->nnear; ++b) {
      int32_t r = (int32_t)d->nr_row[b];
      if (is_leaf(r)) { by_leaf[r].push_back({b, 0}); continue; }
      std::vector<int32_t> ls;
      collect_leaves(r, &ls);
      for (int32_t l : ls) by_leaf[l].push_back({b, d->cl_start[l] - d->cl_start[r]});
    }
    for (int32_t l : leaves_) {
      if (by_leaf[l].empty()) continue;
      std::vector<SegSpec> segs;
      for (auto& br : by_leaf[l]) {
        int64_t b = br.first;
        int32_t s = (int32_t)d->nr_col[b];
        int64_t ncol = size(s);
        segs.push_back({kSegX, d->cl_start[s], (int32_t)ncol, nullptr, d->nr_data[b] + br.second * ncol, true, ncol});
      }
      cur_cl_ = l;
      emit_group(kNear, 0, (int32_t)size(l), segs, &nearv_[l], 0, nullptr, true, 2);
    }
  }
  // ---- coupling + downward pass, top-down (h2.py:211-235)
  {
    std::vector<std::vector<int64_t>> cp_by_row(nc);
    for (int64_t b = 0; b < d->ncoupling; ++b) cp_by_row[d->cp_row[b]].push_back(b);
    std::vector<int32_t> order(nc);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return depth_[a] < depth_[b]; });
    // Level skipping: an "own" cluster (inner, child of a full one) only sums
    // its coupling rows; its children take the grandparent's coefficient
    // through E_c E_p plus E_c times that own sum:
    //   y^_c = E_c (E_p y^_gp + y^_p,own) + y^_c,own       (h2.py:220-235)
    std::vector<char> own_only(nc, 0);
    auto emit_down = [&](int32_t t) {
      int32_t k = (int32_t)d->k_row[t];
      // odd heights (counted from the leaves, so the leaves skip their
      // parent's level), never two "own" levels in a row
      if (t != 0 && opt_.skip_levels && !is_leaf(t) && height_[t] % 2 == 1 && !own_only[parent_[t]] && top(t))
        own_only[t] = 1;
      if (k == 0) return;
      std::vector<SegSpec> segs;
      bool transfer = false;
      if (t != 0 && !own_only[t]) {
        const int32_t p = parent_[t];
        if (!own_only[p]) {
          if (yhat_[p].exists()) {
            segs.push_back({kSegCoef, 0, (int32_t)d->k_row[p], &yhat_[p], d->row_transfer[t], true, d->k_row[p]});
            transfer = true;
          }
        } else if (d->k_row[p] > 0) {
          const int32_t gp = parent_[p];
          const int64_t kp = d->k_row[p];
          if (yhat_[gp].exists()) {  // the chain link: E_t E_p y^_gp
            const int64_t kg = d->k_row[gp];
            const double* ep = product(d->row_transfer[t], d->row_transfer[p], k, kp, kg);
            segs.push_back({kSegCoef, 0, (int32_t)kg, &yhat_[gp], ep, true, kg});
            transfer = true;
          }
          if (yhat_[p].exists())   // the parent's own coupling sum (slack)
            segs.push_back({kSegCoef, 0, (int32_t)kp, &yhat_[p], d->row_transfer[t], true, kp});
        }
      }
      for (int64_t b : cp_by_row[t]) {
        int32_t s = (int32_t)d->cp_col[b];
        if (!xhat_[s].exists()) continue;
        int64_t ks = d->k_col[s];
        segs.push_back({kSegCoef, 0, (int32_t)ks, &xhat_[s], d->cp_data[b], true, ks});
      }
      if (segs.empty()) return;  // coefficient stays None (h2.py:224-226)
      cur_cl_ = t;
      const int32_t qc = is_leaf(t) ? 2 : 1;
      if (!top(t) && transfer) {
        // a bottom cluster's transfer is an item of the downward sweep: a
        // matrix of its own (laid out with its unit's), writing slot 0 of
        // y^_t; the coupling rows append their slots behind it
        std::vector<SegSpec> xfer{segs[0]};
        std::vector<SegSpec> rest(segs.begin() + 1, segs.end());
        cur_region_ = 2;
        emit_group(kDown, depth_[t], k, xfer, &yhat_[t], 0, nullptr, true, qc, true);
        cur_region_ = 0;
        if (!rest.empty()) emit_group(kDown, depth_[t], k, rest, &yhat_[t], 0, nullptr, true, qc, false, true);
        return;
      }
      emit_group(kDown, depth_[t], k, segs, &yhat_[t], 0, nullptr, true, qc, transfer);
    };
    for (int32_t t : order) if (top(t)) emit_down(t);
    for (auto& sub : units) {
      cur_unit_ = d->cl_start[sub[0]];
      std::vector<int32_t> by_depth(sub);
      std::stable_sort(by_depth.begin(), by_depth.end(), [&](int32_t a, int32_t b) { return depth_[a] < depth_[b]; });
      for (int32_t t : by_depth) emit_down(t);
    }
    cur_unit_ = 0;
  }
  // ---- leaf back-transform + near partials -> y (h2.py:227-229, 242-243)
  for (int32_t l : leaves_) {
    std::vector<SegSpec> segs;
    int32_t k = (int32_t)d->k_row[l];
    if (k > 0 && yhat_[l].exists())
      segs.push_back({kSegCoef, 0, k, &yhat_[l], d->row_basis[l], true, k});
    cur_cl_ = l;
    if (opt_.staged) { cur_region_ = 2; cur_unit_ = d->cl_start[broot_[l]]; }
    emit_group(kFinal, 0, (int32_t)size(l), segs, nullptr, d->cl_start[l], &nearv_[l], false, opt_.final_class);
  }
  cur_region_ = 0;
  cur_unit_ = 0;
  // Staged plans: the pool region by region -- the upward sweep's units, the
  // dataflow launch's matrices, the downward sweep's units (transfers and
  // leaf bases of a unit together)
  if (opt_.staged) {
    const size_t G = P.groups.size();
    std::vector<int32_t> perm_g(G);
    std::iota(perm_g.begin(), perm_g.end(), 0);
    auto key = [&](int32_t g) { return P.groups[g].region == 1 ? 0 : P.groups[g].region == 0 ? 1 : 2; };
    std::stable_sort(perm_g.begin(), perm_g.end(), [&](int32_t a, int32_t b) {
      if (key(a) != key(b)) return key(a) < key(b);
      return key(a) == 2 && P.groups[a].unit < P.groups[b].unit;
    });
    std::vector<int32_t> new_id(G);
    std::vector<Group> sorted;
    sorted.reserve(G);
    for (size_t k2 = 0; k2 < G; ++k2) {
      new_id[perm_g[k2]] = (int32_t)k2;
      sorted.push_back(std::move(P.groups[perm_g[k2]]));
    }
    P.groups.swap(sorted);
    for (auto& t : tasks_) t.group = new_id[t.group];
  }
  // Entries never read by the product (e.g. row bases of an operator
  // without coupling blocks) are not packed, so the pool can be smaller.
  {
    int64_t all = 0;
    for (const auto& g : P.groups) all += g.size();
    if (all > entries + P.extra_bytes / 8) {
      *err = "internal: packed pool larger than storage_bytes";
      return H2B_EINVAL;
    }
  }

  const int32_t T = (int32_t)tasks_.size();
  P.rank_lo.assign(1, 0);
  P.rank_hi.assign(1, d->n);
  // staged plans: the sweeps' items
  auto in_up_sweep = [&](const TaskTmp& t) {
    return opt_.staged && (t.kind == kUpLeaf || t.kind == kUpNode) && !top(t.cl);
  };
  auto in_down_sweep = [&](const TaskTmp& t) {
    return opt_.staged && (t.kind == kFinal || (t.kind == kDown && t.transfer && !top(t.cl)));
  };
  // the launches of one group of selected items: [up sweep] dataflow [down
  // sweep]; with `split` the near field gets a launch of its own (mode 2)
  // (the split multi-RHS product forms sweeps too with opt_.split_sweeps;
  // with one sweep CTA per SM they had measured slower, with two faster)
  auto emit_launches = [&](std::vector<Phase>* out, const std::vector<char>& in, int32_t group, bool split) -> int {
    std::vector<int32_t> up, dn, near, rest;
    std::vector<char> in_near(T, 0), in_rest(T, 0);
    const bool sweeps = !split || opt_.split_sweeps;
    for (int32_t i = 0; i < T; ++i) {
      if (!in[i]) continue;
      const TaskTmp& t = tasks_[i];
      if (sweeps && in_up_sweep(t)) up.push_back(i);
      else if (sweeps && in_down_sweep(t)) dn.push_back(i);
      else if (split && t.kind == kNear) { near.push_back(i); in_near[i] = 1; }
      else { rest.push_back(i); in_rest[i] = 1; }
    }
    // closure: the dataflow launch must not wait for an item of the down sweep
    for (int32_t i : rest)
      for (int32_t dp : tasks_[i].deps)
        if (sweeps && in[dp] && in_down_sweep(tasks_[dp])) { *err = "internal: dataflow item depends on the down sweep"; return H2B_EINVAL; }
    int rc2 = H2B_OK;
    if (!up.empty()) {
      out->emplace_back();
      if ((rc2 = finalize_sweep(&out->back(), up, err)) != H2B_OK) return rc2;
      out->back().group = group;
    }
    if (split) {
      out->emplace_back();
      if ((rc2 = finalize(&out->back(), near, in_near, err)) != H2B_OK) return rc2;
      out->back().mode = 2;
      out->back().group = group;
    }
    if (!rest.empty() || (!split && up.empty() && dn.empty()) || (split && sweeps)) {
      out->emplace_back();
      if ((rc2 = finalize(&out->back(), rest, in_rest, err)) != H2B_OK) return rc2;
      out->back().group = group;
    }
    if (!dn.empty()) {
      out->emplace_back();
      if ((rc2 = finalize_sweep(&out->back(), dn, err)) != H2B_OK) return rc2;
      out->back().group = group;
    }
    return H2B_OK;
  };
  if (opt_.world_size <= 1) {
    P.local_bytes = P.stream_bytes;
    assign_bases(std::vector<char>(T, 1));
    rc = emit_launches(&P.ph, std::vector<char>(T, 1), 0, false);
    if (rc != H2B_OK || !opt_.near_split) return rc;
    return emit_launches(&P.ph_split, std::vector<char>(T, 1), 0, true);
  }

  // ---- multi-GPU: byte-balanced contiguous leaf ranges (tree order is a
  // geometric bisection order, so ranges are compact), DESIGN.md §7
  const int32_t W = opt_.world_size, R = opt_.rank;
  std::vector<double> leaf_w(nc, 0.0);
  for (auto& t : tasks_) leaf_w[t.cl] += 8.0 * t.m * t.ncols;
  // granules of the partition: the leaves, or (staged) the bottom subtrees,
  // so that a rank owns whole subtrees and sweeps them by itself
  std::vector<std::pair<int64_t, double>> gran;  // (end position, weight)
  for (size_t i = 0; i < leaves_.size(); ++i) {
    const int32_t l = leaves_[i];
    const bool same = opt_.staged && i > 0 && broot_[l] == broot_[leaves_[i - 1]];
    if (same) { gran.back().first = d->cl_end[l]; gran.back().second += leaf_w[l] + 1.0; }
    else gran.push_back({d->cl_end[l], leaf_w[l] + 1.0});
  }
  double total = 0.0;
  for (auto& g : gran) total += g.second;
  P.rank_lo.assign(W, 0);
  P.rank_hi.assign(W, 0);
  {
    double acc = 0.0;
    int32_t r = 0;
    P.rank_lo[0] = 0;
    for (size_t i = 0; i < gran.size(); ++i) {
      acc += gran[i].second;
      const size_t left = gran.size() - i - 1;
      if (r < W - 1 && (acc >= total * (r + 1) / W || left <= (size_t)(W - 1 - r))) {
        P.rank_hi[r] = gran[i].first;
        ++r;
        P.rank_lo[r] = gran[i].first;
      }
    }
    for (; r < W; ++r) {
      if (r > 0 && P.rank_lo[r] == 0) P.rank_lo[r] = d->n;
      P.rank_hi[r] = d->n;
    }
  }
  const int64_t lo = P.rank_lo[R], hi = P.rank_hi[R];
  auto owner = [&](int32_t c) -> int32_t {
    for (int32_t r = 0; r < W; ++r)
      if (d->cl_start[c] >= P.rank_lo[r] && d->cl_end[c] <= P.rank_hi[r]) return r;
    return -1;  // spans several ranks
  };
  // selection and phase of every task on this rank
  std::vector<char> sel(T, 0), in0(T, 0), in1(T, 0);
  for (int32_t i = 0; i < T; ++i) {
    const TaskTmp& t = tasks_[i];
    const int32_t o = owner(t.cl);
    if (t.kind == kUpLeaf || t.kind == kUpNode) {
      if (o == R) { sel[i] = 1; in0[i] = 1; }
      else if (o < 0) { sel[i] = 1; in1[i] = 1; }
    } else if (t.kind == kDown) {
      if (d->cl_start[t.cl] < hi && d->cl_end[t.cl] > lo) { sel[i] = 1; in1[i] = 1; }
    } else if (o == R) {
      sel[i] = 1; in1[i] = 1;
    }
  }
  // Part of the near field moves to phase 0: it needs only x (replicated),
  // and streams while the upward pass -- a latency-bound chain with little
  // work -- runs; the rest stays in phase 1 beside the downward chain.  The
  // finals in phase 1 then find those partial slots already written.
  if (opt_.near_phase0_pct > 0) {
    int64_t total = 0, moved_b = 0;
    for (int32_t i = 0; i < T; ++i)
      if (sel[i] && tasks_[i].kind == kNear) total += 8 * (int64_t)tasks_[i].m * tasks_[i].ncols;
    const int64_t goal = total * opt_.near_phase0_pct / 100;
    for (int32_t i = 0; i < T && moved_b < goal; ++i)
      if (sel[i] && tasks_[i].kind == kNear) {
        in1[i] = 0;
        in0[i] = 1;
        moved_b += 8 * (int64_t)tasks_[i].m * tasks_[i].ncols;
      }
  }
  // coefficient layout: the x^ vectors of owned clusters move into
  // per-rank exchange regions of equal size at the start of the workspace
  {
    struct Blk { int64_t old_off, size, new_off; };
    std::vector<Blk> blks;
    std::vector<int64_t> region(W, 0);
    std::vector<int32_t> blk_owner;
    for (int32_t c = 0; c < nc; ++c) {
      const Vec& v = xhat_[c];
      if (!v.exists()) continue;
      const int32_t o = owner(c);
      blks.push_back({v.off, (int64_t)v.len * v.nslots, 0});
      blk_owner.push_back(o);
      if (o >= 0) region[o] += (int64_t)v.len * v.nslots;
    }
    int64_t rsz = 0;
    for (int32_t r = 0; r < W; ++r) rsz = std::max(rsz, region[r]);
    std::vector<int64_t> fill(W);
    for (int32_t r = 0; r < W; ++r) fill[r] = (int64_t)r * rsz;
    // everything else keeps its order after the regions
    std::vector<char> moved(P.coef_len, 0);
    for (size_t b2 = 0; b2 < blks.size(); ++b2)
      if (blk_owner[b2] >= 0) {
        blks[b2].new_off = fill[blk_owner[b2]];
        fill[blk_owner[b2]] += blks[b2].size;
        std::fill(moved.begin() + blks[b2].old_off, moved.begin() + blks[b2].old_off + blks[b2].size, 1);
      }
    // map for the rest: compact the unmoved doubles after the regions
    std::vector<int64_t> rest(P.coef_len + 1, 0);
    int64_t nxt = (int64_t)W * rsz;
    for (int64_t o = 0; o < P.coef_len; ++o) {
      rest[o] = nxt;
      if (!moved[o]) ++nxt;
    }
    std::vector<int64_t> newpos(P.coef_len, 0);
    for (int64_t o = 0; o < P.coef_len; ++o) newpos[o] = rest[o];
    for (size_t b2 = 0; b2 < blks.size(); ++b2)
      if (blk_owner[b2] >= 0)
        for (int64_t k = 0; k < blks[b2].size; ++k) newpos[blks[b2].old_off + k] = blks[b2].new_off + k;
    auto map = [&](int64_t o) -> int64_t { return o < P.coef_len ? newpos[o] : o; };
    for (auto& t : tasks_) {
      if (t.kind != kFinal) t.out = map(t.out);
      if (t.bias >= 0) t.bias = map(t.bias);
    }
    for (size_t k = 0; k < s_src_.size(); ++k)
      if (s_kind_[k] == kSegCoef) s_src_[k] = map(s_src_[k]);
    for (auto* vs : {&xhat_, &yhat_, &nearv_})
      for (auto& v : *vs)
        if (v.exists()) v.off = map(v.off);
    P.coef_len = nxt;
    P.exch_off = 0;
    P.exch_count = rsz;
  }
  P.local_bytes = 0;
  for (int32_t i = 0; i < T; ++i)
    if (sel[i]) P.local_bytes += 8 * (int64_t)tasks_[i].m * tasks_[i].ncols;
  // a phase-1 dependency on a phase-1 item of another rank would be a
  // missing exchange: check the selection is closed
  for (int32_t i = 0; i < T; ++i) {
    if (!in1[i]) continue;
    for (int32_t dp : tasks_[i].deps)
      if (!in1[dp] && !(tasks_[dp].kind == kUpLeaf || tasks_[dp].kind == kUpNode ||
                        (tasks_[dp].kind == kNear && in0[dp]))) {
        *err = "internal: rank plan is missing a dependency";
        return H2B_EINVAL;
      }
  }
  // this rank's pool: only the matrices of its selected items (the
  // replicated upper clusters plus its own rows), so per-rank host and
  // device memory scale as 1/world
  assign_bases(sel);
  // group 0 (before the exchange) always has a dataflow launch, possibly
  // empty, so that classic plans keep their two phases
  rc = emit_launches(&P.ph, in0, 0, false);
  if (rc != H2B_OK) return rc;
  return emit_launches(&P.ph, in1, 1, false);
}

void Builder::mark_bottom_subtrees() {
  const h2b_desc* d = d_;
  const int64_t nc = d->nclusters;
  int64_t S = opt_.sweep_nodes > 0 ? opt_.sweep_nodes : 128;
  auto mark = [&](int64_t cap) -> int64_t {
    broot_.assign(nc, -1);
    int64_t roots = 0;
    for (int32_t c : order_) {  // preorder: parents first
      const int32_t p = parent_[c];
      if (p >= 0 && broot_[p] >= 0) broot_[c] = broot_[p];
      else if (size(c) <= cap || is_leaf(c)) { broot_[c] = c; ++roots; }
    }
    return roots;
  };
  int64_t roots = mark(S);
  // Default size: about 256 subtrees per rank (one per resident CTA of the
  // sweep kernels, so that a sweep is one round of similar units and their
  // leaf waves keep every warp busy): measured best on configs 2 and 3 on
  // one GPU and on config 3 split over 8 ranks.
  if (opt_.sweep_nodes <= 0) {
    const int64_t per = d->n / (256 * (int64_t)std::max(1, opt_.world_size));
    S = 128;
    while (S < per && S < 16384) S *= 2;
    roots = mark(S);
  }
  // multi-GPU: ranks own whole subtrees, so there must be enough of them to
  // balance the ranks' bytes
  const int64_t want = opt_.world_size > 1 ? std::min<int64_t>(8 * (int64_t)opt_.world_size, (int64_t)leaves_.size()) : 1;
  while (roots < want && S > 1) {
    S /= 2;
    roots = mark(S);
  }
}

int Builder::finalize_sweep(Phase* F, const std::vector<int32_t>& ids, std::string* err) {
  const int32_t T = (int32_t)ids.size();
  std::vector<int32_t> wave(tasks_.size(), -1);
  // provisional ids grow along dependencies (a producer is emitted before
  // its consumers), so one ascending pass gives the dependency depth
  std::vector<int32_t> sorted(ids);
  std::sort(sorted.begin(), sorted.end());
  std::vector<char> in(tasks_.size(), 0);
  for (int32_t i : sorted) in[i] = 1;
  for (int32_t i : sorted) {
    int32_t w = 0;
    for (int32_t dp : tasks_[i].deps) {
      if (!in[dp]) continue;  // produced by an earlier launch
      if (dp >= i || wave[dp] < 0 || broot_[tasks_[dp].cl] != broot_[tasks_[i].cl]) {
        *err = "internal: sweep dependency outside its subtree";
        return H2B_EINVAL;
      }
      w = std::max(w, wave[dp] + 1);
    }
    wave[i] = w;
  }
  // units in tree order of their roots; items by wave, then emission order
  std::stable_sort(sorted.begin(), sorted.end(), [&](int32_t a, int32_t b) {
    const int32_t ra = broot_[tasks_[a].cl], rb = broot_[tasks_[b].cl];
    if (ra != rb) return d_->cl_start[ra] < d_->cl_start[rb];
    return wave[a] < wave[b];
  });
  F->mode = 1;
  F->t_data.resize(T); F->t_out.resize(T); F->t_bias.resize(T);
  F->t_m.resize(T); F->t_ld.resize(T); F->t_ncols.resize(T); F->t_kind.resize(T);
  F->t_bias_nslots.resize(T); F->t_bias_stride.resize(T); F->t_qclass.assign(T, 0);
  F->t_mlen.assign(T, 0);
  F->t_seg0.assign(T + 1, 0); F->t_dep0.assign(T + 1, 0);
  F->succ0.assign(T + 1, 0);
  F->unit0.clear(); F->wave0.clear();
  int32_t unit_first = 0;
  for (int32_t k = 0; k < T; ++k) {
    const TaskTmp& t = tasks_[sorted[k]];
    const bool new_unit = k == 0 || broot_[t.cl] != broot_[tasks_[sorted[k - 1]].cl];
    if (new_unit) {
      if (k > 0) F->t_mlen[unit_first] = k - unit_first;
      unit_first = k;
      F->unit0.push_back((int32_t)F->wave0.size());
    }
    if (new_unit || wave[sorted[k]] != wave[sorted[k - 1]]) F->wave0.push_back(k);
    F->t_data[k] = t.data; F->t_out[k] = t.out; F->t_bias[k] = t.bias;
    F->t_m[k] = t.m; F->t_ld[k] = t.ld; F->t_ncols[k] = t.ncols; F->t_kind[k] = t.kind;
    F->t_bias_nslots[k] = t.bias_nslots; F->t_bias_stride[k] = t.bias_stride;
    for (int32_t si : t.seg_idx) {
      F->s_src.push_back(s_src_[si]); F->s_ncols.push_back(s_ncols_[si]); F->s_kind.push_back(s_kind_[si]);
      F->s_nslots.push_back(s_nslots_[si]); F->s_stride.push_back(s_stride_[si]);
    }
    F->t_seg0[k + 1] = (int32_t)F->s_ncols.size();
    F->tasks_by_kind[t.kind] += 1;
  }
  if (T > 0) F->t_mlen[unit_first] = T - unit_first;
  F->unit0.push_back((int32_t)F->wave0.size());
  F->wave0.push_back(T);
  F->nnodes = (int64_t)F->unit0.size() - 1;
  // Resident form: per unit the contiguous ranges its CTA copies into shared
  // memory -- matrices, main coefficients (x^ / y^ slots of its clusters),
  // near-field partial slots of its leaves, its x range.
  {
    const int64_t U = F->nnodes;
    F->u_range.assign((size_t)(8 * U), 0);
    F->resident = U > 0;
    std::unordered_map<int32_t, const std::vector<int32_t>*> sub_of;
    for (const auto& sub : units_) sub_of[sub[0]] = &sub;
    const bool up = T > 0 && F->t_kind[0] <= kUpNode;
    for (int64_t u = 0; u < U; ++u) {
      const int32_t k0 = F->wave0[F->unit0[u]], k1 = F->wave0[F->unit0[u + 1]];
      const int32_t root = broot_[tasks_[sorted[k0]].cl];
      // matrices: the groups of the unit's items
      int64_t lo = INT64_MAX, hi = -1, sum = 0;
      std::vector<int32_t> gs;
      for (int32_t k = k0; k < k1; ++k) gs.push_back(tasks_[sorted[k]].group);
      std::sort(gs.begin(), gs.end());
      gs.erase(std::unique(gs.begin(), gs.end()), gs.end());
      for (int32_t g : gs) {
        const Group& G = plan_->groups[g];
        if (G.base < 0) { F->resident = false; continue; }
        lo = std::min(lo, G.base); hi = std::max(hi, G.base + G.size()); sum += G.size();
      }
      if (hi < 0) { lo = hi = 0; }
      if (sum != hi - lo) {
        if (F->resident && std::getenv("H2B_DEBUG_PLAN"))
          std::fprintf(stderr, "[plan] unit %lld (%s): matrices not contiguous (%lld of %lld)\n", (long long)u,
                       up ? "up" : "down", (long long)sum, (long long)(hi - lo));
        F->resident = false;
      }
      int64_t* R = &F->u_range[(size_t)(8 * u)];
      R[0] = lo; R[1] = hi - lo;
      // coefficient ranges of the subtree's clusters
      auto hull = [&](const std::vector<Vec>& vs, bool leaves_only, int64_t* out) {
        int64_t a = INT64_MAX, b = -1, tot = 0;
        for (int32_t c : *sub_of.at(root)) {
          const Vec& v = vs[c];
          if (!v.exists() || (leaves_only && !is_leaf(c))) continue;
          const int64_t len = (int64_t)v.len * v.nslots;
          a = std::min(a, v.off); b = std::max(b, v.off + len); tot += len;
        }
        if (b < 0) { out[0] = out[1] = 0; return; }
        if (tot != b - a) {
          if (F->resident && std::getenv("H2B_DEBUG_PLAN"))
            std::fprintf(stderr, "[plan] unit %lld (%s): %s not contiguous (%lld of %lld)\n", (long long)u,
                         up ? "up" : "down", leaves_only ? "partials" : "coefficients", (long long)tot, (long long)(b - a));
          F->resident = false;
        }
        out[0] = a; out[1] = b - a;
      };
      hull(up ? xhat_ : yhat_, false, R + 2);
      if (!up) hull(nearv_, true, R + 4);
      R[6] = d_->cl_start[root]; R[7] = d_->cl_end[root] - d_->cl_start[root];  // x (upward) / perm (downward)
      {
        const int32_t nwv = F->unit0[u + 1] - F->unit0[u];
        if (nwv > 12) F->resident = false;
        if ((int64_t)F->u_rec.size() < 16 * U) F->u_rec.assign((size_t)(16 * U), 0);
        int64_t* Q = &F->u_rec[(size_t)(16 * u)];
        for (int j = 0; j < 8; ++j) Q[j] = R[j];
        Q[8] = (int64_t)k0 | ((int64_t)(k1 - k0) << 32);
        Q[9] = (int64_t)nwv | ((int64_t)(up ? 1 : 0) << 32);
        int32_t* we = reinterpret_cast<int32_t*>(Q + 10);
        for (int32_t j = 0; j < std::min(nwv, 12); ++j) we[j] = F->wave0[F->unit0[u] + j + 1] - k0;
      }
      F->res_mat_max = std::max(F->res_mat_max, R[1]);
      F->res_vec_max = std::max(F->res_vec_max, R[3] + R[5] + R[7]);
      F->res_items_max = std::max(F->res_items_max, k1 - k0);
    }
  }
  return H2B_OK;
}

void Builder::assign_bases(const std::vector<char>& sel) {
  Plan& P = *plan_;
  std::vector<char> used(P.groups.size(), 0);
  for (size_t i = 0; i < tasks_.size(); ++i)
    if (sel[i]) used[tasks_[i].group] = 1;
  int64_t off = 0;
  for (size_t g = 0; g < P.groups.size(); ++g) {
    P.groups[g].base = used[g] ? off : -1;
    if (used[g]) off += P.groups[g].size();
  }
  P.mat_len = off;
  for (auto& t : tasks_) t.data = P.groups[t.group].base >= 0 ? P.groups[t.group].base + t.goff : -1;
}

int Builder::finalize(Phase* F, std::vector<int32_t> ids, const std::vector<char>& in_phase, std::string* err) {
  // queue order: up-leaf, upward levels, downward levels, near field, finals
  // (only the dependency order matters: the kernel schedules dynamically)
  auto key = [&](int32_t i) {
    const TaskTmp& t = tasks_[i];
    switch (t.kind) {
      case kUpLeaf: return 0;
      case kUpNode: return 1 + t.stage;
      case kDown: return 1000 + t.stage;
      case kNear: return 2000;
      default: return 3000;
    }
  };
  std::stable_sort(ids.begin(), ids.end(), [&](int32_t a, int32_t b) { return key(a) < key(b); });
  const int32_t T = (int32_t)ids.size();

  // ---- fused runs of the far-field chain.  The upward items of the clusters
  // of one band (a cluster whose depth is a multiple of D and its
  // descendants down to D-1 levels below) run on one warp, deepest first;
  // so do the transfer pieces of the downward pass, shallowest first.  A
  // chain of depth L then costs ~L/D scheduling links instead of L.  Both
  // sets are convex (no path leaves the run and comes back), so a run waits
  // only for its external inputs.
  const int D = std::max(1, opt_.band_depth);
  std::vector<std::vector<int32_t>> runs;  // members (provisional ids) in run order
  std::vector<int32_t> run_of(tasks_.size(), -1);
  {
    std::vector<int64_t> run_key_tab;
    std::unordered_map<int64_t, int32_t> by_key;
    for (int32_t i : ids) {
      const TaskTmp& t = tasks_[i];
      int dir = -1;
      if (D > 1) {
        if (t.kind == kUpLeaf || t.kind == kUpNode) dir = 0;
        else if (t.kind == kDown && t.qclass == 0) dir = 1;
      }
      int32_t r;
      if (dir < 0) {
        r = (int32_t)runs.size();
        runs.emplace_back();
      } else {
        int32_t b = t.cl;
        while (depth_[b] % D != 0) b = parent_[b];
        const int64_t k = 2 * (int64_t)b + dir;
        auto it = by_key.find(k);
        if (it == by_key.end()) {
          r = (int32_t)runs.size();
          by_key.emplace(k, r);
          runs.emplace_back();
        } else {
          r = it->second;
        }
      }
      runs[r].push_back(i);
      run_of[i] = r;
    }
    for (auto& R : runs) {
      if (R.size() < 2) continue;
      const bool up = tasks_[R[0]].kind == kUpLeaf || tasks_[R[0]].kind == kUpNode;
      std::stable_sort(R.begin(), R.end(), [&](int32_t a, int32_t b) {
        return up ? depth_[tasks_[a].cl] > depth_[tasks_[b].cl] : depth_[tasks_[a].cl] < depth_[tasks_[b].cl];
      });
    }
  }
  // run graph: external dependencies (within this phase), deduplicated
  const int32_t NR = (int32_t)runs.size();
  std::vector<std::vector<int32_t>> rdeps(NR);
  for (int32_t r = 0; r < NR; ++r) {
    auto& dv = rdeps[r];
    for (int32_t i : runs[r])
      for (int32_t dp : tasks_[i].deps) {
        if (!in_phase[dp]) continue;  // produced before this phase
        const int32_t q = run_of[dp];
        if (q < 0) { *err = "internal: dependency outside the phase"; return H2B_EINVAL; }
        if (q != r) dv.push_back(q);
      }
    std::sort(dv.begin(), dv.end());
    dv.erase(std::unique(dv.begin(), dv.end()), dv.end());
    // internal dependencies must point backwards in run order
    std::vector<int32_t> seen;
    for (int32_t i : runs[r]) {
      for (int32_t dp : tasks_[i].deps)
        if (in_phase[dp] && run_of[dp] == r && std::find(seen.begin(), seen.end(), dp) == seen.end()) {
          *err = "internal: fused run out of dependency order";
          return H2B_EINVAL;
        }
      seen.push_back(i);
    }
  }
  // topological order of the runs (Kahn), by the queue key of their first item
  std::vector<int32_t> order;
  {
    std::vector<int32_t> indeg(NR, 0);
    std::vector<std::vector<int32_t>> rsucc(NR);
    for (int32_t r = 0; r < NR; ++r)
      for (int32_t q : rdeps[r]) { rsucc[q].push_back(r); ++indeg[r]; }
    std::vector<int32_t> firstpos(NR);
    {
      std::vector<int32_t> qpos(tasks_.size(), 0);
      for (int32_t k = 0; k < T; ++k) qpos[ids[k]] = k;
      for (int32_t r = 0; r < NR; ++r) {
        int32_t mn = INT32_MAX;
        for (int32_t i : runs[r]) mn = std::min(mn, qpos[i]);
        firstpos[r] = mn;
      }
    }
    using E = std::pair<int32_t, int32_t>;
    std::priority_queue<E, std::vector<E>, std::greater<E>> pq;
    for (int32_t r = 0; r < NR; ++r) if (indeg[r] == 0) pq.push({firstpos[r], r});
    while (!pq.empty()) {
      const int32_t r = pq.top().second;
      pq.pop();
      order.push_back(r);
      for (int32_t q : rsucc[r]) if (--indeg[q] == 0) pq.push({firstpos[q], q});
    }
    if ((int32_t)order.size() != NR) { *err = "internal: cycle among fused runs"; return H2B_EINVAL; }
  }
  std::vector<int32_t> lead(NR);  // queue position of each run's first item
  {
    int32_t k = 0;
    for (int32_t r : order) { lead[r] = k; k += (int32_t)runs[r].size(); }
  }

  F->t_data.resize(T); F->t_out.resize(T); F->t_bias.resize(T);
  F->t_m.resize(T); F->t_ld.resize(T); F->t_ncols.resize(T); F->t_kind.resize(T);
  F->t_bias_nslots.resize(T); F->t_bias_stride.resize(T); F->t_qclass.resize(T);
  F->t_mlen.assign(T, 0);
  F->t_seg0.assign(T + 1, 0); F->t_dep0.assign(T + 1, 0);
  F->nnodes = NR;
  int32_t i = 0;
  for (int32_t r : order) {
    for (size_t j = 0; j < runs[r].size(); ++j, ++i) {
      const TaskTmp& t = tasks_[runs[r][j]];
      F->t_data[i] = t.data; F->t_out[i] = t.out; F->t_bias[i] = t.bias;
      F->t_m[i] = t.m; F->t_ld[i] = t.ld; F->t_ncols[i] = t.ncols; F->t_kind[i] = t.kind;
      F->t_bias_nslots[i] = t.bias_nslots; F->t_bias_stride[i] = t.bias_stride;
      F->t_qclass[i] = (int8_t)tasks_[runs[r][0]].qclass;
      for (int32_t si : t.seg_idx) {
        F->s_src.push_back(s_src_[si]); F->s_ncols.push_back(s_ncols_[si]); F->s_kind.push_back(s_kind_[si]);
        F->s_nslots.push_back(s_nslots_[si]); F->s_stride.push_back(s_stride_[si]);
      }
      if (j == 0) {
        F->t_mlen[i] = (int32_t)runs[r].size();
        for (int32_t q : rdeps[r]) {
          if (lead[q] >= i) { *err = "internal: dependency not earlier in the queue"; return H2B_EINVAL; }
          F->deps.push_back(lead[q]);
        }
      }
      F->t_seg0[i + 1] = (int32_t)F->s_ncols.size();
      F->t_dep0[i + 1] = (int32_t)F->deps.size();
      F->tasks_by_kind[t.kind] += 1;
    }
  }
  // gated coupling rows: their dependencies (all upward items) are dropped;
  // the kernel releases them once every upward item of the phase is done
  std::vector<char> gated(T, 0);
  if (opt_.gate_coupling) {
    bool any = false;
    for (int32_t k = 0; k < T; ++k) {
      if (F->t_kind[k] != kDown || F->t_qclass[k] == 0 || F->t_mlen[k] == 0) continue;
      const int32_t e0 = F->t_dep0[k], e1 = F->t_dep0[k + 1];
      if (e1 == e0) continue;
      bool up_only = true;
      for (int32_t e = e0; e < e1 && up_only; ++e) up_only = F->t_kind[F->deps[e]] <= kUpNode;
      if (up_only) { gated[k] = 1; any = true; }
    }
    if (any) {
      std::vector<int32_t> nd;
      nd.reserve(F->deps.size());
      std::vector<int32_t> d0(T + 1, 0);
      for (int32_t k = 0; k < T; ++k) {
        if (!gated[k])
          for (int32_t e = F->t_dep0[k]; e < F->t_dep0[k + 1]; ++e) nd.push_back(F->deps[e]);
        d0[k + 1] = (int32_t)nd.size();
      }
      F->deps.swap(nd);
      F->t_dep0.swap(d0);
    }
    std::vector<int32_t> g2;
    for (int32_t k = 0; k < T; ++k) {
      if (!gated[k]) continue;
      if (F->t_qclass[k] == 1) F->gated.push_back(k);
      else g2.push_back(k);
    }
    F->n_gated1 = (int32_t)F->gated.size();
    std::stable_sort(g2.begin(), g2.end(), [&](int32_t a, int32_t b) {
      return (int64_t)F->t_m[a] * F->t_ncols[a] > (int64_t)F->t_m[b] * F->t_ncols[b];
    });
    F->gated.insert(F->gated.end(), g2.begin(), g2.end());
    for (int32_t k = 0; k < T; ++k) F->n_up += (F->t_kind[k] <= kUpNode && F->t_mlen[k] > 0);
  }
  // successor lists for the completion-driven scheduler
  F->succ0.assign(T + 1, 0);
  for (int32_t dp : F->deps) F->succ0[dp + 1] += 1;
  for (int32_t k = 0; k < T; ++k) F->succ0[k + 1] += F->succ0[k];
  F->succ.assign(F->deps.size(), 0);
  {
    std::vector<int32_t> fill(F->succ0.begin(), F->succ0.end() - 1);
    for (int32_t k = 0; k < T; ++k)
      for (int32_t e = F->t_dep0[k]; e < F->t_dep0[k + 1]; ++e) F->succ[fill[F->deps[e]]++] = k;
  }
  // initially ready runs: class 0 first (up-leaf: they start the far-field
  // chain), then the rest (the near field) longest first, so that heavy rows
  // start early and the end of the launch is made of short items
  for (int32_t k = 0; k < T; ++k)
    if (F->t_mlen[k] > 0 && F->t_dep0[k + 1] == F->t_dep0[k] && F->t_qclass[k] == 0 && !gated[k])
      F->ready0.push_back(k);
  F->n_ready0_hi = (int32_t)F->ready0.size();
  {
    std::vector<int32_t> rest;
    for (int32_t k = 0; k < T; ++k)
      if (F->t_mlen[k] > 0 && F->t_dep0[k + 1] == F->t_dep0[k] && F->t_qclass[k] != 0 && !gated[k]) rest.push_back(k);
    auto longer = [&](int32_t a, int32_t b) {
      return (int64_t)F->t_m[a] * F->t_ncols[a] > (int64_t)F->t_m[b] * F->t_ncols[b];
    };
    std::stable_sort(rest.begin(), rest.end(), longer);
    // Staged plans: the coupling rows of the bottom clusters are static too.
    // They are small and gather-bound: behind the near field they would form
    // a slow tail, so the two lists (each longest first) are merged in
    // proportion to their bytes and stream side by side.
    std::vector<int32_t> nearl, cpl;
    for (int32_t k : rest) (F->t_kind[k] == kNear ? nearl : cpl).push_back(k);
    if (opt_.staged && !nearl.empty() && !cpl.empty()) {
      auto bytes = [&](int32_t k) { return (double)F->t_m[k] * F->t_ncols[k]; };
      double bn = 0.0, bc = 0.0;
      for (int32_t k : nearl) bn += bytes(k);
      for (int32_t k : cpl) bc += bytes(k);
      rest.clear();
      size_t i = 0, j = 0;
      double dn = 0.0, dc = 0.0;
      while (i < nearl.size() || j < cpl.size()) {
        // take from the list that is behind its share
        const bool take_near = j >= cpl.size() || (i < nearl.size() && dn * bc <= dc * bn);
        if (take_near) { dn += bytes(nearl[i]); rest.push_back(nearl[i++]); }
        else { dc += bytes(cpl[j]); rest.push_back(cpl[j++]); }
      }
    }
    F->ready0.insert(F->ready0.end(), rest.begin(), rest.end());
  }
  return H2B_OK;
}

}  // namespace

namespace {
void pack_one(const Group& g, double* dst) {
  const int64_t m = g.m;
  for (const auto& s : g.segs) {
    const int64_t cnt = m * s.ncols;
    if (!s.transpose) {
      std::memcpy(dst, s.a, sizeof(double) * cnt);
    } else {
      // row-major (m x ncols) with row stride a_ld -> column-major: tiles
      // of 32 rows so both sides stay in cache lines
      for (int64_t i0 = 0; i0 < m; i0 += 32) {
        const int64_t i1 = std::min<int64_t>(m, i0 + 32);
        for (int64_t j = 0; j < s.ncols; ++j)
          for (int64_t i = i0; i < i1; ++i) dst[j * m + i] = s.a[i * s.a_ld + j];
      }
    }
    dst += cnt;
  }
}
}  // namespace

void pack_groups(const Plan& P, size_t g0, size_t g1, double* dst, int threads) {
  if (g0 >= g1) return;
  int64_t b0 = -1;
  std::vector<size_t> used;
  for (size_t g = g0; g < g1; ++g)
    if (P.groups[g].base >= 0) {
      if (b0 < 0) b0 = P.groups[g].base;
      used.push_back(g);
    }
  if (used.empty()) return;
  threads = std::max(1, std::min<int>(threads, (int)used.size()));
  auto work = [&](int t) {
    for (size_t k = t; k < used.size(); k += threads) {
      const Group& G = P.groups[used[k]];
      pack_one(G, dst + (G.base - b0));
    }
  };
  if (threads == 1) { work(0); return; }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
  for (auto& th : pool) th.join();
}

void pack_pool(Plan* P, int threads) {
  P->mat.assign((size_t)P->mat_len, 0.0);
  pack_groups(*P, 0, P->groups.size(), P->mat.data(), threads);
}

int build_plan(const h2b_desc* d, const PlanOptions& opt, Plan* out, std::string* err) {
  if (opt.world_size < 1 || opt.rank < 0 || opt.rank >= std::max(1, opt.world_size)) {
    *err = "rank must be in [0, world_size)";
    return H2B_EINVAL;
  }
  if (opt.task_bytes < 8 || opt.far_task_bytes < 8) { *err = "task_bytes must be >= 8"; return H2B_EINVAL; }
  Builder b(d, opt, out);
  return b.run(err);
}

}  // namespace h2b
