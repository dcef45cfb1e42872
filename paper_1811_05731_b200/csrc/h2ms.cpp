// h2ms.cpp — native H2MS v1 operator files and CRC-64/XZ.
//
// The reference persists an H2Matrix as "H2MS" v1 (hmatrix/persist.py:22-199):
// little-endian magic, u32 version, u64 N, the permutation, the preorder
// cluster tree, both sides' leaf bases / transfers, the coupling and near
// block lists, and a trailing CRC-64/XZ of every preceding byte.  Its
// reader is a Python byte walk with a table CRC at a few MB/s.
//
// Here a file is read once into memory, its checksum verified by all host
// cores (slicing-by-8 tables per thread, per-thread CRCs joined with the
// GF(2) "combine" identity), and parsed in one pass into an h2b_desc whose
// matrices sit in one aligned pool: h2b_create uploads from it directly, so
// an operator goes from disk to the device layout without Python objects.
// The writer emits the reference's byte layout exactly.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/h2b.h"

namespace h2b_detail {
int set_error(int code, const std::string& msg);  // defined in h2b.cu
}

namespace {

int iofail(const std::string& m) { return h2b_detail::set_error(H2B_EIO, m); }

// ---- CRC-64/XZ: reflected polynomial 0xC96C5795D7870F42, init and xorout
// all ones (persist.py:24-38).
constexpr uint64_t kPoly = 0xC96C5795D7870F42ull;

struct CrcTables {
  uint64_t t[8][256];
  CrcTables() {
    for (int b = 0; b < 256; ++b) {
      uint64_t c = (uint64_t)b;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
      t[0][b] = c;
    }
    for (int b = 0; b < 256; ++b)
      for (int s = 1; s < 8; ++s) t[s][b] = (t[s - 1][b] >> 8) ^ t[0][t[s - 1][b] & 0xff];
  }
};
const CrcTables& tables() {
  static const CrcTables T;
  return T;
}

// Raw register update (no init / xorout), eight bytes per step.
uint64_t crc_update(uint64_t crc, const unsigned char* p, size_t len) {
  const CrcTables& T = tables();
  while (len && ((uintptr_t)p & 7)) {
    crc = T.t[0][(crc ^ *p++) & 0xff] ^ (crc >> 8);
    --len;
  }
  while (len >= 8) {
    uint64_t w;
    std::memcpy(&w, p, 8);
    w ^= crc;
    crc = T.t[7][w & 0xff] ^ T.t[6][(w >> 8) & 0xff] ^ T.t[5][(w >> 16) & 0xff] ^ T.t[4][(w >> 24) & 0xff] ^
          T.t[3][(w >> 32) & 0xff] ^ T.t[2][(w >> 40) & 0xff] ^ T.t[1][(w >> 48) & 0xff] ^ T.t[0][w >> 56];
    p += 8;
    len -= 8;
  }
  while (len--) crc = T.t[0][(crc ^ *p++) & 0xff] ^ (crc >> 8);
  return crc;
}

// GF(2) 64x64 matrices as column vectors: the linear map "append n zero
// bytes" applied to a raw CRC register (the zlib crc32_combine method).
uint64_t gf2_times(const uint64_t* mat, uint64_t vec) {
  uint64_t sum = 0;
  for (int i = 0; vec; ++i, vec >>= 1)
    if (vec & 1) sum ^= mat[i];
  return sum;
}
void gf2_square(uint64_t* sq, const uint64_t* mat) {
  for (int n = 0; n < 64; ++n) sq[n] = gf2_times(mat, mat[n]);
}

// crc(A || B) from crc(A), crc(B) and |B| (all finalised CRC-64/XZ values).
uint64_t crc64_combine(uint64_t crc1, uint64_t crc2, uint64_t len2) {
  if (len2 == 0) return crc1;
  uint64_t even[64], odd[64];
  odd[0] = kPoly;  // one zero bit
  uint64_t row = 1;
  for (int n = 1; n < 64; ++n) {
    odd[n] = row;
    row <<= 1;
  }
  gf2_square(even, odd);  // two zero bits
  gf2_square(odd, even);  // four zero bits
  do {
    gf2_square(even, odd);
    if (len2 & 1) crc1 = gf2_times(even, crc1);
    len2 >>= 1;
    if (!len2) break;
    gf2_square(odd, even);
    if (len2 & 1) crc1 = gf2_times(odd, crc1);
    len2 >>= 1;
  } while (len2);
  return crc1 ^ crc2;
}

uint64_t crc64_parallel(const unsigned char* p, size_t len) {
  constexpr size_t kMinPerThread = 8u << 20;
  unsigned nt = std::max(1u, std::min(std::thread::hardware_concurrency(), 64u));
  if (const char* e = std::getenv("H2B_CRC_THREADS")) nt = std::max(1, std::atoi(e));  // tests
  nt = (unsigned)std::min<size_t>(nt, std::max<size_t>(1, len / kMinPerThread));
  if (nt <= 1) return crc_update(~0ull, p, len) ^ ~0ull;
  const size_t chunk = (len + nt - 1) / nt;
  std::vector<uint64_t> part(nt, 0);
  std::vector<size_t> plen(nt, 0);
  std::vector<std::thread> th;
  for (unsigned i = 0; i < nt; ++i) {
    const size_t b = std::min(len, (size_t)i * chunk), e = std::min(len, b + chunk);
    plen[i] = e - b;
    th.emplace_back([&, i, b, e] { part[i] = crc_update(~0ull, p + b, e - b) ^ ~0ull; });
  }
  for (auto& t : th) t.join();
  uint64_t crc = part[0];
  for (unsigned i = 1; i < nt; ++i) crc = crc64_combine(crc, part[i], plen[i]);
  return crc;
}

// ---- reader
struct Reader {
  const unsigned char* d;
  size_t len, pos = 0;
  bool take(size_t n, const unsigned char** out) {
    if (n > len - pos) return false;
    *out = d + pos;
    pos += n;
    return true;
  }
  bool u64(uint64_t* v) {
    const unsigned char* q;
    if (!take(8, &q)) return false;
    std::memcpy(v, q, 8);
    return true;
  }
};

}  // namespace

struct h2b_h2ms {
  std::vector<unsigned char> file;
  int64_t n = 0, nc = 0;
  std::vector<int64_t> perm, start, end, child, k_row, k_col;
  std::vector<double> bbox;     // [nc * 6] lo xyz, hi xyz
  std::vector<uint8_t> leaf;
  std::vector<double> pool;     // every matrix, 8-byte aligned, file order
  std::vector<int64_t> row_basis, col_basis, row_transfer, col_transfer;  // pool offsets or -1
  std::vector<int64_t> cp_row, cp_col, cp_off, nr_row, nr_col, nr_off;
  // pointer tables for the descriptor view
  std::vector<const double*> p_rb, p_cb, p_rt, p_ct, p_cp, p_nr;
};

namespace {

int parse(h2b_h2ms* f, int64_t expected_n) {
  const std::vector<unsigned char>& data = f->file;
  if (data.size() < 24) return iofail("truncated operator file");
  const size_t body_len = data.size() - 8;
  uint64_t stored;
  std::memcpy(&stored, data.data() + body_len, 8);
  if (crc64_parallel(data.data(), body_len) != stored) return iofail("operator file checksum mismatch");
  Reader rd{data.data(), body_len};
  const unsigned char* q;
  if (!rd.take(4, &q)) return iofail("truncated operator file");
  if (std::memcmp(q, "H2MS", 4) != 0) return iofail("bad magic number in operator file");
  if (!rd.take(4, &q)) return iofail("truncated operator file");
  uint32_t version;
  std::memcpy(&version, q, 4);
  if (version != 1) return iofail("unsupported operator file version " + std::to_string(version));
  uint64_t n;
  if (!rd.u64(&n)) return iofail("truncated operator file");
  if (expected_n >= 0 && (int64_t)n != expected_n)
    return iofail("operator file holds " + std::to_string(n) + " boundary nodes, mesh has " +
                  std::to_string(expected_n));
  if (n > body_len / 8) return iofail("truncated operator file");
  f->n = (int64_t)n;
  f->perm.resize(n);
  if (!rd.take(8 * n, &q)) return iofail("truncated operator file");
  std::memcpy(f->perm.data(), q, 8 * n);
  // cluster tree, preorder (persist.py:76-109)
  uint64_t count;
  if (!rd.u64(&count)) return iofail("truncated operator file");
  if (count > body_len / 65) return iofail("truncated operator file");
  const int64_t nc = (int64_t)count;
  f->nc = nc;
  f->start.assign(nc, 0);
  f->end.assign(nc, 0);
  f->child.assign(2 * nc, -1);
  f->bbox.assign(6 * nc, 0.0);
  f->leaf.assign(nc, 1);
  {
    // iterative preorder: a stack of (cluster id, next child slot to fill)
    int64_t next = 0;
    std::vector<std::pair<int64_t, int>> stack;
    auto read_node = [&](int64_t* id) -> int {
      if (next >= nc) return iofail("inconsistent cluster tree in operator file");
      if (!rd.take(65, &q)) return iofail("truncated operator file");
      const int64_t c = next++;
      uint64_t s, e;
      std::memcpy(&s, q, 8);
      std::memcpy(&e, q + 8, 8);
      f->start[c] = (int64_t)s;
      f->end[c] = (int64_t)e;
      std::memcpy(&f->bbox[6 * c], q + 16, 48);
      f->leaf[c] = q[64] ? 1 : 0;
      *id = c;
      return H2B_OK;
    };
    int64_t root;
    if (int rc = read_node(&root)) return rc;
    if (!f->leaf[root]) stack.push_back({root, 0});
    while (!stack.empty()) {
      auto& top = stack.back();
      if (top.second == 2) {
        stack.pop_back();
        continue;
      }
      int64_t c;
      if (int rc = read_node(&c)) return rc;
      f->child[2 * top.first + top.second] = c;
      ++top.second;
      if (!f->leaf[c]) stack.push_back({c, 0});
    }
    if (next != nc || f->start[0] != 0 || f->end[0] != (int64_t)n)
      return iofail("inconsistent cluster tree in operator file");
  }
  // matrices: first pass records (offset in file, rows, cols), then one
  // aligned pool receives every payload
  struct Mat { size_t at; uint64_t r, c; };
  std::vector<Mat> mats;
  auto matrix = [&](int64_t* idx) -> int {
    uint64_t r, c;
    if (!rd.u64(&r) || !rd.u64(&c)) return iofail("truncated operator file");
    if ((c != 0 && r > data.size() / c) || r * c > data.size()) return iofail("corrupt matrix header in operator file");
    const size_t at = rd.pos;
    if (!rd.take(8 * r * c, &q)) return iofail("truncated operator file");
    *idx = (int64_t)mats.size();
    mats.push_back({at, r, c});
    return H2B_OK;
  };
  f->row_basis.assign(nc, -1);
  f->col_basis.assign(nc, -1);
  f->row_transfer.assign(nc, -1);
  f->col_transfer.assign(nc, -1);
  for (int side = 0; side < 2; ++side) {
    auto& basis = side ? f->col_basis : f->row_basis;
    auto& transfer = side ? f->col_transfer : f->row_transfer;
    for (int64_t c = 0; c < nc; ++c) {
      if (f->leaf[c]) {
        if (int rc = matrix(&basis[c])) return rc;
      } else {
        for (int j = 0; j < 2; ++j)
          if (int rc = matrix(&transfer[f->child[2 * c + j]])) return rc;
      }
    }
  }
  for (int kind = 0; kind < 2; ++kind) {  // coupling (flag 1), then near (flag 0)
    uint64_t nb;
    if (!rd.u64(&nb)) return iofail("truncated operator file");
    if (nb > body_len / 33) return iofail("truncated operator file");
    auto& rr = kind ? f->nr_row : f->cp_row;
    auto& cc = kind ? f->nr_col : f->cp_col;
    auto& off = kind ? f->nr_off : f->cp_off;
    rr.resize(nb);
    cc.resize(nb);
    off.resize(nb);
    for (uint64_t b = 0; b < nb; ++b) {
      if (!rd.take(17, &q)) return iofail("truncated operator file");
      uint64_t r, c;
      std::memcpy(&r, q, 8);
      std::memcpy(&c, q + 8, 8);
      if (q[16] != (kind ? 0 : 1))
        return iofail(kind ? "near-field block with wrong admissibility flag"
                           : "coupling block with wrong admissibility flag");
      rr[b] = (int64_t)r;
      cc[b] = (int64_t)c;
      if (int rc = matrix(&off[b])) return rc;
    }
  }
  if (rd.pos != body_len) return iofail("trailing garbage in operator file");
  // pool
  size_t total = 0;
  std::vector<int64_t> moff(mats.size());
  for (size_t i = 0; i < mats.size(); ++i) {
    moff[i] = (int64_t)total;
    total += mats[i].r * mats[i].c;
  }
  f->pool.resize(std::max<size_t>(1, total));
  {
    const unsigned nt = std::max(1u, std::min(std::thread::hardware_concurrency(), 32u));
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        for (size_t i = t; i < mats.size(); i += nt)
          std::memcpy(f->pool.data() + moff[i], data.data() + mats[i].at, 8 * mats[i].r * mats[i].c);
      });
    for (auto& t : th) t.join();
  }
  // descriptor tables: matrix index -> pointer; ranks as H2Matrix.row_rank /
  // col_rank (h2.py:44-54: leaf basis width, else first child's transfer width)
  auto ptr = [&](int64_t i) -> const double* { return i < 0 ? nullptr : f->pool.data() + moff[i]; };
  auto cols = [&](int64_t i) -> int64_t { return i < 0 ? 0 : (int64_t)mats[i].c; };
  f->k_row.assign(nc, 0);
  f->k_col.assign(nc, 0);
  f->p_rb.assign(nc, nullptr);
  f->p_cb.assign(nc, nullptr);
  f->p_rt.assign(nc, nullptr);
  f->p_ct.assign(nc, nullptr);
  for (int64_t c = 0; c < nc; ++c) {
    f->p_rb[c] = ptr(f->row_basis[c]);
    f->p_cb[c] = ptr(f->col_basis[c]);
    f->p_rt[c] = ptr(f->row_transfer[c]);
    f->p_ct[c] = ptr(f->col_transfer[c]);
    if (f->leaf[c]) {
      f->k_row[c] = cols(f->row_basis[c]);
      f->k_col[c] = cols(f->col_basis[c]);
    } else {
      f->k_row[c] = cols(f->row_transfer[f->child[2 * c]]);
      f->k_col[c] = cols(f->col_transfer[f->child[2 * c]]);
    }
  }
  // shapes must be those of an H2Matrix (the planner relies on them; the
  // reference's reader would only fail later, inside the product)
  {
    auto sz = [&](int64_t c) { return f->end[c] - f->start[c]; };
    auto bad = [&]() { return iofail("inconsistent matrix shapes in operator file"); };
    for (int64_t c = 0; c < nc; ++c) {
      if (f->leaf[c]) {
        for (int side = 0; side < 2; ++side) {
          const int64_t i = side ? f->col_basis[c] : f->row_basis[c];
          if ((int64_t)mats[i].r != sz(c)) return bad();
        }
      } else {
        for (int j = 0; j < 2; ++j) {
          const int64_t ch = f->child[2 * c + j];
          if ((int64_t)mats[f->row_transfer[ch]].r != f->k_row[ch] || (int64_t)mats[f->row_transfer[ch]].c != f->k_row[c] ||
              (int64_t)mats[f->col_transfer[ch]].r != f->k_col[ch] || (int64_t)mats[f->col_transfer[ch]].c != f->k_col[c])
            return bad();
        }
      }
    }
    for (size_t b = 0; b < f->cp_row.size(); ++b) {
      const int64_t t = f->cp_row[b], u = f->cp_col[b];
      if (t < 0 || t >= nc || u < 0 || u >= nc) return iofail("block cluster id out of range in operator file");
      if ((int64_t)mats[f->cp_off[b]].r != f->k_row[t] || (int64_t)mats[f->cp_off[b]].c != f->k_col[u]) return bad();
    }
    for (size_t b = 0; b < f->nr_row.size(); ++b) {
      const int64_t t = f->nr_row[b], u = f->nr_col[b];
      if (t < 0 || t >= nc || u < 0 || u >= nc) return iofail("block cluster id out of range in operator file");
      if ((int64_t)mats[f->nr_off[b]].r != sz(t) || (int64_t)mats[f->nr_off[b]].c != sz(u)) return bad();
    }
  }
  f->p_cp.resize(f->cp_off.size());
  for (size_t b = 0; b < f->cp_off.size(); ++b) f->p_cp[b] = ptr(f->cp_off[b]);
  f->p_nr.resize(f->nr_off.size());
  for (size_t b = 0; b < f->nr_off.size(); ++b) f->p_nr[b] = ptr(f->nr_off[b]);
  f->file.clear();
  f->file.shrink_to_fit();
  return H2B_OK;
}

// ---- writer helpers
struct Out {
  std::vector<unsigned char> buf;
  void put(const void* p, size_t n) {
    const unsigned char* c = (const unsigned char*)p;
    buf.insert(buf.end(), c, c + n);
  }
  void u64(uint64_t v) { put(&v, 8); }
  void matrix(const double* a, int64_t r, int64_t c) {
    u64((uint64_t)r);
    u64((uint64_t)c);
    if (r * c) put(a, 8 * (size_t)(r * c));
  }
};

}  // namespace

extern "C" {

uint64_t h2b_crc64(const void* data, uint64_t len) {
  return crc64_parallel((const unsigned char*)data, (size_t)len);
}

int h2b_h2ms_open(const char* path, int64_t expected_n, h2b_h2ms** out) {
  if (!path || !out) return h2b_detail::set_error(H2B_EINVAL, "null argument");
  *out = nullptr;
  std::unique_ptr<h2b_h2ms> f(new (std::nothrow) h2b_h2ms());
  if (!f) return h2b_detail::set_error(H2B_ENOMEM, "out of host memory");
  FILE* fp = std::fopen(path, "rb");
  if (!fp) return iofail(std::string("cannot open operator file ") + path);
  std::fseek(fp, 0, SEEK_END);
  const long sz = std::ftell(fp);
  std::fseek(fp, 0, SEEK_SET);
  if (sz < 0) {
    std::fclose(fp);
    return iofail("cannot read operator file");
  }
  try {
    f->file.resize((size_t)sz);
  } catch (...) {
    std::fclose(fp);
    return h2b_detail::set_error(H2B_ENOMEM, "out of host memory");
  }
  const size_t got = sz ? std::fread(f->file.data(), 1, (size_t)sz, fp) : 0;
  std::fclose(fp);
  if (got != (size_t)sz) return iofail("cannot read operator file");
  if (int rc = parse(f.get(), expected_n)) return rc;
  *out = f.release();
  return H2B_OK;
}

int h2b_h2ms_desc(const h2b_h2ms* f, h2b_desc* d) {
  if (!f || !d) return h2b_detail::set_error(H2B_EINVAL, "null argument");
  std::memset(d, 0, sizeof(*d));
  d->n = f->n;
  d->nclusters = f->nc;
  d->perm = f->perm.data();
  d->cl_start = f->start.data();
  d->cl_end = f->end.data();
  d->cl_child = f->child.data();
  d->k_row = f->k_row.data();
  d->k_col = f->k_col.data();
  d->row_basis = f->p_rb.data();
  d->col_basis = f->p_cb.data();
  d->row_transfer = f->p_rt.data();
  d->col_transfer = f->p_ct.data();
  d->ncoupling = (int64_t)f->cp_row.size();
  d->cp_row = f->cp_row.data();
  d->cp_col = f->cp_col.data();
  d->cp_data = f->p_cp.data();
  d->nnear = (int64_t)f->nr_row.size();
  d->nr_row = f->nr_row.data();
  d->nr_col = f->nr_col.data();
  d->nr_data = f->p_nr.data();
  return H2B_OK;
}

int h2b_h2ms_tree(const h2b_h2ms* f, double* bbox, uint8_t* leaf) {
  if (!f) return h2b_detail::set_error(H2B_EINVAL, "null argument");
  if (bbox) std::memcpy(bbox, f->bbox.data(), sizeof(double) * f->bbox.size());
  if (leaf) std::memcpy(leaf, f->leaf.data(), f->leaf.size());
  return H2B_OK;
}

void h2b_h2ms_close(h2b_h2ms* f) { delete f; }

int h2b_h2ms_write(const h2b_desc* d, const double* bbox, const char* path) {
  if (!d || !bbox || !path) return h2b_detail::set_error(H2B_EINVAL, "null argument");
  const int64_t nc = d->nclusters;
  Out o;
  try {
    o.put("H2MS", 4);
    const uint32_t version = 1;
    o.put(&version, 4);
    o.u64((uint64_t)d->n);
    o.put(d->perm, 8 * (size_t)d->n);
    // preorder tree: cluster ids are preorder, so id order is file order
    o.u64((uint64_t)nc);
    for (int64_t c = 0; c < nc; ++c) {
      o.u64((uint64_t)d->cl_start[c]);
      o.u64((uint64_t)d->cl_end[c]);
      o.put(bbox + 6 * c, 48);
      const unsigned char lf = d->cl_child[2 * c] < 0 ? 1 : 0;
      o.put(&lf, 1);
    }
    auto size = [&](int64_t c) { return d->cl_end[c] - d->cl_start[c]; };
    for (int side = 0; side < 2; ++side) {
      const double* const* basis = side ? d->col_basis : d->row_basis;
      const double* const* transfer = side ? d->col_transfer : d->row_transfer;
      const int64_t* k = side ? d->k_col : d->k_row;
      for (int64_t c = 0; c < nc; ++c) {
        if (d->cl_child[2 * c] < 0) {
          o.matrix(basis[c], size(c), k[c]);
        } else {
          for (int j = 0; j < 2; ++j) {
            const int64_t ch = d->cl_child[2 * c + j];
            o.matrix(transfer[ch], k[ch], k[c]);
          }
        }
      }
    }
    o.u64((uint64_t)d->ncoupling);
    for (int64_t b = 0; b < d->ncoupling; ++b) {
      o.u64((uint64_t)d->cp_row[b]);
      o.u64((uint64_t)d->cp_col[b]);
      const unsigned char fl = 1;
      o.put(&fl, 1);
      o.matrix(d->cp_data[b], d->k_row[d->cp_row[b]], d->k_col[d->cp_col[b]]);
    }
    o.u64((uint64_t)d->nnear);
    for (int64_t b = 0; b < d->nnear; ++b) {
      o.u64((uint64_t)d->nr_row[b]);
      o.u64((uint64_t)d->nr_col[b]);
      const unsigned char fl = 0;
      o.put(&fl, 1);
      o.matrix(d->nr_data[b], size(d->nr_row[b]), size(d->nr_col[b]));
    }
  } catch (...) {
    return h2b_detail::set_error(H2B_ENOMEM, "out of host memory");
  }
  const uint64_t crc = crc64_parallel(o.buf.data(), o.buf.size());
  o.u64(crc);
  FILE* fp = std::fopen(path, "wb");
  if (!fp) return iofail(std::string("cannot write operator file ") + path);
  const size_t put = std::fwrite(o.buf.data(), 1, o.buf.size(), fp);
  const int cl = std::fclose(fp);
  if (put != o.buf.size() || cl != 0) return iofail(std::string("cannot write operator file ") + path);
  return H2B_OK;
}

}  // extern "C"
