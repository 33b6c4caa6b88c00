// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// Builds the reference's own primitives (/root/reference/proj/src/tensor.cpp
// and id.cpp, compiled where they lie, against the from-scratch Eigen-API shim
// in include/eigen_shim) and exposes them through a C ABI so tests can pin the
// oracle restatement (oracle/tbf_oracle.cpp) against the reference itself.
// id.cpp is #included (by its path under /root/reference, see oracle/Makefile)
// so that its anonymous-namespace helpers qrcp() and proxy_lists() are
// reachable from this translation unit; no reference source is copied.
//
// Output: oracle/_ref/libref.so (git-ignored).
#include "oiobf/id.hpp"
#include "oiobf/rng.hpp"
#include "oiobf/tensor.hpp"

#include REF_TENSOR_CPP
#include REF_ID_CPP

#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>

using namespace oiobf;

namespace {
thread_local std::string g_err;

void cplx_in(const double* p, std::int64_t n, Complex* out) {
  for (std::int64_t i = 0; i < n; ++i) out[i] = Complex(p[2 * i], p[2 * i + 1]);
}
void cplx_out(const Complex* p, std::int64_t n, double* out) {
  for (std::int64_t i = 0; i < n; ++i) {
    out[2 * i] = p[i].real();
    out[2 * i + 1] = p[i].imag();
  }
}
Matrix mat_in(std::int64_t m, std::int64_t n, const double* a) {
  Matrix out(m, n);
  cplx_in(a, m * n, out.data());
  return out;
}

// Kernel catalog restated from BASELINE.json configs / SURVEY.md App. A1 (the
// reference has no kernel code, SPEC.md:329-395 only).  Same formulas as
// oracle/tbf_oracle.cpp; kind: 0 green (d=2 plates / d=3 cubes), 1 dft, 2 radon2d.
struct Spec {
  int kind;
  int d;
  std::int64_t n;
  double kappa;
  double offset[3];
  int bitrev;  // 1: two-sided per-mode bit reversal (DFT)
};

std::int64_t bitrev1(std::int64_t i, std::int64_t n) {  // 1-based
  std::int64_t x = i - 1, r = 0;
  for (std::int64_t b = 1; b < n; b <<= 1) {
    r = (r << 1) | (x & 1);
    x >>= 1;
  }
  return r + 1;
}

Complex eval_spec(const Spec& s, const MultiIndex& i, const MultiIndex& j) {
  const double n = static_cast<double>(s.n);
  if (s.kind == 0) {
    double xs[3] = {0, 0, 0}, ys[3] = {0, 0, 0};
    for (int p = 0; p < s.d; ++p) {
      xs[p] = static_cast<double>(i[p]) / n;
      ys[p] = static_cast<double>(j[p]) / n;
    }
    for (int p = 0; p < 3; ++p) ys[p] += s.offset[p];
    const double dx = xs[0] - ys[0], dy = xs[1] - ys[1], dz = xs[2] - ys[2];
    const double rho = std::sqrt(dx * dx + dy * dy + dz * dz);
    const double ph = s.kappa * rho;
    return Complex(std::cos(ph) / rho, -std::sin(ph) / rho);
  }
  if (s.kind == 1) {
    std::int64_t acc = 0;
    for (int p = 0; p < s.d; ++p) {
      std::int64_t a = s.bitrev ? bitrev1(i[p], s.n) : i[p];
      std::int64_t b = s.bitrev ? bitrev1(j[p], s.n) : j[p];
      acc += (a - 1) * (b - 1 - s.n / 2);
    }
    std::int64_t m = acc % s.n;
    if (m < 0) m += s.n;
    // exp(-2 pi i m / n)
    const double t = 2.0 * static_cast<double>(m) / n;
    return Complex(std::cos(M_PI * t), -std::sin(M_PI * t));
  }
  // radon 2d: Phi = x.k + sqrt(c1^2 k1^2 + c2^2 k2^2)
  const double x1 = static_cast<double>(i[0] - 1) / n, x2 = static_cast<double>(i[1] - 1) / n;
  const std::int64_t k1i = j[0] - 1 - s.n / 2, k2i = j[1] - 1 - s.n / 2;
  const double k1 = static_cast<double>(k1i), k2 = static_cast<double>(k2i);
  const double s1 = std::sin(2.0 * M_PI * x1), s2 = std::sin(2.0 * M_PI * x2);
  const double c1v = std::cos(2.0 * M_PI * x1), c2v = std::cos(2.0 * M_PI * x2);
  const double c1 = (2.0 + s1 * s2) / 16.0, c2 = (2.0 + c1v * c2v) / 16.0;
  std::int64_t num = ((i[0] - 1) * k1i + (i[1] - 1) * k2i) % s.n;
  if (num < 0) num += s.n;
  const double frac = static_cast<double>(num) / n;
  const double phi = frac + std::sqrt(c1 * c1 * k1 * k1 + c2 * c2 * k2 * k2);
  const double ph = 2.0 * M_PI * phi;
  return Complex(std::cos(ph), std::sin(ph));
}

KernelEvaluator make_eval(const Spec& s) {
  KernelEvaluator k;
  k.d = s.d;
  k.row_extents.assign(static_cast<std::size_t>(s.d), s.n);
  k.col_extents.assign(static_cast<std::size_t>(s.d), s.n);
  k.eval = [s](const MultiIndex& i, const MultiIndex& j) { return eval_spec(s, i, j); };
  return k;
}

void write_id(const ColumnID& id, std::int64_t ncols, std::int64_t* rank, std::int64_t* skel, double* interp,
              int* saturated, double* interp_max_abs) {
  *rank = id.rank;
  for (std::int64_t i = 0; i < id.rank; ++i) skel[i] = id.skeleton[static_cast<std::size_t>(i)];
  cplx_out(id.interp.data(), id.rank * ncols, interp);
  if (saturated) *saturated = id.saturated ? 1 : 0;
  if (interp_max_abs) *interp_max_abs = id.interp_max_abs;
}

ProxyStrategy strat(int mode, std::int64_t q, std::int64_t max_retries, std::int64_t row_cap) {
  ProxyStrategy p;
  p.mode = static_cast<ProxyMode>(mode);
  p.q = q;
  p.max_retries = max_retries;
  p.row_cap = row_cap;
  return p;
}

}  // namespace

#define GUARD_BEGIN try {
#define GUARD_END                  \
  }                                \
  catch (const std::exception& e) { \
    g_err = e.what();              \
    return -1;                     \
  }                                \
  return 0;

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::uint64_t ref_splitmix_next(std::uint64_t* state) {
  SplitMix64 g(*state);
  std::uint64_t v = g.next();
  *state = g.state;
  return v;
}

std::uint64_t ref_splitmix_bounded(std::uint64_t* state, std::uint64_t bound) {
  SplitMix64 g(*state);
  std::uint64_t v = g.bounded(bound);
  *state = g.state;
  return v;
}

std::uint64_t ref_derive_seed(std::uint64_t seed, const std::uint64_t* t, int nt) {
  switch (nt) {
    case 0: return derive_seed(seed, {});
    case 1: return derive_seed(seed, {t[0]});
    case 2: return derive_seed(seed, {t[0], t[1]});
    case 3: return derive_seed(seed, {t[0], t[1], t[2]});
    case 4: return derive_seed(seed, {t[0], t[1], t[2], t[3]});
    case 5: return derive_seed(seed, {t[0], t[1], t[2], t[3], t[4]});
    case 6: return derive_seed(seed, {t[0], t[1], t[2], t[3], t[4], t[5]});
    case 7: return derive_seed(seed, {t[0], t[1], t[2], t[3], t[4], t[5], t[6]});
    default: return derive_seed(seed, {t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7]});
  }
}

int ref_select_proxies_count(std::int64_t extent, std::int64_t count, int mode, std::uint64_t seed,
                             std::int64_t* out, std::int64_t* out_n) {
  GUARD_BEGIN
  IndexList l = select_proxies_count(extent, count, static_cast<ProxyMode>(mode), seed);
  *out_n = static_cast<std::int64_t>(l.size());
  for (std::size_t i = 0; i < l.size(); ++i) out[i] = l[i];
  GUARD_END
}

int ref_select_proxies(std::int64_t extent, std::int64_t rank_estimate, int mode, std::int64_t q,
                       std::uint64_t seed, std::int64_t* out, std::int64_t* out_n) {
  GUARD_BEGIN
  IndexList l = select_proxies(extent, rank_estimate, strat(mode, q, 3, 1 << 17), seed);
  *out_n = static_cast<std::int64_t>(l.size());
  for (std::size_t i = 0; i < l.size(); ++i) out[i] = l[i];
  GUARD_END
}

// The reference's private proxy_lists (id.cpp:199-231).  out_counts[nr];
// out_lists concatenated in mode order (skip mode contributes nothing).
int ref_proxy_lists(int nr, const std::int64_t* lo, const std::int64_t* hi, int skip, std::int64_t per_mode,
                    int mode, std::int64_t q, std::int64_t row_cap, std::uint64_t seed, std::int64_t* out_counts,
                    std::int64_t* out_lists) {
  GUARD_BEGIN
  std::vector<IndexRange> ranges(static_cast<std::size_t>(nr));
  for (int p = 0; p < nr; ++p) ranges[static_cast<std::size_t>(p)] = IndexRange{lo[p], hi[p]};
  auto lists = proxy_lists(ranges, static_cast<std::size_t>(skip), per_mode, strat(mode, q, 3, row_cap), seed);
  std::int64_t pos = 0;
  for (int p = 0; p < nr; ++p) {
    const auto& l = lists[static_cast<std::size_t>(p)];
    out_counts[p] = static_cast<std::int64_t>(l.size());
    for (auto v : l) out_lists[pos++] = v;
  }
  GUARD_END
}

// qrcp (id.cpp:24-85): perm (n, 0-based), R (rank x n col-major), rank, saturated.
int ref_qrcp(std::int64_t m, std::int64_t n, const double* a, double tol, std::int64_t limit, std::int64_t* perm,
             double* r, std::int64_t* rank, int* saturated) {
  GUARD_BEGIN
  QrcpResult q = qrcp(mat_in(m, n, a), tol, limit);
  for (std::int64_t j = 0; j < n; ++j) perm[j] = q.perm[static_cast<std::size_t>(j)];
  *rank = q.rank;
  *saturated = q.saturated ? 1 : 0;
  cplx_out(q.r.data(), q.rank * n, r);
  GUARD_END
}

// column_id (id.cpp:124-130); max_rank < 0 means std::nullopt.
int ref_column_id(std::int64_t m, std::int64_t n, const double* a, double tol, std::int64_t max_rank,
                  std::int64_t* rank, std::int64_t* skel, double* interp, int* saturated, double* interp_max_abs) {
  GUARD_BEGIN
  std::optional<std::int64_t> mr;
  if (max_rank >= 0) mr = max_rank;
  ColumnID id = column_id(mat_in(m, n, a), tol, mr);
  write_id(id, n, rank, skel, interp, saturated, interp_max_abs);
  GUARD_END
}

// One butterfly ID slot composed exclusively of reference primitives, exactly
// the per-mode step of tucker_id (id.cpp:257-267) with the target range
// replaced by an explicit target list: proxy_lists -> subtensor_at -> unfold
// -> column_id.  ranges: 2d (lo,hi) pairs; skip = unfolded mode (0-based).
int ref_slot_id(const int* spec_i, const double* spec_f, const std::int64_t* lo, const std::int64_t* hi, int skip,
                const std::int64_t* target, std::int64_t ntarget, std::int64_t per_mode, int mode, std::int64_t q,
                std::int64_t row_cap, std::uint64_t seed, double tol, std::int64_t* rows_out, std::int64_t* rank,
                std::int64_t* skel, double* interp) {
  GUARD_BEGIN
  Spec s{spec_i[0], spec_i[1], spec_i[2], spec_f[0], {spec_f[1], spec_f[2], spec_f[3]}, spec_i[3]};
  KernelEvaluator k = make_eval(s);
  const std::size_t d = static_cast<std::size_t>(s.d);
  std::vector<IndexRange> ranges(2 * d);
  for (std::size_t p = 0; p < 2 * d; ++p) ranges[p] = IndexRange{lo[p], hi[p]};
  auto lists = proxy_lists(ranges, static_cast<std::size_t>(skip), per_mode, strat(mode, q, 3, row_cap), seed);
  lists[static_cast<std::size_t>(skip)] = IndexList(target, target + ntarget);
  std::vector<IndexList> rl(lists.begin(), lists.begin() + static_cast<std::ptrdiff_t>(d));
  std::vector<IndexList> cl(lists.begin() + static_cast<std::ptrdiff_t>(d), lists.end());
  DenseTensor sub = subtensor_at(k, rl, cl);
  Matrix unf = unfold(sub, skip + 1).m;
  *rows_out = unf.rows();
  ColumnID id = column_id(unf, tol);
  // report the skeleton globally (as tucker_id does, id.cpp:274-275)
  for (auto& v : id.skeleton) v = target[v - 1];
  write_id(id, ntarget, rank, skel, interp, nullptr, nullptr);
  GUARD_END
}

// Materialize K(rows, cols) with subtensor_at (tensor.cpp:249-266); lists are
// concatenated, counts per mode; output first-mode-fastest complex.
int ref_subtensor_at(const int* spec_i, const double* spec_f, const std::int64_t* counts, const std::int64_t* lists,
                     double* out) {
  GUARD_BEGIN
  Spec s{spec_i[0], spec_i[1], spec_i[2], spec_f[0], {spec_f[1], spec_f[2], spec_f[3]}, spec_i[3]};
  KernelEvaluator k = make_eval(s);
  std::vector<IndexList> rl, cl;
  std::int64_t pos = 0;
  for (int p = 0; p < 2 * s.d; ++p) {
    IndexList l(lists + pos, lists + pos + counts[p]);
    pos += counts[p];
    (p < s.d ? rl : cl).push_back(std::move(l));
  }
  DenseTensor t = subtensor_at(k, rl, cl);
  cplx_out(t.data().data(), t.size(), out);
  GUARD_END
}

// Full reference tucker_id (id.cpp:235-287).  Outputs: ranks[2d]; skeletons
// concatenated (row modes then col modes); interps concatenated col-major
// (U^k r_k x |tau_k|, then V^k); core first-mode-fastest.
int ref_tucker_id(const int* spec_i, const double* spec_f, const std::int64_t* lo, const std::int64_t* hi, double tol,
                  int mode, std::int64_t q, std::int64_t max_retries, std::int64_t row_cap, std::uint64_t seed,
                  std::int64_t* ranks, std::int64_t* skel, double* interp, double* core, std::int64_t* mem_bytes) {
  GUARD_BEGIN
  Spec s{spec_i[0], spec_i[1], spec_i[2], spec_f[0], {spec_f[1], spec_f[2], spec_f[3]}, spec_i[3]};
  KernelEvaluator k = make_eval(s);
  MultiSet rows, cols;
  for (int p = 0; p < s.d; ++p) rows.push_back(IndexRange{lo[p], hi[p]});
  for (int p = 0; p < s.d; ++p) cols.push_back(IndexRange{lo[s.d + p], hi[s.d + p]});
  TuckerID t = tucker_id(k, rows, cols, tol, strat(mode, q, max_retries, row_cap), seed);
  std::int64_t sp = 0, ip = 0;
  for (int m = 0; m < 2 * s.d; ++m) {
    ranks[m] = t.ranks[static_cast<std::size_t>(m)];
    const IndexList& sk = m < s.d ? t.row_skeletons[static_cast<std::size_t>(m)]
                                  : t.col_skeletons[static_cast<std::size_t>(m - s.d)];
    for (auto v : sk) skel[sp++] = v;
    const Matrix& f = m < s.d ? t.row_interp[static_cast<std::size_t>(m)] : t.col_interp[static_cast<std::size_t>(m - s.d)];
    cplx_out(f.data(), f.size(), interp + 2 * ip);
    ip += f.size();
  }
  cplx_out(t.core.data().data(), t.core.size(), core);
  *mem_bytes = t.memory_bytes();
  GUARD_END
}

// tucker_contract on a tucker_id computed with the same arguments.
int ref_tucker_contract(const int* spec_i, const double* spec_f, const std::int64_t* lo, const std::int64_t* hi,
                        double tol, int mode, std::int64_t q, std::int64_t max_retries, std::int64_t row_cap,
                        std::uint64_t seed, std::int64_t nv, const double* f, double* g) {
  GUARD_BEGIN
  Spec s{spec_i[0], spec_i[1], spec_i[2], spec_f[0], {spec_f[1], spec_f[2], spec_f[3]}, spec_i[3]};
  KernelEvaluator k = make_eval(s);
  MultiSet rows, cols;
  for (int p = 0; p < s.d; ++p) rows.push_back(IndexRange{lo[p], hi[p]});
  for (int p = 0; p < s.d; ++p) cols.push_back(IndexRange{lo[s.d + p], hi[s.d + p]});
  TuckerID t = tucker_id(k, rows, cols, tol, strat(mode, q, max_retries, row_cap), seed);
  std::vector<std::int64_t> shape;
  std::int64_t total = nv;
  for (auto& c : cols) {
    shape.push_back(c.size());
    total *= c.size();
  }
  shape.push_back(nv);
  std::vector<Complex> data(static_cast<std::size_t>(total));
  cplx_in(f, total, data.data());
  DenseTensor ft(shape, data);
  DenseTensor gt = tucker_contract(t, ft);
  cplx_out(gt.data().data(), gt.size(), g);
  GUARD_END
}

// mode_product_blockdiag (tensor.cpp:136-166).  blocks: nb matrices with
// shapes (br[i], bc[i]) concatenated col-major.
int ref_mode_product_blockdiag(int nmodes, const std::int64_t* shape, const double* t, int mode, int nb,
                               const std::int64_t* br, const std::int64_t* bc, const double* blocks, int transpose,
                               double* out) {
  GUARD_BEGIN
  std::vector<std::int64_t> sh(shape, shape + nmodes);
  std::int64_t total = 1;
  for (auto e : sh) total *= e;
  std::vector<Complex> data(static_cast<std::size_t>(total));
  cplx_in(t, total, data.data());
  DenseTensor tt(sh, data);
  std::vector<Matrix> mats;
  std::int64_t pos = 0;
  for (int b = 0; b < nb; ++b) {
    mats.push_back(mat_in(br[b], bc[b], blocks + 2 * pos));
    pos += br[b] * bc[b];
  }
  std::vector<const Matrix*> ptrs;
  for (auto& m : mats) ptrs.push_back(&m);
  DenseTensor o = mode_product_blockdiag(tt, mode, ptrs, transpose != 0);
  cplx_out(o.data().data(), o.size(), out);
  GUARD_END
}

}  // extern "C"
