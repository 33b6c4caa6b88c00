// oiobf drop-in: tensor butterfly (Alg. 1 / Alg. 2).
// The reference ships this module as specification only; this is the API the
// spec defines, backed by the B200 library (factors and cores stay in HBM).
#ifndef OIOBF_DROPIN_BUTTERFLY_HPP
#define OIOBF_DROPIN_BUTTERFLY_HPP

#include <map>
#include <memory>
#include <random>
#include <set>

#include "oiobf/id.hpp"
#include "oiobf/kernels.hpp"

namespace oiobf {

struct TbfMemory {
  std::int64_t V = 0, W = 0, U = 0, P = 0, cores = 0;
  std::int64_t total() const { return V + W + U + P + cores; }
};

// Flat host copy of a factorization (canonical slot order).
struct TbfExport {
  std::int64_t d = 0, n = 0, L = 0, Lc = 0, nmid = 0;
  std::vector<std::int64_t> ranks, ncols, rows, skel, perm, core_rows, core_cols, r_est;
  std::vector<Complex> interp, cores;
};

class TensorButterfly {
 public:
  TensorButterfly() = default;
  TensorButterfly(oiobf_tbf* h, KernelEvaluator k, std::int64_t L, double tol)
      : h_(h, &oiobf_tbf_destroy), eval_(std::move(k)), L_(L), tol_(tol) {}

  std::int64_t d() const { return eval_.d; }
  std::int64_t levels() const { return L_; }
  double tolerance() const { return tol_; }
  const KernelEvaluator& evaluator() const { return eval_; }
  oiobf_tbf* handle() const { return h_.get(); }

  // Core storage for the apply: false = FP64 (exact, default), true = block
  // floating point (the ZFP step of PAPER.md Alg. 2; oiobf_tbf_set_core_format)
  void compress_cores(bool on) { detail::check(oiobf_tbf_set_core_format(h_.get(), on ? 1 : 0)); }

  TbfMemory memory() const {
    std::int64_t m[5];
    detail::check(oiobf_tbf_memory(h_.get(), m));
    return TbfMemory{m[0], m[1], m[2], m[3], m[4]};
  }

  TbfExport export_factors() const {
    std::int64_t info[10];
    detail::check(oiobf_tbf_info(h_.get(), info));
    TbfExport e;
    e.d = info[0];
    e.n = info[1];
    e.L = info[2];
    e.Lc = info[3];
    e.nmid = info[4];
    const auto ns = static_cast<std::size_t>(info[5]);
    e.ranks.resize(ns);
    e.ncols.resize(ns);
    e.rows.resize(ns);
    e.skel.resize(static_cast<std::size_t>(info[6]));
    e.interp.resize(static_cast<std::size_t>(info[7]));
    e.cores.resize(static_cast<std::size_t>(info[8]));
    e.perm.resize(static_cast<std::size_t>(info[9]));
    e.core_rows.resize(static_cast<std::size_t>(e.nmid * e.nmid));
    e.core_cols.resize(static_cast<std::size_t>(e.nmid * e.nmid));
    e.r_est.resize(static_cast<std::size_t>(2 * (e.Lc + 1)));
    detail::check(oiobf_tbf_export(h_.get(), e.ranks.data(), e.ncols.data(), e.rows.data(), e.skel.data(),
                                   reinterpret_cast<double*>(e.interp.data()), e.perm.data(),
                                   reinterpret_cast<double*>(e.cores.data()), e.core_rows.data(), e.core_cols.data(),
                                   e.r_est.data()));
    return e;
  }

 private:
  std::shared_ptr<oiobf_tbf> h_;
  KernelEvaluator eval_;
  std::int64_t L_ = 0;
  double tol_ = 0;
};

// Alg. 1.  L even, n = C_b * 2^L per mode.
inline TensorButterfly tbf_construct(const KernelEvaluator& eval, std::int64_t L, double tol,
                                     const ProxyStrategy& proxies, std::uint64_t seed) {
  const oiobf_kernel_spec& spec = eval.device_spec();
  oiobf_proxy_strategy ps{};
  ps.mode = static_cast<int32_t>(proxies.mode);
  ps.q = proxies.q;
  ps.max_retries = proxies.max_retries;
  ps.row_cap = proxies.row_cap;
  oiobf_tbf* h = nullptr;
  detail::check(oiobf_tbf_construct(&spec, static_cast<int32_t>(L), tol, &ps, seed, &h));
  return TensorButterfly(h, eval, L, tol);
}

// Alg. 2: G = K x_{d+1..2d} F, F of shape (n_1..n_d, n_v) (or (n_1..n_d)).
inline DenseTensor tbf_contract(const TensorButterfly& bf, const DenseTensor& F) {
  const std::int64_t d = bf.d();
  require(F.mode_count() == d || F.mode_count() == d + 1, "tbf_contract: input must have d or d+1 modes");
  for (std::int64_t k = 0; k < d; ++k)
    require(F.extent(k + 1) == bf.evaluator().col_extents[static_cast<std::size_t>(k)], "tbf_contract: shape mismatch");
  const std::int64_t nv = F.mode_count() == d + 1 ? F.extent(d + 1) : 1;
  DenseTensor G(F.shape());
  detail::check(oiobf_tbf_contract(bf.handle(), reinterpret_cast<const double*>(F.data().data()),
                                   reinterpret_cast<double*>(G.data().data()), nv));
  return G;
}

inline TbfMemory tbf_memory(const TensorButterfly& bf) { return bf.memory(); }

// F_e = 1 at n_samples random entries; exact result = sum of
// those kernel columns (evaluated on the GPU); relative Frobenius error.
inline double tbf_error_estimate(const TensorButterfly& bf, const KernelEvaluator& eval, std::int64_t n_samples,
                                 std::uint64_t seed) {
  require(n_samples >= 1, "tbf_error_estimate: n_samples must be >= 1");
  const std::int64_t d = eval.d;
  std::vector<std::int64_t> shape(eval.col_extents.begin(), eval.col_extents.end());
  DenseTensor Fe(shape);
  SplitMix64 g(seed);
  std::set<std::int64_t> picked;
  while (static_cast<std::int64_t>(picked.size()) < std::min<std::int64_t>(n_samples, Fe.size()))
    picked.insert(static_cast<std::int64_t>(g.bounded(static_cast<std::uint64_t>(Fe.size()))));
  for (auto f : picked) Fe.data()[static_cast<std::size_t>(f)] = Complex(1, 0);
  const DenseTensor G = tbf_contract(bf, Fe);
  std::vector<IndexList> full;
  for (auto e : eval.row_extents) full.push_back(range_to_list({1, e}));
  double num = 0, den = 0;
  std::vector<Complex> exact(static_cast<std::size_t>(G.size()), Complex(0, 0));
  for (auto f : picked) {
    const MultiIndex j = Fe.unflatten(f);
    std::vector<IndexList> cols;
    for (std::int64_t k = 0; k < d; ++k) cols.push_back({j[static_cast<std::size_t>(k)]});
    const DenseTensor col = subtensor_at(eval, full, cols);
    for (std::size_t q = 0; q < exact.size(); ++q) exact[q] += col.data()[q];
  }
  for (std::size_t q = 0; q < exact.size(); ++q) {
    num += std::norm(G.data()[q] - exact[q]);
    den += std::norm(exact[q]);
  }
  return std::sqrt(num / den);
}

}  // namespace oiobf

#endif
