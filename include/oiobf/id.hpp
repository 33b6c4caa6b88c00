// oiobf drop-in: interpolative decompositions (reference proj/include/oiobf/
// id.hpp:9-94).  The column-pivoted QR runs on the B200 (oiobf_column_id_batch:
// TSQR + the reference's pivoting on R); entry generation for tucker_id runs on
// the B200 (subtensor_at); proxy index sets are integer metadata computed with
// the reference's rules (bit-exact with the device generator).
#ifndef OIOBF_DROPIN_ID_HPP
#define OIOBF_DROPIN_ID_HPP

#include <algorithm>
#include <numeric>
#include <optional>

#include "oiobf/rng.hpp"
#include "oiobf/tensor.hpp"
#include "oiobf/types.hpp"

namespace oiobf {

struct ColumnID {
  IndexList skeleton;  // sorted, 1-based
  Matrix interp;       // rank x ncols; interp(:, skeleton[i]) = e_i
  std::int64_t rank = 0;
  bool saturated = false;
  double interp_max_abs = 0;
};

struct RowID {
  IndexList skeleton;
  Matrix interp;  // nrows x rank
  std::int64_t rank = 0;
  bool saturated = false;
  double interp_max_abs = 0;
};

struct HybridID {
  RowID row;
  ColumnID col;
  Matrix core;  // K(row.skeleton, col.skeleton)
};

// Batched column IDs on the GPU (all matrices in one launch sequence).
inline std::vector<ColumnID> column_id_batch(const std::vector<const Matrix*>& ks, double tol,
                                             std::optional<std::int64_t> max_rank = std::nullopt) {
  const std::int64_t b = static_cast<std::int64_t>(ks.size());
  std::vector<ColumnID> res(static_cast<std::size_t>(b));
  if (b == 0) return res;
  std::vector<std::int64_t> m, n, aoff, soff, ioff, mr, rank(static_cast<std::size_t>(b));
  std::vector<Complex> A;
  std::int64_t sk = 0, ip = 0;
  for (const Matrix* k : ks) {
    require(k->rows() > 0 && k->cols() > 0, "column_id: empty matrix");
    m.push_back(k->rows());
    n.push_back(k->cols());
    aoff.push_back(static_cast<std::int64_t>(A.size()));
    A.insert(A.end(), k->data(), k->data() + k->size());
    soff.push_back(sk);
    ioff.push_back(ip);
    sk += k->cols();
    ip += k->cols() * k->cols();
    mr.push_back(max_rank.value_or(-1));
  }
  std::vector<std::int64_t> skel(static_cast<std::size_t>(sk)), perm(static_cast<std::size_t>(sk));
  std::vector<Complex> interp(static_cast<std::size_t>(ip));
  std::vector<int32_t> sat(static_cast<std::size_t>(b));
  std::vector<double> imax(static_cast<std::size_t>(b));
  detail::check(oiobf_column_id_batch(b, m.data(), n.data(), aoff.data(), reinterpret_cast<const double*>(A.data()),
                                      tol, mr.data(), rank.data(), soff.data(), skel.data(), ioff.data(),
                                      reinterpret_cast<double*>(interp.data()), perm.data(), sat.data(), imax.data()));
  for (std::int64_t q = 0; q < b; ++q) {
    ColumnID& id = res[static_cast<std::size_t>(q)];
    const std::int64_t r = rank[static_cast<std::size_t>(q)], w = n[static_cast<std::size_t>(q)];
    id.rank = r;
    id.saturated = sat[static_cast<std::size_t>(q)] != 0;
    id.interp_max_abs = imax[static_cast<std::size_t>(q)];
    id.skeleton.assign(skel.begin() + soff[static_cast<std::size_t>(q)],
                       skel.begin() + soff[static_cast<std::size_t>(q)] + r);
    id.interp.resize(r, w);
    std::copy(interp.begin() + ioff[static_cast<std::size_t>(q)],
              interp.begin() + ioff[static_cast<std::size_t>(q)] + r * w, id.interp.data());
  }
  return res;
}

// Any size, like the reference (id.cpp:124-130): up to 96 columns the device
// keeps the ID's w x w triangular factor in shared memory (TSQR + reference
// pivoting on R); wider matrices run the same pivoted Householder QR in global
// memory, one CTA per matrix (slower; the butterfly's own IDs never need it).
inline ColumnID column_id(const Matrix& k, double tol, std::optional<std::int64_t> max_rank = std::nullopt) {
  return column_id_batch({&k}, tol, max_rank)[0];
}

inline RowID row_id(const Matrix& k, double tol, std::optional<std::int64_t> max_rank = std::nullopt) {
  const Matrix kt = k.transpose();
  ColumnID c = column_id(kt, tol, max_rank);
  RowID r;
  r.skeleton = std::move(c.skeleton);
  r.interp = c.interp.transpose();
  r.rank = c.rank;
  r.saturated = c.saturated;
  r.interp_max_abs = c.interp_max_abs;
  return r;
}

inline HybridID hybrid_id(const Matrix& k, double tol) {
  HybridID h;
  h.col = column_id(k, tol);
  h.row = row_id(k, tol);
  h.core.resize(h.row.rank, h.col.rank);
  for (std::int64_t i = 0; i < h.row.rank; ++i)
    for (std::int64_t j = 0; j < h.col.rank; ++j)
      h.core(i, j) = k(h.row.skeleton[static_cast<std::size_t>(i)] - 1, h.col.skeleton[static_cast<std::size_t>(j)] - 1);
  return h;
}

enum class ProxyMode { All, UniformRandom, EvenlySpaced };

struct ProxyStrategy {
  ProxyMode mode = ProxyMode::UniformRandom;
  std::int64_t q = 3;
  std::int64_t max_retries = 3;
  std::int64_t row_cap = 1 << 17;
};

inline IndexList select_proxies_count(std::int64_t extent, std::int64_t count, ProxyMode mode, std::uint64_t seed) {
  require(extent >= 1, "select_proxies: extent must be positive");
  IndexList out(static_cast<std::size_t>(extent));
  std::int64_t got = 0;
  detail::check(oiobf_select_proxies_count(extent, count, static_cast<int32_t>(mode), seed, out.data(), &got));
  out.resize(static_cast<std::size_t>(got));
  return out;
}

inline IndexList select_proxies(std::int64_t extent, std::int64_t rank_estimate, const ProxyStrategy& s,
                                std::uint64_t seed) {
  const std::int64_t count =
      s.mode == ProxyMode::All ? extent : std::min(extent, s.q * std::max<std::int64_t>(rank_estimate, 1));
  return select_proxies_count(extent, count, s.mode, seed);
}

namespace detail {
// proxy row lists of one unfolding (reference id.cpp:199-231 rules)
inline std::vector<IndexList> proxy_lists(const std::vector<IndexRange>& ranges, std::size_t skip,
                                          std::int64_t per_mode, const ProxyStrategy& s, std::uint64_t seed) {
  std::vector<std::int64_t> cnt(ranges.size(), 0);
  for (std::size_t p = 0; p < ranges.size(); ++p)
    if (p != skip) cnt[p] = s.mode == ProxyMode::All ? ranges[p].size() : std::min(ranges[p].size(), per_mode);
  for (;;) {
    std::int64_t rows = 1;
    for (std::size_t p = 0; p < ranges.size(); ++p)
      if (p != skip) rows *= cnt[p];
    if (rows <= s.row_cap) break;
    std::size_t big = skip == 0 ? 1 : 0;
    for (std::size_t p = 0; p < ranges.size(); ++p)
      if (p != skip && cnt[p] > cnt[big]) big = p;
    if (cnt[big] <= 2) break;
    cnt[big] = (cnt[big] + 1) / 2;
  }
  std::vector<IndexList> lists(ranges.size());
  for (std::size_t p = 0; p < ranges.size(); ++p) {
    if (p == skip) continue;
    IndexList l = select_proxies_count(ranges[p].size(), cnt[p], s.mode,
                                       derive_seed(seed, {0x70ULL, static_cast<std::uint64_t>(p)}));
    for (auto& v : l) v += ranges[p].lo - 1;
    lists[p] = std::move(l);
  }
  return lists;
}
}  // namespace detail

struct TuckerID {
  std::int64_t d = 0;
  std::vector<IndexList> row_skeletons;
  std::vector<IndexList> col_skeletons;
  std::vector<Matrix> row_interp;  // U^k: r_k x |tau_k|
  std::vector<Matrix> col_interp;  // V^k: r_k x |nu_k|
  DenseTensor core;
  std::vector<std::int64_t> ranks;  // row modes then col modes
  bool saturated = false;

  std::int64_t memory_bytes() const {
    std::int64_t s = core.size();
    for (const auto& m : row_interp) s += m.size();
    for (const auto& m : col_interp) s += m.size();
    return s * static_cast<std::int64_t>(sizeof(Complex));
  }
};

// reference id.cpp:235-287: per mode, proxy rows + full target range, GPU entry
// generation, unfolding, GPU column ID; core at the skeleton multi-sets.
inline TuckerID tucker_id(const KernelEvaluator& k, const MultiSet& rows, const MultiSet& cols, double tol,
                          const ProxyStrategy& proxies, std::uint64_t seed) {
  const std::size_t d = static_cast<std::size_t>(k.d);
  require(rows.size() == d && cols.size() == d, "tucker_id: wrong mode count");
  std::vector<IndexRange> ranges(rows.begin(), rows.end());
  ranges.insert(ranges.end(), cols.begin(), cols.end());
  TuckerID out;
  out.d = k.d;
  out.row_skeletons.resize(d);
  out.col_skeletons.resize(d);
  out.row_interp.resize(d);
  out.col_interp.resize(d);
  out.ranks.assign(2 * d, 0);
  std::int64_t r_est = 8;
  for (std::size_t mode = 0; mode < 2 * d; ++mode) {
    const IndexRange target = ranges[mode];
    ColumnID id;
    for (std::int64_t attempt = 0;; ++attempt) {
      const std::int64_t per_mode = proxies.q * r_est * (std::int64_t{1} << attempt);
      const std::uint64_t s = derive_seed(seed, {0x1DULL, static_cast<std::uint64_t>(mode),
                                                 static_cast<std::uint64_t>(attempt)});
      auto lists = detail::proxy_lists(ranges, mode, per_mode, proxies, s);
      lists[mode] = range_to_list(target);
      std::vector<IndexList> rl(lists.begin(), lists.begin() + static_cast<std::ptrdiff_t>(d));
      std::vector<IndexList> cl(lists.begin() + static_cast<std::ptrdiff_t>(d), lists.end());
      const Matrix unf = unfold(subtensor_at(k, rl, cl), static_cast<std::int64_t>(mode) + 1).m;
      id = column_id(unf, tol);
      if (!id.saturated || attempt >= proxies.max_retries) break;
    }
    out.saturated = out.saturated || id.saturated;
    out.ranks[mode] = id.rank;
    r_est = std::max(r_est, id.rank);
    IndexList global = id.skeleton;
    for (auto& v : global) v += target.lo - 1;
    if (mode < d) {
      out.row_skeletons[mode] = std::move(global);
      out.row_interp[mode] = std::move(id.interp);
    } else {
      out.col_skeletons[mode - d] = std::move(global);
      out.col_interp[mode - d] = std::move(id.interp);
    }
  }
  out.core = subtensor_at(k, out.row_skeletons, out.col_skeletons);
  return out;
}

inline DenseTensor tucker_reconstruct(const TuckerID& t) {
  DenseTensor acc = t.core;
  for (std::int64_t k = 0; k < t.d; ++k)
    acc = mode_product(acc, k + 1, t.row_interp[static_cast<std::size_t>(k)].transpose());
  for (std::int64_t k = 0; k < t.d; ++k)
    acc = mode_product(acc, t.d + k + 1, t.col_interp[static_cast<std::size_t>(k)].transpose());
  return acc;
}

// G = K x_{d+1..2d} F through the Tucker-ID factors (reference id.cpp:305-329),
// every contraction on the GPU (the core GEMM is a mode-1 product).
inline DenseTensor tucker_contract(const TuckerID& t, const DenseTensor& f) {
  require(f.mode_count() == t.d + 1, "tucker_contract: input must have d+1 modes");
  DenseTensor g = f;
  for (std::int64_t k = 0; k < t.d; ++k) g = mode_product(g, k + 1, t.col_interp[static_cast<std::size_t>(k)]);
  std::vector<std::int64_t> core_rows(t.core.shape().begin(), t.core.shape().begin() + t.d);
  std::vector<std::int64_t> core_cols(t.core.shape().begin() + t.d, t.core.shape().end());
  std::vector<std::int64_t> rm(static_cast<std::size_t>(t.d)), cm(static_cast<std::size_t>(t.d));
  std::iota(rm.begin(), rm.end(), 1);
  std::iota(cm.begin(), cm.end(), t.d + 1);
  const Matrix core_mat = matricize(t.core, rm, cm);
  const std::int64_t nv = f.extent(t.d + 1);
  std::vector<std::int64_t> gshape{detail::prod(core_cols), nv};
  DenseTensor gm(gshape, g.data());  // (prod r_s) x nv, first-fastest == matricize(g, 1..d | d+1)
  DenseTensor prod = mode_product(gm, 1, core_mat);  // (prod r_t) x nv
  std::vector<std::int64_t> oshape = core_rows;
  oshape.push_back(nv);
  DenseTensor out(oshape, prod.data());
  for (std::int64_t k = 0; k < t.d; ++k)
    out = mode_product(out, k + 1, t.row_interp[static_cast<std::size_t>(k)].transpose());
  return out;
}

}  // namespace oiobf

#endif
