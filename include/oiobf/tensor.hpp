// oiobf drop-in: tensor core (reference proj/include/oiobf/tensor.hpp:8-101).
//
// Data movement (flatten, unfold, refold, matricize) is host code; every
// arithmetic operation on the hot path runs on the B200 through the C ABI:
//   mode_product / mode_product_blockdiag  -> oiobf_mode_product_blockdiag
//   subtensor / subtensor_at               -> oiobf_subtensor_at (entry generation)
// KernelEvaluator keeps the reference's std::function layout; the device path
// recovers the POD spec with eval.target<KernelFunctor>().  An
// opaque closure cannot run on the GPU and is rejected (no CPU fallback).
#ifndef OIOBF_DROPIN_TENSOR_HPP
#define OIOBF_DROPIN_TENSOR_HPP

#include <cmath>
#include <functional>
#include <string>

#include "oiobf/types.hpp"
#include "oiobf_b200.h"

namespace oiobf {

namespace detail {
inline void check(int rc) {
  if (rc == OIOBF_OK) return;
  const std::string msg = oiobf_last_error();
  if (rc == OIOBF_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
inline std::int64_t prod(const std::vector<std::int64_t>& v) {
  std::int64_t p = 1;
  for (auto e : v) p *= e;
  return p;
}
}  // namespace detail

// First-mode-fastest dense complex tensor (tensor.hpp:10-45).
class DenseTensor {
 public:
  DenseTensor() = default;
  explicit DenseTensor(std::vector<std::int64_t> shape) : shape_(std::move(shape)) {
    for (auto e : shape_) require(e >= 0, "DenseTensor: negative extent");
    data_.assign(static_cast<std::size_t>(detail::prod(shape_)), Complex(0, 0));
  }
  DenseTensor(std::vector<std::int64_t> shape, std::vector<Complex> data)
      : shape_(std::move(shape)), data_(std::move(data)) {
    require(static_cast<std::int64_t>(data_.size()) == detail::prod(shape_),
            "DenseTensor: data length does not match shape");
  }
  std::int64_t mode_count() const { return static_cast<std::int64_t>(shape_.size()); }
  const std::vector<std::int64_t>& shape() const { return shape_; }
  std::int64_t extent(std::int64_t mode1b) const { return shape_.at(static_cast<std::size_t>(mode1b - 1)); }
  std::int64_t size() const { return static_cast<std::int64_t>(data_.size()); }
  const std::vector<Complex>& data() const { return data_; }
  std::vector<Complex>& data() { return data_; }

  std::int64_t flatten(const MultiIndex& idx) const {
    require(idx.size() == shape_.size(), "flatten: wrong index length");
    std::int64_t off = 0, stride = 1;
    for (std::size_t k = 0; k < shape_.size(); ++k) {
      require(idx[k] >= 1 && idx[k] <= shape_[k], "flatten: index out of range");
      off += (idx[k] - 1) * stride;
      stride *= shape_[k];
    }
    return off;
  }
  MultiIndex unflatten(std::int64_t flat) const {
    MultiIndex idx(shape_.size());
    for (std::size_t k = 0; k < shape_.size(); ++k) {
      idx[k] = flat % shape_[k] + 1;
      flat /= shape_[k];
    }
    return idx;
  }
  Complex at(const MultiIndex& idx) const { return data_[static_cast<std::size_t>(flatten(idx))]; }
  Complex& at(const MultiIndex& idx) { return data_[static_cast<std::size_t>(flatten(idx))]; }
  double frobenius_norm() const {
    double s = 0;
    for (const Complex& z : data_) s += std::norm(z);
    return std::sqrt(s);
  }
  DenseTensor slice(const MultiSet& ranges) const {
    require(static_cast<std::int64_t>(ranges.size()) == mode_count(), "slice: wrong range count");
    std::vector<std::int64_t> oshape;
    for (std::size_t k = 0; k < ranges.size(); ++k) {
      require(ranges[k].lo >= 1 && ranges[k].hi <= shape_[k] && ranges[k].size() >= 0, "slice: range out of bounds");
      oshape.push_back(ranges[k].size());
    }
    DenseTensor out(oshape);
    MultiIndex src(ranges.size());
    for (std::int64_t f = 0; f < out.size(); ++f) {
      const MultiIndex loc = out.unflatten(f);
      for (std::size_t k = 0; k < ranges.size(); ++k) src[k] = ranges[k].lo + loc[k] - 1;
      out.data_[static_cast<std::size_t>(f)] = data_[static_cast<std::size_t>(flatten(src))];
    }
    return out;
  }

 private:
  std::vector<std::int64_t> shape_;
  std::vector<Complex> data_;
};

struct Unfolding {
  std::vector<std::int64_t> source_shape;
  std::int64_t mode = 1;  // 1-based
  Matrix m;
};

// Mode-j unfolding: row = complement multi-index (first listed fastest), column = i_j.
inline Unfolding unfold(const DenseTensor& t, std::int64_t mode) {
  require(mode >= 1 && mode <= t.mode_count(), "unfold: mode out of range");
  const auto& sh = t.shape();
  std::int64_t below = 1;
  for (std::int64_t k = 0; k < mode - 1; ++k) below *= sh[static_cast<std::size_t>(k)];
  const std::int64_t nj = sh[static_cast<std::size_t>(mode - 1)];
  const std::int64_t rows = nj == 0 ? 0 : t.size() / nj;
  Unfolding u;
  u.source_shape = sh;
  u.mode = mode;
  u.m.resize(rows, nj);
  for (std::int64_t f = 0; f < t.size(); ++f) {
    const std::int64_t col = (f / below) % nj;
    const std::int64_t row = f % below + (f / (below * nj)) * below;
    u.m(row, col) = t.data()[static_cast<std::size_t>(f)];
  }
  return u;
}

inline DenseTensor refold(const Unfolding& u) {
  DenseTensor t(u.source_shape);
  std::int64_t below = 1;
  for (std::int64_t k = 0; k < u.mode - 1; ++k) below *= u.source_shape[static_cast<std::size_t>(k)];
  const std::int64_t nj = u.source_shape[static_cast<std::size_t>(u.mode - 1)];
  for (std::int64_t f = 0; f < t.size(); ++f)
    t.data()[static_cast<std::size_t>(f)] = u.m(f % below + (f / (below * nj)) * below, (f / below) % nj);
  return t;
}

// Y = T x_j blockdiag(B_i) on the GPU; transpose_blocks uses B_i instead of B_i^T.
inline DenseTensor mode_product_blockdiag(const DenseTensor& t, std::int64_t mode,
                                          const std::vector<const Matrix*>& blocks, bool transpose_blocks = false) {
  require(mode >= 1 && mode <= t.mode_count(), "mode_product_blockdiag: mode out of range");
  require(!blocks.empty(), "mode_product_blockdiag: no blocks");
  std::vector<std::int64_t> br, bc;
  std::vector<Complex> packed;
  std::int64_t out_total = 0;
  for (const Matrix* b : blocks) {
    br.push_back(b->rows());
    bc.push_back(b->cols());
    out_total += transpose_blocks ? b->cols() : b->rows();
    packed.insert(packed.end(), b->data(), b->data() + b->size());
  }
  std::vector<std::int64_t> oshape = t.shape();
  oshape[static_cast<std::size_t>(mode - 1)] = out_total;
  DenseTensor out(oshape);
  if (packed.empty()) packed.push_back(Complex(0, 0));
  detail::check(oiobf_mode_product_blockdiag(static_cast<int32_t>(t.mode_count()), t.shape().data(),
                                             reinterpret_cast<const double*>(t.data().data()), static_cast<int32_t>(mode),
                                             static_cast<int32_t>(blocks.size()), br.data(), bc.data(),
                                             reinterpret_cast<const double*>(packed.data()),
                                             transpose_blocks ? 1 : 0, reinterpret_cast<double*>(out.data().data())));
  return out;
}

// Y = T x_j X, X (r x n_j): Y^(j) = T^(j) X^T.
inline DenseTensor mode_product(const DenseTensor& t, std::int64_t mode, const Matrix& x) {
  require(mode >= 1 && mode <= t.mode_count(), "mode_product: mode out of range");
  require(x.cols() == t.extent(mode), "mode_product: shape mismatch");
  return mode_product_blockdiag(t, mode, {&x}, false);
}

inline Matrix matricize(const DenseTensor& t, const std::vector<std::int64_t>& row_modes,
                        const std::vector<std::int64_t>& col_modes) {
  const std::int64_t d = t.mode_count();
  std::vector<bool> seen(static_cast<std::size_t>(d), false);
  for (auto m : row_modes) {
    require(m >= 1 && m <= d && !seen[static_cast<std::size_t>(m - 1)], "matricize: bad row modes");
    seen[static_cast<std::size_t>(m - 1)] = true;
  }
  for (auto m : col_modes) {
    require(m >= 1 && m <= d && !seen[static_cast<std::size_t>(m - 1)], "matricize: bad col modes");
    seen[static_cast<std::size_t>(m - 1)] = true;
  }
  for (bool s : seen) require(s, "matricize: modes must cover all modes");
  std::int64_t rows = 1, cols = 1;
  for (auto m : row_modes) rows *= t.extent(m);
  for (auto m : col_modes) cols *= t.extent(m);
  Matrix out(rows, cols);
  for (std::int64_t f = 0; f < t.size(); ++f) {
    const MultiIndex idx = t.unflatten(f);
    std::int64_t r = 0, c = 0, rs = 1, csd = 1;
    for (auto m : row_modes) {
      r += (idx[static_cast<std::size_t>(m - 1)] - 1) * rs;
      rs *= t.extent(m);
    }
    for (auto m : col_modes) {
      c += (idx[static_cast<std::size_t>(m - 1)] - 1) * csd;
      csd *= t.extent(m);
    }
    out(r, c) = t.data()[static_cast<std::size_t>(f)];
  }
  return out;
}

inline DenseTensor fold_matricization(const Matrix& m, const std::vector<std::int64_t>& row_shape,
                                      const std::vector<std::int64_t>& col_shape) {
  std::vector<std::int64_t> shape = row_shape;
  shape.insert(shape.end(), col_shape.begin(), col_shape.end());
  const std::int64_t rows = detail::prod(row_shape), cols = detail::prod(col_shape);
  require(m.rows() == rows && m.cols() == cols, "fold_matricization: shape mismatch");
  // both sides first-fastest: the flat layout is the column-major matrix
  return DenseTensor(shape, std::vector<Complex>(m.data(), m.data() + m.size()));
}

// Device-evaluable entry function: the POD spec of the BASELINE catalog.
// Scalar calls are evaluated on the GPU as well (1 x ... x 1 subtensor).
struct KernelFunctor {
  oiobf_kernel_spec spec{};
  Complex operator()(const MultiIndex& i, const MultiIndex& j) const {
    const std::size_t d = static_cast<std::size_t>(spec.d);
    require(i.size() == d && j.size() == d, "kernel: wrong multi-index length");
    std::vector<std::int64_t> counts(2 * d, 1), lists(i);
    lists.insert(lists.end(), j.begin(), j.end());
    Complex v;
    detail::check(oiobf_subtensor_at(&spec, counts.data(), lists.data(), reinterpret_cast<double*>(&v)));
    return v;
  }
};

struct KernelEvaluator {
  std::int64_t d = 0;
  std::vector<std::int64_t> row_extents;
  std::vector<std::int64_t> col_extents;
  std::function<Complex(const MultiIndex&, const MultiIndex&)> eval;

  Complex operator()(const MultiIndex& i, const MultiIndex& j) const { return eval(i, j); }
  MultiSet full_rows() const {
    MultiSet ms;
    for (auto e : row_extents) ms.push_back({1, e});
    return ms;
  }
  MultiSet full_cols() const {
    MultiSet ms;
    for (auto e : col_extents) ms.push_back({1, e});
    return ms;
  }
  // the device spec behind eval; throws for opaque closures (no CPU fallback)
  const oiobf_kernel_spec& device_spec() const {
    const KernelFunctor* f = eval.target<KernelFunctor>();
    require(f != nullptr,
            "KernelEvaluator: opaque std::function cannot run on the B200 path; build it with make_kernel()");
    return f->spec;
  }
};

inline DenseTensor subtensor_at(const KernelEvaluator& k, const std::vector<IndexList>& rows,
                                const std::vector<IndexList>& cols) {
  const std::size_t d = static_cast<std::size_t>(k.d);
  require(rows.size() == d && cols.size() == d, "subtensor_at: wrong mode count");
  std::vector<std::int64_t> shape, lists;
  for (const auto& l : rows) {
    shape.push_back(static_cast<std::int64_t>(l.size()));
    lists.insert(lists.end(), l.begin(), l.end());
  }
  for (const auto& l : cols) {
    shape.push_back(static_cast<std::int64_t>(l.size()));
    lists.insert(lists.end(), l.begin(), l.end());
  }
  DenseTensor t(shape);
  if (t.size() == 0) return t;
  detail::check(oiobf_subtensor_at(&k.device_spec(), shape.data(), lists.data(),
                                   reinterpret_cast<double*>(t.data().data())));
  return t;
}

inline DenseTensor subtensor(const KernelEvaluator& k, const MultiSet& rows, const MultiSet& cols) {
  require(static_cast<std::int64_t>(rows.size()) == k.d && static_cast<std::int64_t>(cols.size()) == k.d,
          "subtensor: wrong mode count");
  std::vector<IndexList> rl, cl;
  for (std::size_t p = 0; p < rows.size(); ++p) {
    require(rows[p].lo >= 1 && rows[p].hi <= k.row_extents[p], "subtensor: row range out of bounds");
    rl.push_back(range_to_list(rows[p]));
  }
  for (std::size_t p = 0; p < cols.size(); ++p) {
    require(cols[p].lo >= 1 && cols[p].hi <= k.col_extents[p], "subtensor: col range out of bounds");
    cl.push_back(range_to_list(cols[p]));
  }
  return subtensor_at(k, rl, cl);
}

}  // namespace oiobf

#endif
