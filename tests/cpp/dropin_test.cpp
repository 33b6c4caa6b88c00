// Drop-in check: reference-style C++ call sites against the B200 library.
// Prints one JSON object; tests/test_dropin_cpp.py compares it with the
// reference harness / oracle.
#include <cstdio>
#include <iostream>
#include <random>
#include <sstream>

#include "oiobf/butterfly.hpp"
#include "oiobf/id.hpp"
#include "oiobf/kernels.hpp"
#include "oiobf/tensor.hpp"

using namespace oiobf;

static std::string list_json(const IndexList& l) {
  std::ostringstream o;
  o << "[";
  for (std::size_t i = 0; i < l.size(); ++i) o << (i ? "," : "") << l[i];
  o << "]";
  return o.str();
}

int main(int argc, char** argv) {
  const bool compile_only = argc > 1 && std::string(argv[1]) == "--compile-only";
  if (compile_only) return 0;
  std::ostringstream js;
  js << "{";
  // 1. column_id on an exactly rank-5 matrix
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  Matrix A(60, 12), B(60, 5), C(5, 12);
  for (int i = 0; i < 60; ++i)
    for (int j = 0; j < 5; ++j) B(i, j) = Complex(nd(rng), nd(rng));
  for (int i = 0; i < 5; ++i)
    for (int j = 0; j < 12; ++j) C(i, j) = Complex(nd(rng), nd(rng));
  A = B * C;
  ColumnID id = column_id(A, 1e-10);
  js << "\"cid_rank\":" << id.rank << ",\"cid_skel\":" << list_json(id.skeleton) << ",";
  // identity sub-block
  bool ident = true;
  for (std::int64_t i = 0; i < id.rank; ++i)
    for (std::int64_t k = 0; k < id.rank; ++k) {
      const Complex v = id.interp(i, id.skeleton[static_cast<std::size_t>(k)] - 1);
      if (std::abs(v - Complex(i == k ? 1.0 : 0.0, 0)) > 0) ident = false;
    }
  js << "\"cid_identity\":" << (ident ? "true" : "false") << ",";
  // 2. tucker_id on the plates kernel (reference id.cpp:235 semantics)
  KernelEvaluator k = make_kernel(green_plates(16));
  MultiSet rows = k.full_rows(), cols = k.full_cols();
  TuckerID t = tucker_id(k, rows, cols, 1e-6, ProxyStrategy{}, 11);
  js << "\"tucker_ranks\":" << list_json(IndexList(t.ranks.begin(), t.ranks.end())) << ",\"tucker_skel\":[";
  for (int m = 0; m < 4; ++m)
    js << (m ? "," : "") << list_json(m < 2 ? t.row_skeletons[static_cast<std::size_t>(m)]
                                            : t.col_skeletons[static_cast<std::size_t>(m - 2)]);
  js << "],\"tucker_mem\":" << t.memory_bytes() << ",";
  // tucker_contract vs dense product
  DenseTensor F({16, 16, 1});
  for (auto& z : F.data()) z = Complex(nd(rng), nd(rng));
  DenseTensor G = tucker_contract(t, F);
  Matrix K = dense_oracle(k);
  double num = 0, den = 0;
  for (int i = 0; i < 256; ++i) {
    Complex s(0, 0);
    for (int j = 0; j < 256; ++j) s += K(i, j) * F.data()[static_cast<std::size_t>(j)];
    num += std::norm(G.data()[static_cast<std::size_t>(i)] - s);
    den += std::norm(s);
  }
  js << "\"tucker_contract_err\":" << std::sqrt(num / den) << ",";
  // 3. tensor butterfly construct + contract vs the dense product
  KernelEvaluator k2 = make_kernel(green_plates(32));
  TensorButterfly bf = tbf_construct(k2, 2, 1e-6, ProxyStrategy{}, 3);
  DenseTensor F2({32, 32});
  for (auto& z : F2.data()) z = Complex(nd(rng), nd(rng));
  DenseTensor G2 = tbf_contract(bf, F2);
  Matrix K2 = dense_oracle(k2);
  num = den = 0;
  for (int i = 0; i < 1024; ++i) {
    Complex s(0, 0);
    for (int j = 0; j < 1024; ++j) s += K2(i, j) * F2.data()[static_cast<std::size_t>(j)];
    num += std::norm(G2.data()[static_cast<std::size_t>(i)] - s);
    den += std::norm(s);
  }
  const TbfMemory mem = tbf_memory(bf);
  js << "\"tbf_err\":" << std::sqrt(num / den) << ",\"tbf_mem\":" << mem.total() << ",";
  js << "\"tbf_err_estimate\":" << tbf_error_estimate(bf, k2, 5, 9) << ",";
  // 4. an opaque closure must be rejected (no CPU fallback)
  KernelEvaluator opaque = k2;
  opaque.eval = [](const MultiIndex&, const MultiIndex&) { return Complex(1, 0); };
  bool rejected = false;
  try {
    (void)subtensor(opaque, opaque.full_rows(), opaque.full_cols());
  } catch (const std::invalid_argument&) {
    rejected = true;
  }
  js << "\"opaque_rejected\":" << (rejected ? "true" : "false") << ",";
  // 5. argument errors map to std::invalid_argument
  bool bad_tol = false;
  try {
    column_id(A, 0.0);
  } catch (const std::invalid_argument&) {
    bad_tol = true;
  }
  js << "\"bad_tol_rejected\":" << (bad_tol ? "true" : "false") << ",";
  // 5b. IDs wider than the shared-memory kernels hold (150 > 96 columns / rows):
  // column_id, row_id and hybrid_id of a rank-30 matrix reconstruct it
  {
    Matrix Bw(140, 30), Cw(30, 150);
    for (int i = 0; i < 140; ++i)
      for (int j = 0; j < 30; ++j) Bw(i, j) = Complex(nd(rng), nd(rng));
    for (int i = 0; i < 30; ++i)
      for (int j = 0; j < 150; ++j) Cw(i, j) = Complex(nd(rng), nd(rng));
    const Matrix Aw = Bw * Cw;
    double an = 0;
    for (int i = 0; i < 140; ++i)
      for (int j = 0; j < 150; ++j) an += std::norm(Aw(i, j));
    const ColumnID cw = column_id(Aw, 1e-9);
    double ce = 0;  // || A(:, J) X - A ||
    for (int i = 0; i < 140; ++i)
      for (int j = 0; j < 150; ++j) {
        Complex acc(0, 0);
        for (std::int64_t q = 0; q < cw.rank; ++q) acc += Aw(i, cw.skeleton[static_cast<std::size_t>(q)] - 1) * cw.interp(q, j);
        ce += std::norm(acc - Aw(i, j));
      }
    const RowID rw = row_id(Aw, 1e-9);
    double re = 0;  // || X A(I, :) - A ||
    for (int i = 0; i < 140; ++i)
      for (int j = 0; j < 150; ++j) {
        Complex acc(0, 0);
        for (std::int64_t q = 0; q < rw.rank; ++q) acc += rw.interp(i, q) * Aw(rw.skeleton[static_cast<std::size_t>(q)] - 1, j);
        re += std::norm(acc - Aw(i, j));
      }
    js << "\"wide_cid_rank\":" << cw.rank << ",\"wide_cid_err\":" << std::sqrt(ce / an) << ",\"wide_rid_rank\":" << rw.rank
       << ",\"wide_rid_err\":" << std::sqrt(re / an) << ",";
  }
  // 6. scalar evaluation through the functor (GPU) == batched entry
  const Complex e1 = k2(MultiIndex{3, 4}, MultiIndex{5, 6});
  const DenseTensor e2 = subtensor_at(k2, {{3}, {4}}, {{5}, {6}});
  js << "\"scalar_matches\":" << (e1 == e2.data()[0] ? "true" : "false");
  js << "}";
  std::cout << js.str() << std::endl;
  return 0;
}
