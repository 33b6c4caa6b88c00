// In-process multi-device butterfly (include/oiobf/sharded.hpp) against the
// single-GPU butterfly of the same operator: usage
//   sharded_test WORLD [case] [balanced]   (every rank on device 0 -- a one-GPU box)
// balanced: tbf_construct_sharded_balanced (byte-balanced ownership map)
// case: cubes32 (d = 3, L = 2), radon64 (d = 2, L = 2), plates64L4 (d = 2,
// L = 4), dft6 (d = 6, n = 4, C_b = 1, L = 2, all ranks 1).  Prints one JSON line.
#include <cmath>
#include <iostream>
#include <random>
#include <string>

#include "oiobf/butterfly.hpp"
#include "oiobf/kernels.hpp"
#include "oiobf/sharded.hpp"

using namespace oiobf;

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "--compile-only") return 0;
  if (argc > 3 && std::string(argv[1]) == "--owners") {  // balanced_owners(weights, world): host logic only
    const std::int64_t world = std::atoll(argv[2]);
    std::vector<double> w;
    for (int i = 3; i < argc; ++i) w.push_back(std::atof(argv[i]));
    const std::vector<std::int32_t> own = balanced_owners(w, world);
    std::cout << "[";
    for (std::size_t i = 0; i < own.size(); ++i) std::cout << (i ? "," : "") << own[i];
    std::cout << "]" << std::endl;
    return 0;
  }
  const int world = argc > 1 ? std::atoi(argv[1]) : 2;
  const std::string which = argc > 2 ? argv[2] : "cubes32";
  KernelSpec s;
  std::int64_t L = 2;
  double tol = 1e-6;
  if (which == "cubes32") s = green_cubes(32);
  else if (which == "radon64") s = radon2d(64);
  else if (which == "plates64L4") {
    s = green_plates(64);
    L = 4;
    tol = 1e-4;
  } else if (which == "dft6") {
    s = dft(6, 4);
    L = 2;
    tol = 1e-8;
  } else {
    std::cerr << "unknown case " << which << "\n";
    return 2;
  }
  const KernelEvaluator k = make_kernel(s);
  const TensorButterfly single = tbf_construct(k, L, tol, ProxyStrategy{}, 5);
  const bool balanced = argc > 3 && std::string(argv[3]) == "balanced";
  const ShardedTensorButterfly sh =
      balanced ? tbf_construct_sharded_balanced(k, L, tol, ProxyStrategy{}, 5, std::vector<int>(world, 0))
               : tbf_construct_sharded(k, L, tol, ProxyStrategy{}, 5, std::vector<int>(world, 0));
  // heaviest rank's core bytes over the mean (phase-1 imbalance)
  const std::vector<double> w = sh.core_bytes_per_s();
  std::vector<double> load(static_cast<std::size_t>(world), 0.0);
  double tot = 0;
  for (std::size_t i = 0; i < w.size(); ++i) {
    load[static_cast<std::size_t>(sh.owner_of(static_cast<std::int64_t>(i)))] += w[i];
    tot += w[i];
  }
  const double imb = *std::max_element(load.begin(), load.end()) / (tot / world);
  std::vector<std::int64_t> shape(k.col_extents.begin(), k.col_extents.end());
  shape.push_back(2);  // n_v = 2
  DenseTensor F(shape);
  std::mt19937_64 rng(3);
  std::normal_distribution<double> nd;
  for (auto& z : F.data()) z = Complex(nd(rng), nd(rng));
  const DenseTensor G1 = tbf_contract(single, F);
  const DenseTensor G = tbf_contract(sh, F);
  double num = 0, den = 0;
  for (std::size_t i = 0; i < G.data().size(); ++i) {
    num += std::norm(G.data()[i] - G1.data()[i]);
    den += std::norm(G1.data()[i]);
  }
  std::int64_t sent = 0;
  for (int r = 0; r < world; ++r) sent += sh.layout(static_cast<std::size_t>(r)).send_total();
  std::cout << "{\"case\":\"" << which << "\",\"world\":" << world << ",\"nmid\":" << sh.nmid()
            << ",\"rel\":" << std::sqrt(num / den) << ",\"exchanged_elems\":" << sent
            << ",\"mapped\":" << (sh.owners().empty() ? 0 : 1) << ",\"core_max_over_mean\":" << imb << "}" << std::endl;
  return 0;
}
