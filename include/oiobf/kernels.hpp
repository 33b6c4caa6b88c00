// oiobf drop-in: kernel catalog (BASELINE.json configs).
//
// make_kernel() returns a reference-layout KernelEvaluator whose std::function
// holds a KernelFunctor (POD device spec), so every evaluation -- scalar or
// batched -- runs on the B200.
#ifndef OIOBF_DROPIN_KERNELS_HPP
#define OIOBF_DROPIN_KERNELS_HPP

#include <cmath>

#include "oiobf/tensor.hpp"

namespace oiobf {

enum class KernelKind {
  Green = OIOBF_KERNEL_GREEN,
  DFT = OIOBF_KERNEL_DFT,
  Radon2D = OIOBF_KERNEL_RADON2D,
  Radon3D = OIOBF_KERNEL_RADON3D,
  NUDFT = OIOBF_KERNEL_NUDFT
};

struct KernelSpec {
  KernelKind kind = KernelKind::Green;
  std::int64_t d = 2;
  std::int64_t n = 0;
  double kappa = 0;                     // Green wavenumber
  double offset[3] = {0, 0, 0};         // Green source offset
  bool bitrev = false;                  // DFT: two-sided per-mode bit reversal
  std::uint32_t seed = 0;               // NUDFT: seed of the random target locations
};

inline KernelEvaluator make_kernel(const KernelSpec& s) {
  require(s.d >= 1 && s.d <= 6, "make_kernel: d must be in [1, 6]");
  require(s.n >= 1, "make_kernel: n must be positive");
  require(s.kind != KernelKind::Radon2D || s.d == 2, "make_kernel: radon2d needs d = 2");
  require(s.kind != KernelKind::Radon3D || s.d == 3, "make_kernel: radon3d needs d = 3");
  require(s.kind != KernelKind::NUDFT || !s.bitrev, "make_kernel: nudft has no bit-reversed ordering");
  require(s.kind != KernelKind::Green || s.d <= 3, "make_kernel: green needs d <= 3");
  KernelFunctor f;
  f.spec.kind = static_cast<int32_t>(s.kind);
  f.spec.d = static_cast<int32_t>(s.d);
  f.spec.n = s.n;
  f.spec.bitrev = s.bitrev ? 1 : 0;
  f.spec.seed = s.seed;
  f.spec.kappa = s.kappa;
  for (int p = 0; p < 3; ++p) f.spec.offset[p] = s.offset[p];
  KernelEvaluator k;
  k.d = s.d;
  k.row_extents.assign(static_cast<std::size_t>(s.d), s.n);
  k.col_extents.assign(static_cast<std::size_t>(s.d), s.n);
  k.eval = f;
  return k;
}

// BASELINE.json configs (points per wavelength 8)
inline KernelSpec green_plates(std::int64_t n, double ppw = 8) {
  KernelSpec s;
  s.kind = KernelKind::Green;
  s.d = 2;
  s.n = n;
  s.kappa = 2 * M_PI * static_cast<double>(n) / ppw;
  s.offset[2] = 1;
  return s;
}
inline KernelSpec green_cubes(std::int64_t n, double ppw = 8) {
  KernelSpec s = green_plates(n, ppw);
  s.d = 3;
  s.offset[0] = 2;
  s.offset[2] = 0;
  return s;
}
inline KernelSpec dft(std::int64_t d, std::int64_t n, bool bitrev = true) {
  KernelSpec s;
  s.kind = KernelKind::DFT;
  s.d = d;
  s.n = n;
  s.bitrev = bitrev;
  return s;
}
inline KernelSpec radon2d(std::int64_t n) {
  KernelSpec s;
  s.kind = KernelKind::Radon2D;
  s.d = 2;
  s.n = n;
  return s;
}
// Phi = x.k + c|k|, c = (3 + sin 2 pi x1 sin 2 pi x2 sin 2 pi x3) / 100
inline KernelSpec radon3d(std::int64_t n) {
  KernelSpec s;
  s.kind = KernelKind::Radon3D;
  s.d = 3;
  s.n = n;
  return s;
}
// PAPER.md:707 type-2 NUDFT: seeded random target locations in [0, n-1]^d
inline KernelSpec nudft(std::int64_t d, std::int64_t n, std::uint32_t seed = 1) {
  KernelSpec s;
  s.kind = KernelKind::NUDFT;
  s.d = d;
  s.n = n;
  s.seed = seed;
  return s;
}

// Per-mode bit-reversed index maps on both sides; involution.
inline KernelEvaluator reorder_bit_reversal(const KernelEvaluator& k) {
  oiobf_kernel_spec sp = k.device_spec();
  require((sp.n & (sp.n - 1)) == 0, "reorder_bit_reversal: extent must be a power of two");
  KernelFunctor f;
  f.spec = sp;
  f.spec.bitrev = sp.bitrev ? 0 : 1;
  KernelEvaluator out = k;
  out.eval = f;
  return out;
}

// Fully materialised matricization (rows = modes 1..d) for desk-scale checks,
// generated on the GPU; refused above `cap` entries.
inline Matrix dense_oracle(const KernelEvaluator& k, std::int64_t cap = std::int64_t{1} << 26) {
  std::int64_t rows = 1, cols = 1;
  for (auto e : k.row_extents) rows *= e;
  for (auto e : k.col_extents) cols *= e;
  require(rows * cols <= cap, "dense_oracle: entry count exceeds the cap");
  const DenseTensor t = subtensor(k, k.full_rows(), k.full_cols());
  Matrix m(rows, cols);
  std::copy(t.data().begin(), t.data().end(), m.data());  // first-fastest == column-major matricization
  return m;
}

}  // namespace oiobf

#endif
