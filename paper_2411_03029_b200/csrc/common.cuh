// Shared device-side definitions for the B200 tensor-butterfly path.
//
// * complex128 = double2 (interleaved re/im, zero-copy with std::complex<double>)
// * splitmix64 / derive_seed / proxy selection: bit-exact with the reference
//   (rng.hpp:12-47, id.cpp:155-231), evaluated on the device so construction
//   never round-trips proxy sets through the host.
// * kernel entry functors for the BASELINE catalog (green / dft / radon2d).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/oiobf_b200.h"

namespace tbf {

using i64 = long long;
using u64 = unsigned long long;

#define TBF_CUDA(x)                                                                                       \
  do {                                                                                                    \
    cudaError_t e__ = (x);                                                                                \
    if (e__ != cudaSuccess)                                                                               \
      throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e__) + " at " + __FILE__ + \
                               ":" + std::to_string(__LINE__) + " (" #x ")");                             \
  } while (0)

// Every dynamic-smem kernel gets the same (device maximum) opt-in once per
// launch site, so CUDA-graph captures never see a smaller attribute than an
// earlier captured node needs.
constexpr int kMaxDynSmem = 220 * 1024;  // leaves room for static __shared__

// ------------------------------------------------------------------ complex
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// conj(a) * b
__host__ __device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
__host__ __device__ __forceinline__ double cnorm2(double2 a) { return a.x * a.x + a.y * a.y; }
// a += b * c
__device__ __forceinline__ void cfma(double2& a, double2 b, double2 c) {
  a.x = fma(b.x, c.x, fma(-b.y, c.y, a.x));
  a.y = fma(b.x, c.y, fma(b.y, c.x, a.y));
}
// a += conj(b) * c
__device__ __forceinline__ void cfmac(double2& a, double2 b, double2 c) {
  a.x = fma(b.x, c.x, fma(b.y, c.y, a.x));
  a.y = fma(b.x, c.y, fma(-b.y, c.x, a.y));
}
// complex division a / b (Smith)
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, den = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / den, (a.y - a.x * r) / den);
  }
  const double r = b.x / b.y, den = b.x * r + b.y;
  return make_double2((a.x * r + a.y) / den, (a.y * r - a.x) / den);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double2 warp_sum2(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// ------------------------------------------------------ rng.hpp:12-47 (exact)
__host__ __device__ __forceinline__ u64 splitmix_next(u64& state) {
  u64 z = (state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ u64 splitmix_bounded(u64& state, u64 bound) {
  const u64 threshold = (0ULL - bound) % bound;
  for (;;) {
    const u64 r = splitmix_next(state);
    if (r >= threshold) return r % bound;
  }
}
__host__ __device__ __forceinline__ u64 derive_seed(u64 seed, const u64* tags, int nt) {
  u64 g = seed ^ 0x6a09e667f3bcc909ULL;
  u64 h = splitmix_next(g);
  for (int i = 0; i < nt; ++i) {
    u64 m = h ^ (tags[i] + 0x9e3779b97f4a7c15ULL);
    h = splitmix_next(m);
  }
  return h;
}

// select_proxies_count (id.cpp:155-185), UniformRandom branch, without the
// O(extent) pool: a partial Fisher-Yates only touches <= 2*count positions, so
// a sparse (position -> value) map of the displaced entries reproduces the
// reference's swap sequence exactly.  out: `count` sorted 1-based values.
// Requires count <= kMaxProxy.
constexpr int kMaxProxy = 64;
__host__ __device__ inline void select_uniform_sparse(i64 extent, i64 count, u64 seed, int* out) {
  i64 pos[2 * kMaxProxy];
  i64 val[2 * kMaxProxy];
  int nmap = 0;
  auto lookup = [&](i64 p) -> i64 {
    for (int q = 0; q < nmap; ++q)
      if (pos[q] == p) return val[q];
    return p + 1;  // pool initialised to iota(1..extent)
  };
  auto store = [&](i64 p, i64 v) {
    for (int q = 0; q < nmap; ++q)
      if (pos[q] == p) {
        val[q] = v;
        return;
      }
    pos[nmap] = p;
    val[nmap] = v;
    ++nmap;
  };
  u64 st = seed;
  for (i64 i = 0; i < count; ++i) {
    const i64 j = i + static_cast<i64>(splitmix_bounded(st, static_cast<u64>(extent - i)));
    const i64 vi = lookup(i), vj = lookup(j);
    store(i, vj);
    store(j, vi);
  }
  for (i64 i = 0; i < count; ++i) out[i] = static_cast<int>(lookup(i));
  // insertion sort (count <= 64)
  for (i64 i = 1; i < count; ++i) {
    const int x = out[i];
    i64 k = i - 1;
    while (k >= 0 && out[k] > x) {
      out[k + 1] = out[k];
      --k;
    }
    out[k + 1] = x;
  }
}

// full select_proxies_count semantics for all three modes
__host__ __device__ inline i64 select_proxies(i64 extent, i64 count, int mode, u64 seed, int* out) {
  count = count < 1 ? 1 : count;
  count = count > extent ? extent : count;
  if (mode == OIOBF_PROXY_ALL) {
    for (i64 i = 0; i < extent; ++i) out[i] = static_cast<int>(i + 1);
    return extent;
  }
  if (mode == OIOBF_PROXY_EVENLY_SPACED) {
    i64 stride = extent / count;
    stride = stride < 1 ? 1 : stride;
    for (i64 i = 0; i < count; ++i) out[i] = static_cast<int>(1 + i * stride);
    return count;
  }
  select_uniform_sparse(extent, count, seed, out);
  return count;
}

// proxy_lists count rule (id.cpp:202-220): per-mode counts for 2d ranges with
// `skip` excluded, halving the first-largest count while the product exceeds
// row_cap.  Pure integer arithmetic, identical on host and device.
__host__ __device__ inline void proxy_counts(int nr, const i64* sizes, int skip, i64 per_mode, int mode, i64 row_cap,
                                             i64* counts) {
  for (int p = 0; p < nr; ++p) {
    if (p == skip) {
      counts[p] = 0;
      continue;
    }
    counts[p] = mode == OIOBF_PROXY_ALL ? sizes[p] : (sizes[p] < per_mode ? sizes[p] : per_mode);
  }
  for (;;) {
    i64 rows = 1;
    for (int p = 0; p < nr; ++p)
      if (p != skip) rows *= counts[p];
    if (rows <= row_cap) break;
    int argmax = skip == 0 ? 1 : 0;
    for (int p = 0; p < nr; ++p)
      if (p != skip && counts[p] > counts[argmax]) argmax = p;
    if (counts[argmax] <= 2) break;
    counts[argmax] = (counts[argmax] + 1) / 2;
  }
}

// ------------------------------------------------------------ kernel entries
// Same formulas and operation order as the oracle (no FMA contraction in the
// geometry so rho matches the CPU to the last bit; sin/cos are CUDA's).
struct KSpec {
  int kind, d;
  i64 n;
  int bitrev;
  unsigned seed;  // NUDFT locations
  double kappa, off0, off1, off2;
};

// NUDFT target location x^i_k in [0, n-1] (SPEC.md kernels: uniform per
// coordinate, counter-based from the seed and the flattened index)
__host__ __device__ __forceinline__ double nudft_loc(unsigned seed, i64 flat, int k, i64 n) {
  const u64 tags[3] = {0x4EULL, static_cast<u64>(flat), static_cast<u64>(k)};
  const u64 h = derive_seed(static_cast<u64>(seed), tags, 3);
  const double u = static_cast<double>(h >> 11) * 0x1.0p-53;
#ifdef __CUDA_ARCH__
  return __dmul_rn(u, static_cast<double>(n - 1));
#else
  return u * static_cast<double>(n - 1);
#endif
}

__device__ __forceinline__ i64 bitrev1(i64 i, i64 n) {
  i64 x = i - 1, r = 0;
  for (i64 b = 1; b < n; b <<= 1) {
    r = (r << 1) | (x & 1);
    x >>= 1;
  }
  return r + 1;
}

// Green geometry, split so row-invariant coordinates can be hoisted:
// target coordinate p of index i: i / n; source coordinate p: j / n + off_p
// (modes >= d stay 0 / off_p).  green_from_coords finishes the entry.
__device__ __forceinline__ double green_x(const KSpec& s, int i) {
  return __ddiv_rn(static_cast<double>(i), static_cast<double>(s.n));
}
__device__ __forceinline__ double green_y(const KSpec& s, int p, int j) {
  const double off = p == 0 ? s.off0 : p == 1 ? s.off1 : s.off2;
  return __dadd_rn(__ddiv_rn(static_cast<double>(j), static_cast<double>(s.n)), off);
}
__device__ __forceinline__ double2 green_from_coords(const KSpec& s, const double* xs, const double* ys) {
  const double dx = __dsub_rn(xs[0], ys[0]), dy = __dsub_rn(xs[1], ys[1]), dz = __dsub_rn(xs[2], ys[2]);
  const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  const double rho = __dsqrt_rn(r2);
  const double ph = __dmul_rn(s.kappa, rho);
  double sn, cs;
  sincos(ph, &sn, &cs);
  return make_double2(__ddiv_rn(cs, rho), __ddiv_rn(-sn, rho));
}

// Same entry with one reciprocal of rho instead of two divisions (each part
// within 1 ulp of the divided one) -- the ID panels' generator, where the
// entries only feed the pivoted QR (differences of this size are far below
// the 1e-12 pivot tie rule); cores and dense check rows keep the divisions.
__device__ __forceinline__ double2 green_from_coords_rcp(const KSpec& s, const double* xs, const double* ys) {
  const double dx = __dsub_rn(xs[0], ys[0]), dy = __dsub_rn(xs[1], ys[1]), dz = __dsub_rn(xs[2], ys[2]);
  const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  const double rho = __dsqrt_rn(r2);
  const double ph = __dmul_rn(s.kappa, rho);
  double sn, cs;
  sincos(ph, &sn, &cs);
  const double inv = __drcp_rn(rho);
  return make_double2(__dmul_rn(cs, inv), -__dmul_rn(sn, inv));
}

// Radon 2D entry given sin / cos(2 pi x_p) of the two target coordinates
// (hoistable: they depend on the target index only)
__device__ __forceinline__ double2 radon2d_entry_sc(const KSpec& s, const int* i, const int* j, double s1, double c1v,
                                                    double s2, double c2v) {
  const double n = static_cast<double>(s.n);
  const i64 k1i = j[0] - 1 - s.n / 2, k2i = j[1] - 1 - s.n / 2;
  const double k1 = static_cast<double>(k1i), k2 = static_cast<double>(k2i);
  const double c1 = __ddiv_rn(__dadd_rn(2.0, __dmul_rn(s1, s2)), 16.0);
  const double c2 = __ddiv_rn(__dadd_rn(2.0, __dmul_rn(c1v, c2v)), 16.0);
  i64 num = ((i[0] - 1) * k1i + (i[1] - 1) * k2i) % s.n;
  if (num < 0) num += s.n;
  const double frac = __ddiv_rn(static_cast<double>(num), n);
  const double q = __dadd_rn(__dmul_rn(__dmul_rn(__dmul_rn(c1, c1), k1), k1), __dmul_rn(__dmul_rn(__dmul_rn(c2, c2), k2), k2));
  const double phi = __dadd_rn(frac, __dsqrt_rn(q));
  double sn, cs;
  sincos(__dmul_rn(2.0 * M_PI, phi), &sn, &cs);
  return make_double2(cs, sn);
}

// i[], j[]: 1-based multi-indices
__device__ __forceinline__ double2 kernel_entry(const KSpec& s, const int* i, const int* j) {
  const double n = static_cast<double>(s.n);
  if (s.kind == OIOBF_KERNEL_GREEN) {
    double xs[3] = {0, 0, 0}, ys[3] = {s.off0, s.off1, s.off2};
    for (int p = 0; p < s.d; ++p) {
      xs[p] = green_x(s, i[p]);
      ys[p] = green_y(s, p, j[p]);
    }
    return green_from_coords(s, xs, ys);
  }
  if (s.kind == OIOBF_KERNEL_DFT) {
    i64 acc = 0;
    for (int p = 0; p < s.d; ++p) {
      const i64 a = s.bitrev ? bitrev1(i[p], s.n) : i[p];
      const i64 b = s.bitrev ? bitrev1(j[p], s.n) : j[p];
      acc += (a - 1) * (b - 1 - s.n / 2);
    }
    i64 m = acc % s.n;
    if (m < 0) m += s.n;
    const double t = __ddiv_rn(2.0 * static_cast<double>(m), n);
    double sn, cs;
    sincos(__dmul_rn(M_PI, t), &sn, &cs);
    return make_double2(cs, -sn);
  }
  if (s.kind == OIOBF_KERNEL_RADON3D) {  // exp(2 pi i (x.k + c |k|)), c = (3 + prod sin 2 pi x_p) / 100
    i64 num = 0;
    double ss = 1, kk = 0;
    for (int p = 0; p < 3; ++p) {
      const double x = __ddiv_rn(static_cast<double>(i[p] - 1), n);
      const i64 ki = j[p] - 1 - s.n / 2;
      num += (i[p] - 1) * ki;
      ss = __dmul_rn(ss, sin(__dmul_rn(2.0 * M_PI, x)));
      kk = __dadd_rn(kk, __dmul_rn(static_cast<double>(ki), static_cast<double>(ki)));
    }
    num %= s.n;
    if (num < 0) num += s.n;
    const double c = __ddiv_rn(__dadd_rn(3.0, ss), 100.0);
    const double phi = __dadd_rn(__ddiv_rn(static_cast<double>(num), n), __dmul_rn(c, __dsqrt_rn(kk)));
    double sn, cs;
    sincos(__dmul_rn(2.0 * M_PI, phi), &sn, &cs);
    return make_double2(cs, sn);
  }
  if (s.kind == OIOBF_KERNEL_NUDFT) {  // exp(2 pi i x^i . y^j), y^j_k = (j_k - 1) / n
    i64 flat = 0, st = 1;
    for (int p = 0; p < s.d; ++p) {
      flat += (i[p] - 1) * st;
      st *= s.n;
    }
    double phi = 0;
    for (int p = 0; p < s.d; ++p)
      phi = __dadd_rn(phi, __ddiv_rn(__dmul_rn(nudft_loc(s.seed, flat, p, s.n), static_cast<double>(j[p] - 1)), n));
    phi = __dsub_rn(phi, floor(phi));
    double sn, cs;
    sincos(__dmul_rn(2.0 * M_PI, phi), &sn, &cs);
    return make_double2(cs, sn);
  }
  // radon 2d
  const double x1 = __ddiv_rn(static_cast<double>(i[0] - 1), n), x2 = __ddiv_rn(static_cast<double>(i[1] - 1), n);
  double s1, c1v, s2, c2v;
  sincos(__dmul_rn(2.0 * M_PI, x1), &s1, &c1v);
  sincos(__dmul_rn(2.0 * M_PI, x2), &s2, &c2v);
  return radon2d_entry_sc(s, i, j, s1, c1v, s2, c2v);
}

inline KSpec kspec_from(const oiobf_kernel_spec& k) {
  KSpec s;
  s.kind = k.kind;
  s.d = k.d;
  s.n = k.n;
  s.bitrev = k.bitrev;
  s.seed = k.seed;
  s.kappa = k.kappa;
  s.off0 = k.offset[0];
  s.off1 = k.offset[1];
  s.off2 = k.offset[2];
  return s;
}

}  // namespace tbf
