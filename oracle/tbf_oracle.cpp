// ORACLE — TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library, and
// only as the checker or the CPU baseline.  The product (paper_2411_03029_b200)
// never links or calls it.
//
// CPU restatement of the reference semantics for the tensor-butterfly hot path
// (plain C++, no Eigen):
//   rng            rng.hpp:12-47          splitmix64, bounded, derive_seed
//   proxies        id.cpp:155-192,199-231 select_proxies(_count), proxy_lists
//   qrcp / ID      id.cpp:24-130          qrcp, id_from_qrcp, column_id
//   subtensor      tensor.cpp:249-266, 75-104 (subtensor_at + unfold, fused)
//   tucker_id      id.cpp:235-287
//   mode products  tensor.cpp:136-166     mode_product_blockdiag
//   butterfly      PAPER.md:295-341 (Alg. 1), PAPER.md:350-389 (Alg. 2),
//                  SPEC.md:268-317, SURVEY.md App. A (level rule, seeds, r_est)
//   kernels        BASELINE.json configs, SURVEY.md App. A1
//
// Arithmetic follows the sequential summation order of include/eigen_shim (the
// stand-in Eigen the reference compiles against here), so this oracle and
// oracle/_ref/libref.so agree bit for bit; tests/test_oracle_vs_ref.py pins it.
//
// Tie handling: qrcp records, per ID, the smallest pivot
// gap (best - runner-up residual norm, relative to |R11|) and the rank-threshold
// gap.  In replay mode a forced pivot / rank (e.g. the GPU's) is accepted only
// where the oracle's own choice is tied within tie_eps; any other disagreement
// is flagged as a mismatch.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

using i64 = std::int64_t;
using u64 = std::uint64_t;
using Cx = std::complex<double>;

thread_local std::string g_err;

// ---------------------------------------------------------------- rng.hpp:12-47
struct SplitMix64 {
  u64 state;
  explicit SplitMix64(u64 s) : state(s) {}
  u64 next() {
    u64 z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  u64 bounded(u64 bound) {
    const u64 threshold = -bound % bound;
    for (;;) {
      const u64 r = next();
      if (r >= threshold) return r % bound;
    }
  }
};

u64 derive_seed(u64 seed, const u64* tags, int nt) {
  SplitMix64 g(seed ^ 0x6a09e667f3bcc909ULL);
  u64 h = g.next();
  for (int i = 0; i < nt; ++i) {
    SplitMix64 m(h ^ (tags[i] + 0x9e3779b97f4a7c15ULL));
    h = m.next();
  }
  return h;
}

// -------------------------------------------------------------- id.cpp:155-192
enum ProxyMode { All = 0, UniformRandom = 1, EvenlySpaced = 2 };

struct Strategy {
  int mode = UniformRandom;
  i64 q = 3;
  i64 max_retries = 3;
  i64 row_cap = 1 << 17;
};

std::vector<i64> select_proxies_count(i64 extent, i64 count, int mode, u64 seed) {
  if (extent < 1) throw std::invalid_argument("select_proxies: extent must be positive");
  count = std::min(extent, std::max<i64>(count, 1));
  std::vector<i64> out;
  if (mode == All) {
    out.resize(static_cast<size_t>(extent));
    std::iota(out.begin(), out.end(), 1);
  } else if (mode == EvenlySpaced) {
    const i64 stride = std::max<i64>(1, extent / count);
    for (i64 i = 0; i < count; ++i) out.push_back(1 + i * stride);
  } else {
    std::vector<i64> pool(static_cast<size_t>(extent));
    std::iota(pool.begin(), pool.end(), 1);
    SplitMix64 g(seed);
    for (i64 i = 0; i < count; ++i) {
      const i64 j = i + static_cast<i64>(g.bounded(static_cast<u64>(extent - i)));
      std::swap(pool[static_cast<size_t>(i)], pool[static_cast<size_t>(j)]);
    }
    out.assign(pool.begin(), pool.begin() + count);
    std::sort(out.begin(), out.end());
  }
  return out;
}

// -------------------------------------------------------------- id.cpp:199-231
struct Range {
  i64 lo, hi;
  i64 size() const { return hi - lo + 1; }
};

std::vector<std::vector<i64>> proxy_lists(const std::vector<Range>& ranges, size_t skip, i64 per_mode,
                                          const Strategy& st, u64 seed) {
  std::vector<i64> counts(ranges.size(), 0);
  for (size_t p = 0; p < ranges.size(); ++p) {
    if (p == skip) continue;
    counts[p] = st.mode == All ? ranges[p].size() : std::min(ranges[p].size(), per_mode);
  }
  auto rows_of = [&]() {
    i64 r = 1;
    for (size_t p = 0; p < ranges.size(); ++p)
      if (p != skip) r *= counts[p];
    return r;
  };
  while (rows_of() > st.row_cap) {
    size_t argmax = skip == 0 ? 1 : 0;
    for (size_t p = 0; p < ranges.size(); ++p)
      if (p != skip && counts[p] > counts[argmax]) argmax = p;
    if (counts[argmax] <= 2) break;
    counts[argmax] = (counts[argmax] + 1) / 2;
  }
  std::vector<std::vector<i64>> lists(ranges.size());
  for (size_t p = 0; p < ranges.size(); ++p) {
    if (p == skip) continue;
    const u64 tags[2] = {0x70, static_cast<u64>(p)};
    auto local = select_proxies_count(ranges[p].size(), counts[p], st.mode, derive_seed(seed, tags, 2));
    for (auto& v : local) v += ranges[p].lo - 1;
    lists[p] = std::move(local);
  }
  return lists;
}

// --------------------------------------------------------------- id.cpp:24-120
struct Replay {  // forced decisions, used only where the oracle's own are tied
  const i64* perm = nullptr;  // forced pivot sequence (0-based original columns)
  i64 rank = -1;
  double tie_eps = 1e-12;
};

struct Qrcp {
  std::vector<i64> perm;
  std::vector<Cx> r;  // rank x n col-major
  i64 rank = 0;
  bool saturated = false;
  double min_gap = INFINITY;   // min over steps of (best - second) / ref
  double rank_gap = INFINITY;  // |eta - tol*ref| / ref at the stopping step
  bool mismatch = false;
};

// a: m x n column-major, modified in place.
Qrcp qrcp(std::vector<Cx>& a, i64 m, i64 n, double tol, i64 rank_limit, const Replay* rp) {
  auto A = [&](i64 i, i64 j) -> Cx& { return a[static_cast<size_t>(i + j * m)]; };
  Qrcp res;
  res.perm.resize(static_cast<size_t>(n));
  std::iota(res.perm.begin(), res.perm.end(), 0);
  const i64 limit = std::min({m, n, rank_limit});
  double ref = 0;
  i64 k = 0;
  std::vector<double> nrm(static_cast<size_t>(n));
  for (;; ++k) {
    i64 jmax = -1;
    double best = -1;
    for (i64 j = k; j < n; ++j) {
      double c = 0;
      for (i64 i = k; i < m; ++i) c += std::norm(A(i, j));
      nrm[static_cast<size_t>(j)] = c;
      if (c > best) {
        best = c;
        jmax = j;
      }
    }
    double eta = jmax >= 0 ? std::sqrt(best) : 0;
    const double refk = k == 0 ? eta : ref;
    // tie bookkeeping
    if (jmax >= 0 && refk > 0) {
      double second = -1;
      for (i64 j = k; j < n; ++j)
        if (j != jmax) second = std::max(second, nrm[static_cast<size_t>(j)]);
      if (second >= 0) res.min_gap = std::min(res.min_gap, (eta - std::sqrt(second)) / refk);
    }
    bool stop;
    if (k == 0) {
      ref = eta;
      stop = (ref == 0);
    } else {
      stop = (jmax < 0 || eta <= tol * ref);
      if (jmax >= 0 && ref > 0) {
        const double g = std::fabs(eta - tol * ref) / ref;
        if (rp && rp->rank >= 0 && g <= rp->tie_eps) stop = (k == rp->rank);
        else if (rp && rp->rank >= 0 && stop != (k == rp->rank)) res.mismatch = true;
        if (stop) res.rank_gap = g;
      }
    }
    if (stop) break;
    if (k == limit) {
      res.saturated = (eta > tol * ref) && (limit < n);
      break;
    }
    if (rp && rp->perm) {  // forced pivot where tied
      const i64 want = rp->perm[k];
      i64 pos = -1;
      for (i64 j = k; j < n; ++j)
        if (res.perm[static_cast<size_t>(j)] == want) pos = j;
      if (pos < 0) {
        res.mismatch = true;
      } else if (pos != jmax) {
        const double gap = (eta - std::sqrt(nrm[static_cast<size_t>(pos)])) / (ref > 0 ? ref : 1);
        if (gap <= rp->tie_eps) {
          jmax = pos;
          eta = std::sqrt(nrm[static_cast<size_t>(pos)]);
        } else {
          res.mismatch = true;
        }
      }
    }
    // a.col(k).swap(a.col(jmax))
    for (i64 i = 0; i < m; ++i) std::swap(A(i, k), A(i, jmax));
    std::swap(res.perm[static_cast<size_t>(k)], res.perm[static_cast<size_t>(jmax)]);
    // Householder reflector zeroing a(k+1:m, k)
    const i64 tail = m - k;
    double xs = 0;
    for (i64 i = k; i < m; ++i) xs += std::norm(A(i, k));
    const double xnorm = std::sqrt(xs);
    if (xnorm > 0) {
      const Cx alpha = A(k, k);
      const Cx sign = (alpha == Cx(0, 0)) ? Cx(1, 0) : alpha / std::abs(alpha);
      std::vector<Cx> v(static_cast<size_t>(tail));
      for (i64 i = 0; i < tail; ++i) v[static_cast<size_t>(i)] = A(k + i, k);
      v[0] += sign * xnorm;
      double vn2 = 0;
      for (const Cx& z : v) vn2 += std::norm(z);
      if (vn2 > 0) {
        const double beta = 2.0 / vn2;
        std::vector<Cx> w(static_cast<size_t>(n - k));
        for (i64 j = k; j < n; ++j) {
          Cx s(0, 0);
          for (i64 i = 0; i < tail; ++i) s += std::conj(v[static_cast<size_t>(i)]) * A(k + i, j);
          w[static_cast<size_t>(j - k)] = beta * s;
        }
        for (i64 j = k; j < n; ++j)
          for (i64 i = 0; i < tail; ++i) A(k + i, j) -= v[static_cast<size_t>(i)] * w[static_cast<size_t>(j - k)];
      }
      for (i64 i = k; i < m; ++i) A(i, k) = Cx(0, 0);
      A(k, k) = -sign * xnorm;
    }
  }
  res.rank = k;
  res.r.resize(static_cast<size_t>(k * n));
  for (i64 j = 0; j < n; ++j)
    for (i64 i = 0; i < k; ++i) res.r[static_cast<size_t>(i + j * k)] = A(i, j);
  return res;
}

struct ColumnID {
  std::vector<i64> skeleton;  // 1-based, sorted
  std::vector<Cx> interp;     // rank x n col-major
  i64 rank = 0;
  bool saturated = false;
  double interp_max_abs = 0;
  std::vector<i64> perm;
  double min_gap = INFINITY, rank_gap = INFINITY;
  bool mismatch = false;
};

ColumnID id_from_qrcp(const Qrcp& q, i64 n) {
  ColumnID id;
  id.rank = q.rank;
  id.saturated = q.saturated;
  id.perm = q.perm;
  id.min_gap = q.min_gap;
  id.rank_gap = q.rank_gap;
  id.mismatch = q.mismatch;
  const i64 r = q.rank;
  auto R = [&](i64 i, i64 j) { return q.r[static_cast<size_t>(i + j * r)]; };
  // t = R11^{-1} R12 by back substitution (eigen_shim UpperTri::solve order)
  std::vector<Cx> t(static_cast<size_t>(r * std::max<i64>(n - r, 0)));
  for (i64 c = 0; c < n - r; ++c)
    for (i64 i = r - 1; i >= 0; --i) {
      Cx s = R(i, r + c);
      for (i64 k = i + 1; k < r; ++k) s -= R(i, k) * t[static_cast<size_t>(k + c * r)];
      t[static_cast<size_t>(i + c * r)] = s / R(i, i);
    }
  std::vector<i64> order(static_cast<size_t>(r));
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(),
            [&](i64 a, i64 b) { return q.perm[static_cast<size_t>(a)] < q.perm[static_cast<size_t>(b)]; });
  id.skeleton.resize(static_cast<size_t>(r));
  id.interp.assign(static_cast<size_t>(r * n), Cx(0, 0));
  for (i64 i = 0; i < r; ++i) {
    const i64 p = order[static_cast<size_t>(i)];
    id.skeleton[static_cast<size_t>(i)] = q.perm[static_cast<size_t>(p)] + 1;
    id.interp[static_cast<size_t>(i + q.perm[static_cast<size_t>(p)] * r)] = Cx(1, 0);
    for (i64 j = r; j < n; ++j)
      id.interp[static_cast<size_t>(i + q.perm[static_cast<size_t>(j)] * r)] = t[static_cast<size_t>(p + (j - r) * r)];
  }
  double mx = 0;
  for (const Cx& z : id.interp) mx = std::max(mx, std::abs(z));
  id.interp_max_abs = (r > 0 && n > 0) ? mx : 0.0;
  return id;
}

ColumnID column_id(std::vector<Cx> a, i64 m, i64 n, double tol, i64 max_rank, const Replay* rp) {
  if (!(m > 0 && n > 0)) throw std::invalid_argument("column_id: empty matrix");
  if (!(tol > 0 && tol < 1)) throw std::invalid_argument("column_id: tolerance must be in (0,1)");
  const i64 limit = max_rank >= 0 ? max_rank : std::min(m, n);
  Qrcp q = qrcp(a, m, n, tol, limit, rp);
  return id_from_qrcp(q, n);
}

// ----------------------------------------------------- kernels
struct Spec {
  int kind = 0;  // 0 green, 1 dft, 2 radon2d, 3 radon3d, 4 nudft
  int d = 2;
  i64 n = 0;
  int bitrev = 0;
  u64 seed = 0;  // nudft locations
  double kappa = 0;
  double offset[3] = {0, 0, 0};
};

// NUDFT target location x^i_k in [0, n-1]: uniform per coordinate, counter-based
// from the seed and the flattened (0-based, mode-0-fastest) target index
// (SPEC.md kernels design decisions; "random in [0, n-1]")
double nudft_loc(u64 seed, i64 flat, int k, i64 n) {
  const u64 tags[3] = {0x4EULL, static_cast<u64>(flat), static_cast<u64>(k)};
  const u64 h = derive_seed(seed, tags, 3);
  return static_cast<double>(h >> 11) * 0x1.0p-53 * static_cast<double>(n - 1);
}

i64 bitrev1(i64 i, i64 n) {
  i64 x = i - 1, r = 0;
  for (i64 b = 1; b < n; b <<= 1) {
    r = (r << 1) | (x & 1);
    x >>= 1;
  }
  return r + 1;
}

// i, j: 1-based multi-indices (d entries each)
Cx kernel_eval(const Spec& s, const i64* i, const i64* j) {
  const double n = static_cast<double>(s.n);
  if (s.kind == 0) {  // exp(-i kappa rho) / rho
    double xs[3] = {0, 0, 0}, ys[3] = {0, 0, 0};
    for (int p = 0; p < s.d; ++p) {
      xs[p] = static_cast<double>(i[p]) / n;
      ys[p] = static_cast<double>(j[p]) / n;
    }
    for (int p = 0; p < 3; ++p) ys[p] += s.offset[p];
    const double dx = xs[0] - ys[0], dy = xs[1] - ys[1], dz = xs[2] - ys[2];
    const double rho = std::sqrt(dx * dx + dy * dy + dz * dz);
    const double ph = s.kappa * rho;
    return Cx(std::cos(ph) / rho, -std::sin(ph) / rho);
  }
  if (s.kind == 1) {  // exp(-2 pi i x.k), x=(i-1)/n, k=j-1-n/2, exact phase mod n
    i64 acc = 0;
    for (int p = 0; p < s.d; ++p) {
      const i64 a = s.bitrev ? bitrev1(i[p], s.n) : i[p];
      const i64 b = s.bitrev ? bitrev1(j[p], s.n) : j[p];
      acc += (a - 1) * (b - 1 - s.n / 2);
    }
    i64 m = acc % s.n;
    if (m < 0) m += s.n;
    const double t = 2.0 * static_cast<double>(m) / n;
    return Cx(std::cos(M_PI * t), -std::sin(M_PI * t));
  }
  if (s.kind == 3) {  // Radon 3D: Phi = x.k + c|k|, c = (3 + prod sin 2 pi x_p)/100
    i64 num = 0;
    double ss = 1, kk = 0;
    for (int p = 0; p < 3; ++p) {
      const double x = static_cast<double>(i[p] - 1) / n;
      const i64 ki = j[p] - 1 - s.n / 2;
      num += (i[p] - 1) * ki;
      ss = ss * std::sin(2.0 * M_PI * x);
      kk = kk + static_cast<double>(ki) * static_cast<double>(ki);
    }
    num %= s.n;
    if (num < 0) num += s.n;
    const double c = (3.0 + ss) / 100.0;
    const double phi = static_cast<double>(num) / n + c * std::sqrt(kk);
    const double ph = 2.0 * M_PI * phi;
    return Cx(std::cos(ph), std::sin(ph));
  }
  if (s.kind == 4) {  // type-2 NUDFT: exp(2 pi i x^i . y^j), y^j_k = (j_k - 1)/n
    i64 flat = 0, st = 1;
    for (int p = 0; p < s.d; ++p) {
      flat += (i[p] - 1) * st;
      st *= s.n;
    }
    double phi = 0;
    for (int p = 0; p < s.d; ++p) phi = phi + nudft_loc(s.seed, flat, p, s.n) * static_cast<double>(j[p] - 1) / n;
    phi = phi - std::floor(phi);
    const double ph = 2.0 * M_PI * phi;
    return Cx(std::cos(ph), std::sin(ph));
  }
  // generalized Radon 2D: exp(2 pi i Phi)
  const double x1 = static_cast<double>(i[0] - 1) / n, x2 = static_cast<double>(i[1] - 1) / n;
  const i64 k1i = j[0] - 1 - s.n / 2, k2i = j[1] - 1 - s.n / 2;
  const double k1 = static_cast<double>(k1i), k2 = static_cast<double>(k2i);
  const double s1 = std::sin(2.0 * M_PI * x1), s2 = std::sin(2.0 * M_PI * x2);
  const double c1v = std::cos(2.0 * M_PI * x1), c2v = std::cos(2.0 * M_PI * x2);
  const double c1 = (2.0 + s1 * s2) / 16.0, c2 = (2.0 + c1v * c2v) / 16.0;
  i64 num = ((i[0] - 1) * k1i + (i[1] - 1) * k2i) % s.n;
  if (num < 0) num += s.n;
  const double frac = static_cast<double>(num) / n;
  const double phi = frac + std::sqrt(c1 * c1 * k1 * k1 + c2 * c2 * k2 * k2);
  const double ph = 2.0 * M_PI * phi;
  return Cx(std::cos(ph), std::sin(ph));
}

Spec spec_from(const int* si, const double* sf) {
  Spec s;
  s.kind = si[0];
  s.d = si[1];
  s.n = si[2];
  s.bitrev = si[3];
  s.seed = static_cast<u64>(static_cast<uint32_t>(si[4]));
  s.kappa = sf[0];
  s.offset[0] = sf[1];
  s.offset[1] = sf[2];
  s.offset[2] = sf[3];
  if (s.d < 1 || s.d > 6) throw std::invalid_argument("kernel spec: d must be in [1,6]");
  if (s.kind == 2 && s.d != 2) throw std::invalid_argument("kernel spec: radon2d needs d=2");
  if (s.kind == 0 && s.d > 3) throw std::invalid_argument("kernel spec: green needs d<=3");
  if (s.kind == 3 && s.d != 3) throw std::invalid_argument("kernel spec: radon3d needs d=3");
  if (s.kind < 0 || s.kind > 4) throw std::invalid_argument("make_kernel: unknown kernel kind");
  return s;
}

// Mode-`skip` unfolding of K(lists) (subtensor_at + unfold, tensor.cpp:249-266,
// 75-104): rows flatten the complement modes in increasing order, first
// fastest; column c is lists[skip][c].
std::vector<Cx> unfolding(const Spec& s, const std::vector<std::vector<i64>>& lists, size_t skip, i64* m_out) {
  const int D = 2 * s.d;
  i64 m = 1;
  for (int p = 0; p < D; ++p)
    if (static_cast<size_t>(p) != skip) m *= static_cast<i64>(lists[static_cast<size_t>(p)].size());
  const i64 w = static_cast<i64>(lists[skip].size());
  std::vector<Cx> a(static_cast<size_t>(m * w));
  std::vector<i64> idx(static_cast<size_t>(D));
  i64 ii[6], jj[6];
  for (i64 c = 0; c < w; ++c) {
    std::fill(idx.begin(), idx.end(), 0);
    for (i64 r = 0; r < m; ++r) {
      for (int p = 0; p < D; ++p) {
        const i64 v = static_cast<size_t>(p) == skip ? lists[skip][static_cast<size_t>(c)]
                                                       : lists[static_cast<size_t>(p)][static_cast<size_t>(idx[static_cast<size_t>(p)])];
        if (p < s.d) ii[p] = v;
        else jj[p - s.d] = v;
      }
      a[static_cast<size_t>(r + c * m)] = kernel_eval(s, ii, jj);
      for (int p = 0; p < D; ++p) {  // advance mixed radix over complement modes
        if (static_cast<size_t>(p) == skip) continue;
        if (++idx[static_cast<size_t>(p)] < static_cast<i64>(lists[static_cast<size_t>(p)].size())) break;
        idx[static_cast<size_t>(p)] = 0;
      }
    }
  }
  *m_out = m;
  return a;
}

// ------------------------------------------------------------ thread helper
void parallel_for(i64 n, int nthreads, const std::function<void(i64)>& f) {
  if (nthreads <= 1 || n <= 1) {
    for (i64 i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<i64> next{0};
  std::vector<std::thread> th;
  std::exception_ptr err;
  std::atomic<bool> failed{false};
  for (int t = 0; t < nthreads; ++t)
    th.emplace_back([&]() {
      for (;;) {
        const i64 i = next.fetch_add(1);
        if (i >= n || failed.load()) break;
        try {
          f(i);
        } catch (...) {
          if (!failed.exchange(true)) err = std::current_exception();
        }
      }
    });
  for (auto& t : th) t.join();
  if (err) std::rethrow_exception(err);
}

// ------------------------------------------------------------ butterfly (Alg 1)
struct Slot {
  i64 rank = 0, ncols = 0, rows = 0;
  std::vector<i64> skel;    // global 1-based, sorted
  std::vector<i64> target;  // global 1-based candidate columns
  std::vector<Cx> interp;   // rank x ncols
  std::vector<i64> perm;    // pivot order (0-based into target)
  double min_gap = INFINITY, rank_gap = INFINITY;
  bool mismatch = false, saturated = false;
};

struct TBF {
  Spec spec;
  int L = 0, Lc = 0;
  double tol = 0;
  Strategy st;
  u64 seed = 0;
  i64 nmid = 0;                                // 2^{d Lc} mid multi-sets per side
  std::vector<std::vector<Slot>> side[2];      // [0]=V/W (column side), [1]=U/P
  std::vector<std::vector<Cx>> cores;          // pair p = s*nmid + t, col-major (prod r_t) x (prod r_s)
  std::vector<i64> core_rows, core_cols;
  std::vector<i64> r_est[2];                   // r_est used at each level
};

i64 ipow(i64 b, i64 e) {
  i64 r = 1;
  while (e-- > 0) r *= b;
  return r;
}

Range node_range(i64 n, int level, i64 pos) {
  const i64 sz = n >> level;
  return Range{pos * sz + 1, (pos + 1) * sz};
}

// slot index within level l: ((outer * nin + inner) * d + k) * nj + j
struct LevelShape {
  i64 nin, nj, count;
};
LevelShape level_shape(const TBF& b, int l) {
  const int d = b.spec.d;
  LevelShape ls;
  ls.nin = ipow(2, static_cast<i64>(d) * l);
  ls.nj = ipow(2, b.Lc - l);
  ls.count = b.nmid * ls.nin * d * ls.nj;
  return ls;
}

// Build one level of one side.  side 0 (V/W): outer = s (mid col multi-set),
// inner = tau (level-l row multi-set), node nu at level L-l inside s_k, unfold
// mode d+k.  side 1 (U/P): outer = t, inner = nu (level-l col multi-set), node
// tau at level L-l inside t_k, unfold mode k.
void build_level(TBF& b, int sd, int l, i64 r_est, int nthreads, const Replay* const* replay) {
  const int d = b.spec.d;
  const i64 n = b.spec.n;
  const i64 mid_per_mode = ipow(2, b.Lc);
  const LevelShape ls = level_shape(b, l);
  auto& slots = b.side[sd][static_cast<size_t>(l)];
  slots.assign(static_cast<size_t>(ls.count), Slot{});
  const i64 per_mode = b.st.q * r_est;  // attempt 0: q * r_est * 2^0 (id.cpp:257)
  parallel_for(ls.count, nthreads, [&](i64 idx) {
    const i64 j = idx % ls.nj;
    const i64 k = (idx / ls.nj) % d;
    const i64 inner = (idx / (ls.nj * d)) % ls.nin;
    const i64 outer = idx / (ls.nj * d * ls.nin);
    std::vector<Range> ranges(static_cast<size_t>(2 * d));
    i64 outer_pos[6], inner_pos[6];
    for (int p = 0; p < d; ++p) {
      outer_pos[p] = (outer / ipow(mid_per_mode, p)) % mid_per_mode;
      inner_pos[p] = (inner / ipow(ipow(2, l), p)) % ipow(2, l);
    }
    const i64 node_pos = outer_pos[k] * ls.nj + j;  // at level L-l
    const int mid_off = sd == 0 ? d : 0;             // side whose ranges are mid nodes
    const int in_off = sd == 0 ? 0 : d;
    for (int p = 0; p < d; ++p) {
      ranges[static_cast<size_t>(mid_off + p)] = node_range(n, b.Lc, outer_pos[p]);
      ranges[static_cast<size_t>(in_off + p)] = node_range(n, l, inner_pos[p]);
    }
    const size_t skip = static_cast<size_t>(mid_off + k);
    ranges[skip] = node_range(n, b.L - l, node_pos);
    Slot& sl = slots[static_cast<size_t>(idx)];
    if (l == 0) {
      for (i64 v = ranges[skip].lo; v <= ranges[skip].hi; ++v) sl.target.push_back(v);
    } else {
      i64 pin = 0;  // parent inner multi-set at level l-1
      for (int p = d - 1; p >= 0; --p) pin = pin * ipow(2, l - 1) + inner_pos[p] / 2;
      const LevelShape lp = level_shape(b, l - 1);
      for (i64 c = 0; c < 2; ++c) {
        const i64 cidx = ((outer * lp.nin + pin) * d + k) * lp.nj + 2 * j + c;
        const Slot& ch = b.side[sd][static_cast<size_t>(l - 1)][static_cast<size_t>(cidx)];
        sl.target.insert(sl.target.end(), ch.skel.begin(), ch.skel.end());
      }
    }
    const u64 tags[7] = {sd == 0 ? 0x56ULL : 0x55ULL, static_cast<u64>(l), static_cast<u64>(outer),
                         static_cast<u64>(inner), static_cast<u64>(k), static_cast<u64>(j), 0ULL};
    const u64 s = derive_seed(b.seed, tags, 7);
    auto lists = proxy_lists(ranges, skip, per_mode, b.st, s);
    lists[skip] = sl.target;
    sl.ncols = static_cast<i64>(sl.target.size());
    if (sl.ncols == 0) return;  // both children rank 0: empty slot
    i64 m = 0;
    std::vector<Cx> a = unfolding(b.spec, lists, skip, &m);
    sl.rows = m;
    const Replay* rp = replay ? replay[idx] : nullptr;
    ColumnID id = column_id(std::move(a), m, sl.ncols, b.tol, -1, rp);
    sl.rank = id.rank;
    sl.saturated = id.saturated;
    sl.interp = std::move(id.interp);
    sl.perm = std::move(id.perm);
    sl.min_gap = id.min_gap;
    sl.rank_gap = id.rank_gap;
    sl.mismatch = id.mismatch;
    for (i64 v : id.skeleton) sl.skel.push_back(sl.target[static_cast<size_t>(v - 1)]);
  });
}

int level_rule(i64 n, i64 cb) {  // largest even L with n / 2^L >= C_b
  int L = 0;
  while ((n >> (L + 2)) >= cb && (n % (i64{1} << (L + 2))) == 0) L += 2;
  return L;
}

void build_cores(TBF& b, int nthreads) {
  const int d = b.spec.d;
  const i64 P = b.nmid * b.nmid;
  b.cores.assign(static_cast<size_t>(P), {});
  b.core_rows.assign(static_cast<size_t>(P), 0);
  b.core_cols.assign(static_cast<size_t>(P), 0);
  const LevelShape ls = level_shape(b, b.Lc);  // nj == 1 at l = Lc
  parallel_for(P, nthreads, [&](i64 p) {
    const i64 s = p / b.nmid, t = p % b.nmid;
    std::vector<const std::vector<i64>*> rl(static_cast<size_t>(d)), cl(static_cast<size_t>(d));
    i64 R = 1, C = 1;
    for (int k = 0; k < d; ++k) {
      const Slot& u = b.side[1][static_cast<size_t>(b.Lc)][static_cast<size_t>((t * ls.nin + s) * d + k)];
      const Slot& v = b.side[0][static_cast<size_t>(b.Lc)][static_cast<size_t>((s * ls.nin + t) * d + k)];
      rl[static_cast<size_t>(k)] = &u.skel;
      cl[static_cast<size_t>(k)] = &v.skel;
      R *= static_cast<i64>(u.skel.size());
      C *= static_cast<i64>(v.skel.size());
    }
    std::vector<Cx>& core = b.cores[static_cast<size_t>(p)];
    core.resize(static_cast<size_t>(R * C));
    i64 ii[6], jj[6];
    for (i64 f = 0; f < R * C; ++f) {
      i64 rem = f;
      for (int k = 0; k < d; ++k) {
        const i64 e = static_cast<i64>(rl[static_cast<size_t>(k)]->size());
        ii[k] = (*rl[static_cast<size_t>(k)])[static_cast<size_t>(rem % e)];
        rem /= e;
      }
      for (int k = 0; k < d; ++k) {
        const i64 e = static_cast<i64>(cl[static_cast<size_t>(k)]->size());
        jj[k] = (*cl[static_cast<size_t>(k)])[static_cast<size_t>(rem % e)];
        rem /= e;
      }
      core[static_cast<size_t>(f)] = kernel_eval(b.spec, ii, jj);
    }
    b.core_rows[static_cast<size_t>(p)] = R;
    b.core_cols[static_cast<size_t>(p)] = C;
  });
}

// ------------------------------------------------------------ tensor helpers
struct Tensor {
  std::vector<i64> shape;  // first mode fastest
  std::vector<Cx> data;
};

// mode_product_blockdiag (tensor.cpp:136-166) with the eigen_shim product order:
// out(row, co + o) = sum_i unf(row, ci + i) * X(i, o), X = B^T (or B if transposed)
Tensor mode_product_blockdiag(const Tensor& t, int mode /*0-based*/, const std::vector<const Cx*>& blocks,
                              const std::vector<i64>& br, const std::vector<i64>& bc, bool transpose) {
  const size_t nb = blocks.size();
  i64 in_total = 0, out_total = 0;
  for (size_t b = 0; b < nb; ++b) {
    in_total += transpose ? br[b] : bc[b];
    out_total += transpose ? bc[b] : br[b];
  }
  if (in_total != t.shape[static_cast<size_t>(mode)]) throw std::invalid_argument("mode_product_blockdiag: shape mismatch");
  i64 below = 1, above = 1;
  for (int k = 0; k < mode; ++k) below *= t.shape[static_cast<size_t>(k)];
  for (size_t k = static_cast<size_t>(mode) + 1; k < t.shape.size(); ++k) above *= t.shape[k];
  const i64 nin = in_total;
  Tensor o;
  o.shape = t.shape;
  o.shape[static_cast<size_t>(mode)] = out_total;
  o.data.assign(static_cast<size_t>(below * above * out_total), Cx(0, 0));
  i64 ci = 0, co = 0;
  for (size_t b = 0; b < nb; ++b) {
    const i64 bin = transpose ? br[b] : bc[b];
    const i64 bout = transpose ? bc[b] : br[b];
    const Cx* B = blocks[b];
    const i64 ldb = br[b];
    for (i64 a = 0; a < above; ++a)
      for (i64 oo = 0; oo < bout; ++oo)
        for (i64 w = 0; w < below; ++w) {
          Cx s(0, 0);
          for (i64 i = 0; i < bin; ++i) {
            const Cx x = transpose ? B[i + oo * ldb] : B[oo + i * ldb];
            s += t.data[static_cast<size_t>(w + below * ((ci + i) + nin * a))] * x;
          }
          o.data[static_cast<size_t>(w + below * ((co + oo) + out_total * a))] = s;
        }
    ci += bin;
    co += bout;
  }
  return o;
}

// Alg. 2.  F: n^d x nv, G: n^d x nv, first mode fastest.
// Sharded apply (mirrors paper_2411_03029_b200/sharded.py): phase 1 = V/W
// levels + core mat-vec for the owned column multi-sets s, blocks G_{t,s}
// written at send_off[t*nmid+s]*nv; phase 2 = P/U levels for the owned row
// multi-sets t, blocks read at recv_off[t*nmid+s]*nv.  phase 0 = everything.
struct ShardIO {
  int phase = 0, rank = 0, world = 1;
  const int* owner = nullptr;  // ownership map of the middle multi-sets (null: index % world)
  Cx* send = nullptr;
  const i64* send_off = nullptr;
  const Cx* recv = nullptr;
  const i64* recv_off = nullptr;
};

void tbf_contract(const TBF& b, const Cx* F, Cx* G, i64 nv, int nthreads, const ShardIO* io = nullptr) {
  const int phase = io ? io->phase : 0;
  auto own = [&](i64 outer) {
    if (!io || io->world <= 1) return true;
    return (io->owner ? static_cast<i64>(io->owner[outer]) : outer % io->world) == io->rank;
  };
  const int d = b.spec.d;
  const i64 n = b.spec.n;
  const i64 mpm = ipow(2, b.Lc);
  const i64 mid_sz = n >> b.Lc;
  const i64 N = ipow(n, d);
  auto pos_of = [&](i64 idx, i64 base, int p) { return (idx / ipow(base, p)) % base; };
  auto gather_blocks = [&](int sd, int l, i64 outer, i64 inner, int k, std::vector<const Cx*>& ptr,
                           std::vector<i64>& br, std::vector<i64>& bc) {
    const LevelShape ls = level_shape(b, l);
    ptr.clear();
    br.clear();
    bc.clear();
    for (i64 j = 0; j < ls.nj; ++j) {
      const Slot& sl = b.side[sd][static_cast<size_t>(l)][static_cast<size_t>(((outer * ls.nin + inner) * d + k) * ls.nj + j)];
      ptr.push_back(sl.interp.data());
      br.push_back(sl.rank);
      bc.push_back(sl.ncols);
    }
  };
  // Step 1: F_{tau,s}
  std::vector<std::vector<Tensor>> Fl(static_cast<size_t>(b.Lc + 1));
  for (int l = 0; l <= b.Lc; ++l) {
    const LevelShape ls = level_shape(b, l);
    Fl[static_cast<size_t>(l)].assign(static_cast<size_t>(b.nmid * ls.nin), Tensor{});
    parallel_for(b.nmid * ls.nin, nthreads, [&](i64 it) {
      const i64 s = it / ls.nin, tau = it % ls.nin;
      if (phase == 2 || !own(s)) return;
      Tensor x;
      if (l == 0) {
        x.shape.assign(static_cast<size_t>(d), mid_sz);
        x.shape.push_back(nv);
        i64 tot = ipow(mid_sz, d) * nv;
        x.data.resize(static_cast<size_t>(tot));
        for (i64 f = 0; f < tot; ++f) {
          i64 rem = f, g = 0, stride = 1;
          for (int p = 0; p < d; ++p) {
            const i64 loc = rem % mid_sz;
            rem /= mid_sz;
            g += (pos_of(s, mpm, p) * mid_sz + loc) * stride;
            stride *= n;
          }
          g += rem * N;
          x.data[static_cast<size_t>(f)] = F[g];
        }
      } else {
        i64 ptau = 0;
        for (int p = d - 1; p >= 0; --p) ptau = ptau * ipow(2, l - 1) + pos_of(tau, ipow(2, l), p) / 2;
        x = Fl[static_cast<size_t>(l - 1)][static_cast<size_t>(s * ipow(2, static_cast<i64>(d) * (l - 1)) + ptau)];
      }
      std::vector<const Cx*> ptr;
      std::vector<i64> br, bc;
      for (int k = 0; k < d; ++k) {
        gather_blocks(0, l, s, tau, k, ptr, br, bc);
        x = mode_product_blockdiag(x, k, ptr, br, bc, false);
      }
      Fl[static_cast<size_t>(l)][static_cast<size_t>(it)] = std::move(x);
    });
  }
  // Step 2: G_{t,s} = K(tbar, sbar) x F_{t,s}; stored per (t, nu=s) at level Lc
  std::vector<std::vector<Tensor>> Gl(static_cast<size_t>(b.Lc + 1));
  const LevelShape lc = level_shape(b, b.Lc);
  Gl[static_cast<size_t>(b.Lc)].assign(static_cast<size_t>(b.nmid * b.nmid), Tensor{});
  parallel_for(b.nmid * b.nmid, nthreads, [&](i64 it) {
    const i64 t = it / b.nmid, s = it % b.nmid;  // G index = t * nmid + nu
    if (phase == 2 || !own(s)) return;
    const i64 p = s * b.nmid + t;
    const Tensor& x = Fl[static_cast<size_t>(b.Lc)][static_cast<size_t>(s * lc.nin + t)];
    const i64 R = b.core_rows[static_cast<size_t>(p)], C = b.core_cols[static_cast<size_t>(p)];
    const Cx* K = b.cores[static_cast<size_t>(p)].data();
    Tensor g;
    for (int k = 0; k < d; ++k)
      g.shape.push_back(b.side[1][static_cast<size_t>(b.Lc)][static_cast<size_t>((t * lc.nin + s) * d + k)].rank);
    g.shape.push_back(nv);
    g.data.assign(static_cast<size_t>(R * nv), Cx(0, 0));
    for (i64 v = 0; v < nv; ++v)
      for (i64 r = 0; r < R; ++r) {
        Cx acc(0, 0);
        for (i64 c = 0; c < C; ++c) acc += K[r + c * R] * x.data[static_cast<size_t>(c + v * C)];
        g.data[static_cast<size_t>(r + v * R)] = acc;
      }
    if (phase == 1) {
      Cx* dst = io->send + io->send_off[t * b.nmid + s] * nv;
      std::copy(g.data.begin(), g.data.end(), dst);
      return;
    }
    Gl[static_cast<size_t>(b.Lc)][static_cast<size_t>(it)] = std::move(g);
  });
  if (phase == 1) return;
  if (phase == 2) {  // the blocks G_{t,s} of the owned t arrive from the exchange
    for (i64 t = 0; t < b.nmid; ++t) {
      if (!own(t)) continue;
      for (i64 s = 0; s < b.nmid; ++s) {
        Tensor g;
        i64 R = 1;
        for (int k = 0; k < d; ++k) {
          g.shape.push_back(b.side[1][static_cast<size_t>(b.Lc)][static_cast<size_t>((t * lc.nin + s) * d + k)].rank);
          R *= g.shape.back();
        }
        g.shape.push_back(nv);
        const Cx* src = io->recv + io->recv_off[t * b.nmid + s] * nv;
        g.data.assign(src, src + R * nv);
        Gl[static_cast<size_t>(b.Lc)][static_cast<size_t>(t * b.nmid + s)] = std::move(g);
      }
    }
  }
  // Step 3: l = Lc..1 accumulate through P^T into parents; l = 0 through U^T
  for (int l = b.Lc; l >= 0; --l) {
    const LevelShape ls = level_shape(b, l);
    if (l > 0) {
      const i64 npar = ipow(2, static_cast<i64>(d) * (l - 1));
      Gl[static_cast<size_t>(l - 1)].assign(static_cast<size_t>(b.nmid * npar), Tensor{});
      parallel_for(b.nmid * npar, nthreads, [&](i64 it) {
        const i64 t = it / npar, pnu = it % npar;
        if (!own(t)) return;
        Tensor acc;
        bool first = true;
        for (i64 nu = 0; nu < ls.nin; ++nu) {  // children of pnu, ascending
          i64 par = 0;
          for (int p = d - 1; p >= 0; --p) par = par * ipow(2, l - 1) + pos_of(nu, ipow(2, l), p) / 2;
          if (par != pnu) continue;
          Tensor x = Gl[static_cast<size_t>(l)][static_cast<size_t>(t * ls.nin + nu)];
          std::vector<const Cx*> ptr;
          std::vector<i64> br, bc;
          for (int k = 0; k < d; ++k) {
            gather_blocks(1, l, t, nu, k, ptr, br, bc);
            x = mode_product_blockdiag(x, k, ptr, br, bc, true);
          }
          if (first) {
            acc = std::move(x);
            first = false;
          } else {
            for (size_t q = 0; q < acc.data.size(); ++q) acc.data[q] += x.data[q];
          }
        }
        Gl[static_cast<size_t>(l - 1)][static_cast<size_t>(it)] = std::move(acc);
      });
    } else {
      parallel_for(b.nmid, nthreads, [&](i64 t) {
        if (!own(t)) return;
        Tensor x = Gl[0][static_cast<size_t>(t)];
        std::vector<const Cx*> ptr;
        std::vector<i64> br, bc;
        for (int k = 0; k < d; ++k) {
          gather_blocks(1, 0, t, 0, k, ptr, br, bc);
          x = mode_product_blockdiag(x, k, ptr, br, bc, true);
        }
        const i64 tot = ipow(mid_sz, d) * nv;
        for (i64 f = 0; f < tot; ++f) {
          i64 rem = f, g = 0, stride = 1;
          for (int p = 0; p < d; ++p) {
            const i64 loc = rem % mid_sz;
            rem /= mid_sz;
            g += (pos_of(t, mpm, p) * mid_sz + loc) * stride;
            stride *= n;
          }
          g += rem * N;
          G[g] = x.data[static_cast<size_t>(f)];
        }
      });
    }
  }
}

// ------------------------------------------------------------ tucker_id
struct Tucker {
  int d = 0;
  std::vector<std::vector<i64>> skel;   // 2d lists (row modes then col modes), global
  std::vector<std::vector<Cx>> interp;  // 2d factors r_k x |range_k|
  std::vector<i64> ranks;
  std::vector<Cx> core;
  bool saturated = false;
};

// id.cpp:235-287
Tucker tucker_id(const Spec& sp, const std::vector<Range>& ranges, double tol, const Strategy& st, u64 seed) {
  const size_t d = static_cast<size_t>(sp.d);
  if (ranges.size() != 2 * d) throw std::invalid_argument("tucker_id: wrong mode count");
  Tucker out;
  out.d = sp.d;
  out.skel.resize(2 * d);
  out.interp.resize(2 * d);
  out.ranks.assign(2 * d, 0);
  i64 r_est = 8;
  for (size_t mode = 0; mode < 2 * d; ++mode) {
    const Range target = ranges[mode];
    ColumnID id;
    std::vector<i64> tl;
    for (i64 v = target.lo; v <= target.hi; ++v) tl.push_back(v);
    for (i64 attempt = 0;; ++attempt) {
      const i64 per_mode = st.q * r_est * (i64{1} << attempt);
      const u64 tags[3] = {0x1D, static_cast<u64>(mode), static_cast<u64>(attempt)};
      const u64 s = derive_seed(seed, tags, 3);
      auto lists = proxy_lists(ranges, mode, per_mode, st, s);
      lists[mode] = tl;
      i64 m = 0;
      std::vector<Cx> a = unfolding(sp, lists, mode, &m);
      id = column_id(std::move(a), m, static_cast<i64>(tl.size()), tol, -1, nullptr);
      if (!id.saturated || attempt >= st.max_retries) break;
    }
    out.saturated = out.saturated || id.saturated;
    out.ranks[mode] = id.rank;
    r_est = std::max(r_est, id.rank);
    for (auto v : id.skeleton) out.skel[mode].push_back(v + target.lo - 1);
    out.interp[mode] = std::move(id.interp);
  }
  // core = subtensor_at(row skeletons, col skeletons)
  i64 tot = 1;
  for (auto& s : out.skel) tot *= static_cast<i64>(s.size());
  out.core.resize(static_cast<size_t>(tot));
  i64 ii[6], jj[6];
  for (i64 f = 0; f < tot; ++f) {
    i64 rem = f;
    for (size_t p = 0; p < 2 * d; ++p) {
      const i64 e = static_cast<i64>(out.skel[p].size());
      const i64 v = out.skel[p][static_cast<size_t>(rem % e)];
      rem /= e;
      if (p < d) ii[p] = v;
      else jj[p - d] = v;
    }
    out.core[static_cast<size_t>(f)] = kernel_eval(sp, ii, jj);
  }
  return out;
}

void cx_out(const std::vector<Cx>& v, double* out) {
  for (size_t i = 0; i < v.size(); ++i) {
    out[2 * i] = v[i].real();
    out[2 * i + 1] = v[i].imag();
  }
}
std::vector<Cx> cx_in(const double* p, i64 n) {
  std::vector<Cx> v(static_cast<size_t>(n));
  for (i64 i = 0; i < n; ++i) v[static_cast<size_t>(i)] = Cx(p[2 * i], p[2 * i + 1]);
  return v;
}

Strategy strat(int mode, i64 q, i64 max_retries, i64 row_cap) {
  Strategy s;
  s.mode = mode;
  s.q = q;
  s.max_retries = max_retries;
  s.row_cap = row_cap;
  return s;
}

}  // namespace

#define GUARD_BEGIN try {
#define GUARD_END                    \
  }                                  \
  catch (const std::exception& e) {  \
    g_err = e.what();                \
    return -1;                       \
  }                                  \
  return 0;

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

u64 oracle_derive_seed(u64 seed, const u64* t, int nt) { return derive_seed(seed, t, nt); }

int oracle_select_proxies_count(i64 extent, i64 count, int mode, u64 seed, i64* out, i64* out_n) {
  GUARD_BEGIN
  auto l = select_proxies_count(extent, count, mode, seed);
  *out_n = static_cast<i64>(l.size());
  std::copy(l.begin(), l.end(), out);
  GUARD_END
}

int oracle_proxy_lists(int nr, const i64* lo, const i64* hi, int skip, i64 per_mode, int mode, i64 q, i64 row_cap,
                       u64 seed, i64* out_counts, i64* out_lists) {
  GUARD_BEGIN
  std::vector<Range> r(static_cast<size_t>(nr));
  for (int p = 0; p < nr; ++p) r[static_cast<size_t>(p)] = Range{lo[p], hi[p]};
  auto lists = proxy_lists(r, static_cast<size_t>(skip), per_mode, strat(mode, q, 3, row_cap), seed);
  i64 pos = 0;
  for (int p = 0; p < nr; ++p) {
    out_counts[p] = static_cast<i64>(lists[static_cast<size_t>(p)].size());
    for (auto v : lists[static_cast<size_t>(p)]) out_lists[pos++] = v;
  }
  GUARD_END
}

// column_id with full diagnostics.  forced_perm may be null; forced_rank < 0 = none.
int oracle_column_id(i64 m, i64 n, const double* a, double tol, i64 max_rank, const i64* forced_perm,
                     i64 forced_rank, double tie_eps, i64* rank, i64* skel, double* interp, i64* perm,
                     int* saturated, double* interp_max_abs, double* gaps /*[min_gap, rank_gap]*/, int* mismatch) {
  GUARD_BEGIN
  Replay rp;
  rp.perm = forced_perm;
  rp.rank = forced_rank;
  rp.tie_eps = tie_eps;
  const bool use = forced_perm != nullptr || forced_rank >= 0;
  ColumnID id = column_id(cx_in(a, m * n), m, n, tol, max_rank, use ? &rp : nullptr);
  *rank = id.rank;
  std::copy(id.skeleton.begin(), id.skeleton.end(), skel);
  cx_out(id.interp, interp);
  std::copy(id.perm.begin(), id.perm.end(), perm);
  *saturated = id.saturated;
  *interp_max_abs = id.interp_max_abs;
  gaps[0] = id.min_gap;
  gaps[1] = id.rank_gap;
  *mismatch = id.mismatch;
  GUARD_END
}

int oracle_kernel_eval(const int* si, const double* sf, i64 count, const i64* I, const i64* J, double* out) {
  GUARD_BEGIN
  Spec s = spec_from(si, sf);
  for (i64 e = 0; e < count; ++e) {
    const Cx v = kernel_eval(s, I + e * s.d, J + e * s.d);
    out[2 * e] = v.real();
    out[2 * e + 1] = v.imag();
  }
  GUARD_END
}

// Unfolding matrix of K over explicit per-mode lists (2d lists concatenated).
int oracle_unfolding(const int* si, const double* sf, const i64* counts, const i64* lists, int skip, double* out,
                     i64* m_out) {
  GUARD_BEGIN
  Spec s = spec_from(si, sf);
  std::vector<std::vector<i64>> l(static_cast<size_t>(2 * s.d));
  i64 pos = 0;
  for (int p = 0; p < 2 * s.d; ++p) {
    l[static_cast<size_t>(p)].assign(lists + pos, lists + pos + counts[p]);
    pos += counts[p];
  }
  auto a = unfolding(s, l, static_cast<size_t>(skip), m_out);
  cx_out(a, out);
  GUARD_END
}

int oracle_mode_product_blockdiag(int nmodes, const i64* shape, const double* t, int mode, int nb, const i64* br,
                                  const i64* bc, const double* blocks, int transpose, double* out) {
  GUARD_BEGIN
  Tensor x;
  x.shape.assign(shape, shape + nmodes);
  i64 tot = 1;
  for (auto e : x.shape) tot *= e;
  x.data = cx_in(t, tot);
  std::vector<std::vector<Cx>> mats;
  std::vector<const Cx*> ptr;
  std::vector<i64> vr(br, br + nb), vc(bc, bc + nb);
  i64 pos = 0;
  for (int b = 0; b < nb; ++b) {
    mats.push_back(cx_in(blocks + 2 * pos, br[b] * bc[b]));
    pos += br[b] * bc[b];
  }
  for (auto& m : mats) ptr.push_back(m.data());
  Tensor o = mode_product_blockdiag(x, mode - 1, ptr, vr, vc, transpose != 0);
  cx_out(o.data, out);
  GUARD_END
}

int oracle_tucker_id(const int* si, const double* sf, const i64* lo, const i64* hi, double tol, int mode, i64 q,
                     i64 max_retries, i64 row_cap, u64 seed, i64* ranks, i64* skel, double* interp, double* core) {
  GUARD_BEGIN
  Spec s = spec_from(si, sf);
  std::vector<Range> r(static_cast<size_t>(2 * s.d));
  for (int p = 0; p < 2 * s.d; ++p) r[static_cast<size_t>(p)] = Range{lo[p], hi[p]};
  Tucker t = tucker_id(s, r, tol, strat(mode, q, max_retries, row_cap), seed);
  i64 sp = 0, ip = 0;
  for (int m = 0; m < 2 * s.d; ++m) {
    ranks[m] = t.ranks[static_cast<size_t>(m)];
    for (auto v : t.skel[static_cast<size_t>(m)]) skel[sp++] = v;
    cx_out(t.interp[static_cast<size_t>(m)], interp + 2 * ip);
    ip += static_cast<i64>(t.interp[static_cast<size_t>(m)].size());
  }
  cx_out(t.core, core);
  GUARD_END
}

int oracle_level_rule(i64 n, i64 cb) { return level_rule(n, cb); }

// ---- butterfly handle API -------------------------------------------------
// replay (nullable): per global slot (V levels 0..Lc, then U levels 0..Lc),
// forced_rank[slot] (<0: none) and forced perms at perm_off[slot] into forced_perm.
int oracle_tbf_construct(const int* si, const double* sf, int L, double tol, int mode, i64 q, i64 max_retries,
                         i64 row_cap, u64 seed, int nthreads, const i64* forced_rank, const i64* perm_off,
                         const i64* forced_perm, double tie_eps, void** out) {
  GUARD_BEGIN
  auto b = std::make_unique<TBF>();
  b->spec = spec_from(si, sf);
  const i64 n = b->spec.n;
  if (L < 0 || L % 2 != 0) throw std::invalid_argument("tbf_construct: L must be even and >= 0");
  if ((n >> L) < 1 || (n % (i64{1} << L)) != 0) throw std::invalid_argument("tbf_construct: extent not C_b*2^L");
  b->L = L;
  b->Lc = L / 2;
  b->tol = tol;
  b->st = strat(mode, q, max_retries, row_cap);
  b->seed = seed;
  b->nmid = ipow(2, static_cast<i64>(b->spec.d) * b->Lc);
  i64 slot_base = 0;
  for (int sd = 0; sd < 2; ++sd) {
    b->side[sd].resize(static_cast<size_t>(b->Lc + 1));
    i64 r_est = 8;
    for (int l = 0; l <= b->Lc; ++l) {
      const LevelShape ls = level_shape(*b, l);
      std::vector<Replay> rps;
      std::vector<const Replay*> rpp;
      if (forced_rank) {
        rps.resize(static_cast<size_t>(ls.count));
        rpp.resize(static_cast<size_t>(ls.count));
        for (i64 i = 0; i < ls.count; ++i) {
          rps[static_cast<size_t>(i)].rank = forced_rank[slot_base + i];
          rps[static_cast<size_t>(i)].perm = forced_perm + perm_off[slot_base + i];
          rps[static_cast<size_t>(i)].tie_eps = tie_eps;
          rpp[static_cast<size_t>(i)] = forced_rank[slot_base + i] >= 0 ? &rps[static_cast<size_t>(i)] : nullptr;
        }
      }
      b->r_est[sd].push_back(r_est);
      // diagnostic (accuracy root-cause runs): ORACLE_DIAG_ALL="side:level,..."
      // builds the listed (side, level) batches with ProxyMode::All
      const Strategy keep = b->st;
      if (const char* dg = std::getenv("ORACLE_DIAG_ALL")) {
        const std::string tag = std::to_string(sd) + ":" + std::to_string(l);
        const std::string lst = std::string(",") + dg + ",";
        if (lst.find("," + tag + ",") != std::string::npos) b->st.mode = All;
      }
      build_level(*b, sd, l, r_est, nthreads, forced_rank ? rpp.data() : nullptr);
      b->st = keep;
      i64 mx = 0;
      for (const Slot& s : b->side[sd][static_cast<size_t>(l)]) mx = std::max(mx, s.rank);
      r_est = std::max(r_est, mx);  // level-synchronous running max
      slot_base += ls.count;
    }
  }
  build_cores(*b, nthreads);
  *out = b.release();
  GUARD_END
}

void oracle_tbf_free(void* h) { delete static_cast<TBF*>(h); }

// Build an oracle TBF from an exported factorization (e.g. the GPU's), so the
// CPU apply runs on exactly the same factors ("same factors" parity, and the
// CPU apply baseline without a CPU construction).  Layout as oracle_tbf_export.
int oracle_tbf_import(const int* si, const double* sf, int L, double tol, const i64* ranks, const i64* ncols,
                      const i64* skel, const double* interp, const double* cores, const i64* core_rows,
                      const i64* core_cols, void** out) {
  GUARD_BEGIN
  auto b = std::make_unique<TBF>();
  b->spec = spec_from(si, sf);
  b->L = L;
  b->Lc = L / 2;
  b->tol = tol;
  b->nmid = ipow(2, static_cast<i64>(b->spec.d) * b->Lc);
  i64 g = 0, sk = 0, ip = 0;
  for (int sd = 0; sd < 2; ++sd) {
    b->side[sd].resize(static_cast<size_t>(b->Lc + 1));
    for (int l = 0; l <= b->Lc; ++l) {
      const LevelShape ls = level_shape(*b, l);
      auto& lv = b->side[sd][static_cast<size_t>(l)];
      lv.resize(static_cast<size_t>(ls.count));
      for (auto& s : lv) {
        s.rank = ranks[g];
        s.ncols = ncols[g];
        s.skel.assign(skel + sk, skel + sk + s.rank);
        s.interp = cx_in(interp + 2 * ip, s.rank * s.ncols);
        sk += s.rank;
        ip += s.rank * s.ncols;
        ++g;
      }
    }
  }
  const i64 P = b->nmid * b->nmid;
  b->cores.resize(static_cast<size_t>(P));
  b->core_rows.assign(core_rows, core_rows + P);
  b->core_cols.assign(core_cols, core_cols + P);
  i64 co = 0;
  for (i64 p = 0; p < P; ++p) {
    const i64 sz = core_rows[p] * core_cols[p];
    b->cores[static_cast<size_t>(p)] = cx_in(cores + 2 * co, sz);
    co += sz;
  }
  *out = b.release();
  GUARD_END
}

// info[0..]: d, n, L, Lc, nmid, total_slots, total_skel, total_interp, total_core, total_perm
int oracle_tbf_info(void* h, i64* info) {
  GUARD_BEGIN
  const TBF& b = *static_cast<TBF*>(h);
  i64 slots = 0, sk = 0, ip = 0, co = 0, pm = 0;
  for (int sd = 0; sd < 2; ++sd)
    for (auto& lv : b.side[sd])
      for (auto& s : lv) {
        ++slots;
        sk += s.rank;
        ip += s.rank * s.ncols;
        pm += s.ncols;
      }
  for (auto& c : b.cores) co += static_cast<i64>(c.size());
  info[0] = b.spec.d;
  info[1] = b.spec.n;
  info[2] = b.L;
  info[3] = b.Lc;
  info[4] = b.nmid;
  info[5] = slots;
  info[6] = sk;
  info[7] = ip;
  info[8] = co;
  info[9] = pm;
  GUARD_END
}

// Flat export in canonical slot order (V l=0..Lc, then U l=0..Lc).
// per slot: ranks, ncols, rows, gaps[2], flags (bit0 saturated, bit1 mismatch);
// skel / interp / perm concatenated; cores concatenated (pair p = s*nmid+t,
// col-major), core_rows/core_cols per pair; r_est[2*(Lc+1)].
int oracle_tbf_export(void* h, i64* ranks, i64* ncols, i64* rows, double* gaps, int* flags, i64* skel,
                      double* interp, i64* perm, double* cores, i64* core_rows, i64* core_cols, i64* r_est) {
  GUARD_BEGIN
  const TBF& b = *static_cast<TBF*>(h);
  i64 si = 0, sk = 0, ip = 0, pm = 0;
  for (int sd = 0; sd < 2; ++sd)
    for (auto& lv : b.side[sd])
      for (auto& s : lv) {
        ranks[si] = s.rank;
        ncols[si] = s.ncols;
        rows[si] = s.rows;
        gaps[2 * si] = s.min_gap;
        gaps[2 * si + 1] = s.rank_gap;
        flags[si] = (s.saturated ? 1 : 0) | (s.mismatch ? 2 : 0);
        for (auto v : s.skel) skel[sk++] = v;
        cx_out(s.interp, interp + 2 * ip);
        ip += static_cast<i64>(s.interp.size());
        for (auto v : s.perm) perm[pm++] = v;
        ++si;
      }
  i64 co = 0;
  for (size_t p = 0; p < b.cores.size(); ++p) {
    cx_out(b.cores[p], cores + 2 * co);
    co += static_cast<i64>(b.cores[p].size());
    core_rows[p] = b.core_rows[p];
    core_cols[p] = b.core_cols[p];
  }
  i64 q = 0;
  for (int sd = 0; sd < 2; ++sd)
    for (auto v : b.r_est[sd]) r_est[q++] = v;
  GUARD_END
}

// memory breakdown in bytes: V, W, U, P, cores
int oracle_tbf_memory(void* h, i64* out) {
  GUARD_BEGIN
  const TBF& b = *static_cast<TBF*>(h);
  for (int i = 0; i < 5; ++i) out[i] = 0;
  for (int sd = 0; sd < 2; ++sd)
    for (size_t l = 0; l < b.side[sd].size(); ++l)
      for (auto& s : b.side[sd][l]) out[(sd == 0 ? 0 : 2) + (l > 0 ? 1 : 0)] += s.rank * s.ncols * 16;
  for (auto& c : b.cores) out[4] += static_cast<i64>(c.size()) * 16;
  GUARD_END
}

int oracle_tbf_contract(void* h, const double* F, double* G, i64 nv, int nthreads) {
  GUARD_BEGIN
  const TBF& b = *static_cast<TBF*>(h);
  const i64 N = ipow(b.spec.n, b.spec.d) * nv;
  std::vector<Cx> f = cx_in(F, N), g(static_cast<size_t>(N));
  tbf_contract(b, f.data(), g.data(), nv, nthreads);
  cx_out(g, G);
  GUARD_END
}

// Sharded apply phases (test backend for paper_2411_03029_b200/sharded.py).
int oracle_tbf_contract_phase_owned(void* h, int phase, int rank, int world, const int* owner, const double* in,
                                    double* out, const i64* send_off, const i64* recv_off, i64 send_elems,
                                    i64 recv_elems, i64 nv, int nthreads);
int oracle_tbf_contract_phase(void* h, int phase, int rank, int world, const double* in, double* out,
                              const i64* send_off, const i64* recv_off, i64 send_elems, i64 recv_elems, i64 nv,
                              int nthreads) {
  return oracle_tbf_contract_phase_owned(h, phase, rank, world, nullptr, in, out, send_off, recv_off, send_elems,
                                         recv_elems, nv, nthreads);
}

// owner: ownership map of the middle multi-sets (nmid ints in [0, world)), or null for index % world
int oracle_tbf_contract_phase_owned(void* h, int phase, int rank, int world, const int* owner, const double* in,
                                    double* out, const i64* send_off, const i64* recv_off, i64 send_elems,
                                    i64 recv_elems, i64 nv, int nthreads) {
  GUARD_BEGIN
  const TBF& b = *static_cast<TBF*>(h);
  const i64 N = ipow(b.spec.n, b.spec.d) * nv;
  ShardIO io;
  io.phase = phase;
  io.rank = rank;
  io.world = world;
  io.owner = owner;
  io.send_off = send_off;
  io.recv_off = recv_off;
  if (phase == 1) {
    std::vector<Cx> f = cx_in(in, N), snd(static_cast<size_t>(std::max<i64>(send_elems * nv, 1)));
    io.send = snd.data();
    tbf_contract(b, f.data(), nullptr, nv, nthreads, &io);
    cx_out(snd, out);
  } else {
    std::vector<Cx> rcv = cx_in(in, std::max<i64>(recv_elems * nv, 1)), g = cx_in(out, N);
    io.recv = rcv.data();
    tbf_contract(b, nullptr, g.data(), nv, nthreads, &io);
    cx_out(g, out);
  }
  GUARD_END
}

// Direct dense sums G(i, v) = sum_j K(i, j) F(j, v) at sampled output flat
// indices (first-mode-fastest over n^d), Neumaier-compensated.
int oracle_dense_rows(const int* si, const double* sf, const double* F, i64 nv, i64 nrows, const i64* rows_flat,
                      double* out, int nthreads) {
  GUARD_BEGIN
  Spec s = spec_from(si, sf);
  const i64 N = ipow(s.n, s.d);
  parallel_for(nrows, nthreads, [&](i64 r) {
    i64 ii[6], jj[6];
    i64 rem = rows_flat[r];
    for (int p = 0; p < s.d; ++p) {
      ii[p] = rem % s.n + 1;
      rem /= s.n;
    }
    for (i64 v = 0; v < nv; ++v) {
      double sr = 0, si_ = 0, cr = 0, ci = 0;
      for (i64 f = 0; f < N; ++f) {
        i64 rr = f;
        for (int p = 0; p < s.d; ++p) {
          jj[p] = rr % s.n + 1;
          rr /= s.n;
        }
        const Cx k = kernel_eval(s, ii, jj);
        const Cx x(F[2 * (f + v * N)], F[2 * (f + v * N) + 1]);
        const Cx pr = k * x;
        double t = sr + pr.real();
        cr += std::fabs(sr) >= std::fabs(pr.real()) ? (sr - t) + pr.real() : (pr.real() - t) + sr;
        sr = t;
        t = si_ + pr.imag();
        ci += std::fabs(si_) >= std::fabs(pr.imag()) ? (si_ - t) + pr.imag() : (pr.imag() - t) + si_;
        si_ = t;
      }
      out[2 * (r + v * nrows)] = sr + cr;
      out[2 * (r + v * nrows) + 1] = si_ + ci;
    }
  });
  GUARD_END
}

}  // extern "C"
