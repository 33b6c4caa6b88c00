// Batched interpolative decompositions for one (side, level) of the butterfly
// construction (Alg. 1; reference primitives id.cpp:24-130,199-231,
// tensor.cpp:249-266).  Per ID slot:
//   k_gen_proxies  proxy index lists, bit-exact with id.cpp:199-231 (device)
//   k_targets      candidate columns: leaf range (l=0) or children skeletons
//   k_panel        entry generation fused with a TSQR: each CTA streams a row
//                  partition of the proxy unfolding through shared memory in
//                  panels and folds it into a w x w triangular factor with
//                  Householder reflections (no HBM copy of the ID matrix)
//   k_finish       combines the partition factors, then runs the reference's
//                  column-pivoted QR (id.cpp:24-85) on the w x w R -- column
//                  residual norms of R equal those of A (Q unitary) -- with the
//                  1e-12 tie rule of SURVEY App. A7, and id_from_qrcp
//                  (id.cpp:87-120): T = R11^{-1} R12, sorted skeleton, interp.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "kernels.h"

namespace tbf {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__global__ void k_gen_proxies(LevelDesc L, int* __restrict__ proxies) {
  const i64 tid = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int D = 2 * L.d;
  if (tid >= L.nslots * D) return;
  const i64 slot = tid / D;
  const int p = static_cast<int>(tid % D);
  const SlotPos s = decode_slot(L, slot);
  if (p == s.skip || !owns_outer(L, s.outer)) return;
  const u64 tags[7] = {L.side_tag, static_cast<u64>(L.l), static_cast<u64>(s.outer), static_cast<u64>(s.inner),
                       static_cast<u64>(s.k), static_cast<u64>(s.j), 0ULL};
  const u64 sseed = derive_seed(L.seed, tags, 7);
  const u64 ptags[2] = {0x70ULL, static_cast<u64>(p)};
  const u64 pseed = derive_seed(sseed, ptags, 2);
  int* out = proxies + slot * L.psize + L.poff[s.k][p];
  if (L.proxy_mode == OIOBF_PROXY_UNIFORM_RANDOM && L.counts[s.k][p] > kMaxProxy) return;  // k_gen_proxies_big
  const i64 cnt = select_proxies(s.sz[p], L.counts[s.k][p], L.proxy_mode, pseed, out);
  (void)cnt;
  for (int q = 0; q < L.counts[s.k][p]; ++q) out[q] += static_cast<int>(s.lo[p] - 1);
}

// UniformRandom lists longer than kMaxProxy: one 32-thread CTA per (slot,
// mode) runs the reference's partial Fisher-Yates (id.cpp:171-181) on a full
// pool in shared memory (extent ints), then writes the chosen values in
// ascending order (the sort of id.cpp:180) by scanning a membership bitmap.
__global__ void k_gen_proxies_big(LevelDesc L, int* __restrict__ proxies) {
  extern __shared__ int pool[];  // extent ints, then extent flag bytes
  const int D = 2 * L.d;
  const i64 slot = blockIdx.x / D;
  const int p = static_cast<int>(blockIdx.x % D);
  const SlotPos s = decode_slot(L, slot);
  const int cnt = L.counts[s.k][p];
  if (p == s.skip || !owns_outer(L, s.outer) || cnt <= kMaxProxy) return;
  const i64 extent = s.sz[p];
  unsigned char* flag = reinterpret_cast<unsigned char*>(pool + extent);
  for (i64 i = threadIdx.x; i < extent; i += blockDim.x) {
    pool[i] = static_cast<int>(i + 1);
    flag[i] = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const u64 tags[7] = {L.side_tag, static_cast<u64>(L.l), static_cast<u64>(s.outer), static_cast<u64>(s.inner),
                         static_cast<u64>(s.k), static_cast<u64>(s.j), 0ULL};
    const u64 sseed = derive_seed(L.seed, tags, 7);
    const u64 ptags[2] = {0x70ULL, static_cast<u64>(p)};
    u64 st = derive_seed(sseed, ptags, 2);
    for (i64 i = 0; i < cnt; ++i) {
      const i64 j = i + static_cast<i64>(splitmix_bounded(st, static_cast<u64>(extent - i)));
      const int t = pool[i];
      pool[i] = pool[j];
      pool[j] = t;
    }
  }
  __syncthreads();
  for (i64 i = threadIdx.x; i < cnt; i += blockDim.x) flag[pool[i] - 1] = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    int* out = proxies + slot * L.psize + L.poff[s.k][p];
    const int shift = static_cast<int>(s.lo[p] - 1);
    int q = 0;
    for (i64 v = 0; v < extent; ++v)
      if (flag[v]) out[q++] = static_cast<int>(v + 1) + shift;
  }
}

// one warp per slot
__global__ void k_targets(LevelDesc L, const int* __restrict__ crank, const i64* __restrict__ cskel_off,
                          const int* __restrict__ cskel, int* __restrict__ targets, int* __restrict__ width) {
  const i64 slot = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (slot >= L.nslots) return;
  const SlotPos s = decode_slot(L, slot);
  int* out = targets + slot * L.wmax;
  if (!owns_outer(L, s.outer)) {  // another rank's slot: empty candidate set
    if (lane == 0) width[slot] = 0;
    return;
  }
  if (L.l == 0) {
    for (i64 c = lane; c < s.sz[s.skip]; c += 32) out[c] = static_cast<int>(s.lo[s.skip] + c);
    if (lane == 0) width[slot] = static_cast<int>(s.sz[s.skip]);
    return;
  }
  const i64 c0 = child_slot(L, s, 0), c1 = child_slot(L, s, 1);
  const int r0 = crank[c0], r1 = crank[c1];
  for (int c = lane; c < r0; c += 32) out[c] = cskel[cskel_off[c0] + c];
  for (int c = lane; c < r1; c += 32) out[r0 + c] = cskel[cskel_off[c1] + c];
  if (lane == 0) width[slot] = r0 + r1;
}

// Fold panel X (nrows x w, col-major, ld pr) into upper-triangular R (w x w,
// col-major, ld w) with Householder reflections.  Column k is owned by warp
// k % kWarps for the whole panel, so one __syncthreads per column suffices.
// Reflector for x = [alpha; X(:, j)] (sig = |X(:, j)|^2 > 0) in the normalised
// form v = [1; X(:, j) * scale], scale = 1 / (alpha + sign * |x|), tau in [1, 2]:
// |v_i| <= 1, so nothing overflows when sig is tiny (a panel whose rows are
// exhausted leaves only rounding noise in its trailing columns; the textbook
// beta = 2 / (|v0|^2 + sig) overflows there and poisons R with Inf*0).
struct Bcast {
  double2 scale;
  double tau;
  int active;
};

// The reflector set-up is on the critical path of every column step (the
// other warps wait for it at the step's barrier), so it is written with two
// reciprocal square roots and one reciprocal instead of two square roots and
// five IEEE divisions.  With sign = alpha / |alpha| and s = |alpha| + |x|:
// v0 = alpha + sign |x| = sign s, so scale = 1 / v0 = conj(sign) / s, and
// tau = 2 / (1 + sig / s^2) = 2 s^2 / (2 |x| s) = 1 + |alpha| / |x|
// (|x|^2 = |alpha|^2 + sig) -- the same reflector, a few ulps apart.
__device__ __forceinline__ Bcast make_reflector(double2 alpha, double sig, double2* rjj) {
  Bcast b;
  if (!(sig > 0)) {
    b.scale = make_double2(0, 0);
    b.tau = 0;
    b.active = 0;
    return b;
  }
  const double a2 = cnorm2(alpha);
  const double x2 = a2 + sig;
  const double rx = rsqrt(x2);
  const double xnorm = x2 * rx;
  double aa = 0;
  double2 sign = make_double2(1, 0);
  if (a2 > 0) {
    const double ra = rsqrt(a2);
    aa = a2 * ra;
    sign = make_double2(alpha.x * ra, alpha.y * ra);
  }
  const double inv = __drcp_rn(aa + xnorm);
  b.scale = make_double2(sign.x * inv, -sign.y * inv);
  b.tau = fma(aa, rx, 1.0);
  b.active = 1;
  *rjj = make_double2(-sign.x * xnorm, -sign.y * xnorm);
  return b;
}

// apply H = I - tau v v^H (v0 = 1) to the column pair (r = R(j, k), X(:, k)):
// s = r + conj(scale) * sum conj(X_ij) X_ik ; r -= tau s ; X_ik -= X_ij * scale * tau s
__device__ __forceinline__ double2 reflect_coeff(const Bcast& b, double2 r, double2 dot) {
  double2 s = r;
  cfmac(s, b.scale, dot);  // + conj(scale) * dot
  return cscale(b.tau, s);
}

// Column k is owned by warp k % kWarps for the whole panel.  Look-ahead: the
// owner of column j+1 updates that column first in step j and immediately
// builds reflector j+1 into the other broadcast slot, so its norm reduction
// and reflector set-up overlap the other warps' updates of step j (one
// __syncthreads per column; the critical path no longer stalls every warp on
// a single warp's reduction).
// R (w x w upper triangular) is kept packed column by column in shared
// memory: element (j, k), j <= k, at k (k + 1) / 2 + j -- half the footprint
// of a full w x w array, which leaves room for taller row panels.
__device__ __forceinline__ int rpk(int j, int k) { return k * (k + 1) / 2 + j; }

__device__ __forceinline__ void panel_reflector(double2* __restrict__ R, const double2* __restrict__ X, int w, int j,
                                                int nrows, int pr, Bcast* slot) {
  const int lane = threadIdx.x & 31;
  double sig = 0;
  for (int i = lane; i < nrows; i += 32) sig += cnorm2(X[i + j * pr]);
  sig = warp_sum(sig);
  if (lane == 0) *slot = make_reflector(R[rpk(j, j)], sig, &R[rpk(j, j)]);
  __syncwarp();
}

// apply reflector j (broadcast b) to trailing column k: R(j, k) and X(:, k)
__device__ __forceinline__ void reflect_col(const Bcast& b, double2* __restrict__ R, double2* __restrict__ X, int j,
                                            int k, int nrows, int pr, int lane) {
  double2 da = make_double2(0, 0), db = make_double2(0, 0);  // even / odd row blocks (shorter chains)
  for (int i = lane, r = 0; i < nrows; i += 32, ++r) cfmac((r & 1) ? db : da, X[i + j * pr], X[i + k * pr]);
  const double2 dot = warp_sum2(cadd(da, db));
  const double2 ws = reflect_coeff(b, R[rpk(j, k)], dot);
  const double2 t = cmul(b.scale, ws);
  if (lane == 0) R[rpk(j, k)] = csub(R[rpk(j, k)], ws);
  for (int i = lane; i < nrows; i += 32) X[i + k * pr] = csub(X[i + k * pr], cmul(X[i + j * pr], t));
}

// look-ahead column k = j + 1: apply reflector j, accumulate the updated
// column's norm in the same pass, and build reflector k into `slot`
// (replaces reflect_col + panel_reflector: one read of the column, and the
// norm reduction starts as soon as the update is done)
__device__ __forceinline__ void reflect_col_next(const Bcast& b, double2* __restrict__ R, double2* __restrict__ X,
                                                 int j, int k, int nrows, int pr, int lane, Bcast* slot) {
  double2 da = make_double2(0, 0), db = make_double2(0, 0);
  for (int i = lane, r = 0; i < nrows; i += 32, ++r) cfmac((r & 1) ? db : da, X[i + j * pr], X[i + k * pr]);
  const double2 rjk = R[rpk(j, k)];
  const double2 dot = warp_sum2(cadd(da, db));
  const double2 ws = reflect_coeff(b, rjk, dot);
  const double2 t = cmul(b.scale, ws);
  double sig = 0;
  for (int i = lane; i < nrows; i += 32) {
    const double2 x = csub(X[i + k * pr], cmul(X[i + j * pr], t));
    X[i + k * pr] = x;
    sig += cnorm2(x);
  }
  sig = warp_sum(sig);
  if (lane == 0) {
    R[rpk(j, k)] = csub(rjk, ws);
    *slot = make_reflector(R[rpk(k, k)], sig, &R[rpk(k, k)]);
  }
  __syncwarp();
}

// two columns at once: the two dot products and shuffle reductions interleave
// (independent dependency chains), halving the per-step latency of wide panels
__device__ __forceinline__ void reflect_col2(const Bcast& b, double2* __restrict__ R, double2* __restrict__ X, int j,
                                             int k1, int k2, int nrows, int pr, int lane) {
  double2 d1 = make_double2(0, 0), d2 = make_double2(0, 0), e1 = make_double2(0, 0), e2 = make_double2(0, 0);
  for (int i = lane, r = 0; i < nrows; i += 32, ++r) {
    const double2 xj = X[i + j * pr];
    cfmac((r & 1) ? e1 : d1, xj, X[i + k1 * pr]);
    cfmac((r & 1) ? e2 : d2, xj, X[i + k2 * pr]);
  }
  d1 = cadd(d1, e1);
  d2 = cadd(d2, e2);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    d1.x += __shfl_xor_sync(0xffffffffu, d1.x, o);
    d1.y += __shfl_xor_sync(0xffffffffu, d1.y, o);
    d2.x += __shfl_xor_sync(0xffffffffu, d2.x, o);
    d2.y += __shfl_xor_sync(0xffffffffu, d2.y, o);
  }
  const double2 w1 = reflect_coeff(b, R[rpk(j, k1)], d1), w2 = reflect_coeff(b, R[rpk(j, k2)], d2);
  const double2 t1 = cmul(b.scale, w1), t2 = cmul(b.scale, w2);
  if (lane == 0) {
    R[rpk(j, k1)] = csub(R[rpk(j, k1)], w1);
    R[rpk(j, k2)] = csub(R[rpk(j, k2)], w2);
  }
  for (int i = lane; i < nrows; i += 32) {
    const double2 xj = X[i + j * pr];
    X[i + k1 * pr] = csub(X[i + k1 * pr], cmul(xj, t1));
    X[i + k2 * pr] = csub(X[i + k2 * pr], cmul(xj, t2));
  }
}

// Register-cached variants (RPL = rows per lane = panel rows / 32, compile
// time): the reflector column X(:, j) is loaded into registers once per step
// and each updated column once per pair -- the same operations in the same
// order as reflect_col / reflect_col2 (bit-identical results) with about half
// the instructions; the absorb is 93-98% of the construction time.
template <int RPL>
__device__ __forceinline__ void reflect_col_r(const Bcast& b, double2* __restrict__ R, double2* __restrict__ X,
                                              const double2 (&xj)[RPL], int j, int k, int nrows, int pr, int lane) {
  double2 xk[RPL];
  double2 da = make_double2(0, 0), db = make_double2(0, 0);
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int i = lane + 32 * r;
    xk[r] = X[i + k * pr];
    cfmac((r & 1) ? db : da, xj[r], xk[r]);
  }
  const double2 dot = warp_sum2(cadd(da, db));
  const double2 ws = reflect_coeff(b, R[rpk(j, k)], dot);
  const double2 t = cmul(b.scale, ws);
  if (lane == 0) R[rpk(j, k)] = csub(R[rpk(j, k)], ws);
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int i = lane + 32 * r;
    X[i + k * pr] = csub(xk[r], cmul(xj[r], t));
  }
}

template <int RPL>
__device__ __forceinline__ void reflect_col_next_r(const Bcast& b, double2* __restrict__ R, double2* __restrict__ X,
                                                   const double2 (&xj)[RPL], int j, int k, int pr, int lane,
                                                   Bcast* slot) {
  double2 xk[RPL];
  double2 da = make_double2(0, 0), db = make_double2(0, 0);
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int i = lane + 32 * r;
    xk[r] = X[i + k * pr];
    cfmac((r & 1) ? db : da, xj[r], xk[r]);
  }
  const double2 rjk = R[rpk(j, k)];
  const double2 dot = warp_sum2(cadd(da, db));
  const double2 ws = reflect_coeff(b, rjk, dot);
  const double2 t = cmul(b.scale, ws);
  double sig = 0;
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int i = lane + 32 * r;
    xk[r] = csub(xk[r], cmul(xj[r], t));
    X[i + k * pr] = xk[r];
    sig += cnorm2(xk[r]);
  }
  sig = warp_sum(sig);
  if (lane == 0) {
    R[rpk(j, k)] = csub(rjk, ws);
    *slot = make_reflector(R[rpk(k, k)], sig, &R[rpk(k, k)]);
  }
  __syncwarp();
}

template <int RPL>
__device__ __forceinline__ void reflect_col2_r(const Bcast& b, double2* __restrict__ R, double2* __restrict__ X,
                                               const double2 (&xj)[RPL], int j, int k1, int k2, int nrows, int pr,
                                               int lane) {
  double2 x1[RPL], x2[RPL];
  double2 d1 = make_double2(0, 0), d2 = make_double2(0, 0), e1 = make_double2(0, 0), e2 = make_double2(0, 0);
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int i = lane + 32 * r;
    x1[r] = X[i + k1 * pr];
    x2[r] = X[i + k2 * pr];
    cfmac((r & 1) ? e1 : d1, xj[r], x1[r]);
    cfmac((r & 1) ? e2 : d2, xj[r], x2[r]);
  }
  d1 = cadd(d1, e1);
  d2 = cadd(d2, e2);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    d1.x += __shfl_xor_sync(0xffffffffu, d1.x, o);
    d1.y += __shfl_xor_sync(0xffffffffu, d1.y, o);
    d2.x += __shfl_xor_sync(0xffffffffu, d2.x, o);
    d2.y += __shfl_xor_sync(0xffffffffu, d2.y, o);
  }
  const double2 w1 = reflect_coeff(b, R[rpk(j, k1)], d1), w2 = reflect_coeff(b, R[rpk(j, k2)], d2);
  const double2 t1 = cmul(b.scale, w1), t2 = cmul(b.scale, w2);
  if (lane == 0) {
    R[rpk(j, k1)] = csub(R[rpk(j, k1)], w1);
    R[rpk(j, k2)] = csub(R[rpk(j, k2)], w2);
  }
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int i = lane + 32 * r;
    X[i + k1 * pr] = csub(x1[r], cmul(xj[r], t1));
    X[i + k2 * pr] = csub(x2[r], cmul(xj[r], t2));
  }
}

// `hook(j, owns_next)` runs at the end of column step j, before its barrier
// (the pipelined panel kernel generates entries of the NEXT panel there, into
// columns of X that are already dead)
template <int NW, int RPL, class Hook>
__device__ void absorb_panel_r(double2* __restrict__ R, double2* __restrict__ X, int w, int nrows, int pr,
                               Bcast* bc, Hook hook) {
  constexpr int kWarps = NW;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) panel_reflector(R, X, w, 0, nrows, pr, &bc[0]);
  __syncthreads();
  for (int j = 0; j < w; ++j) {
    const Bcast b = bc[j & 1];
    const bool owns_next = j + 1 < w && warp == (j + 1) % kWarps;
    int k = j + 1 + ((warp - (j + 1) % kWarps) % kWarps + kWarps) % kWarps;
    if (b.active) {
      if (k < w) {
        double2 xj[RPL];  // reflector column j, this lane's rows
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const int i = lane + 32 * r;
          xj[r] = X[i + j * pr];
        }
        if (owns_next) {  // look-ahead column first, then its reflector
          reflect_col_next_r<RPL>(b, R, X, xj, j, k, pr, lane, &bc[(j + 1) & 1]);
          k += kWarps;
        }
        if constexpr (RPL >= 8 || (NW <= 8 && RPL >= 4)) {  // one column at a time (two would spill)
          for (; k < w; k += kWarps) reflect_col_r<RPL>(b, R, X, xj, j, k, nrows, pr, lane);
        } else {
          for (; k + kWarps < w; k += 2 * kWarps) reflect_col2_r<RPL>(b, R, X, xj, j, k, k + kWarps, nrows, pr, lane);
          if (k < w) reflect_col_r<RPL>(b, R, X, xj, j, k, nrows, pr, lane);
        }
      }
    } else if (owns_next) {
      panel_reflector(R, X, w, j + 1, nrows, pr, &bc[(j + 1) & 1]);
    }
    hook(j, owns_next);
    __syncthreads();
  }
}

template <int NW, class Hook>  // warps in the CTA (columns are owned round-robin)
__device__ void absorb_panel(double2* __restrict__ R, double2* __restrict__ X, int w, int nrows, int pr,
                             Bcast* bc, Hook hook) {
  constexpr int kWarps = NW;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) panel_reflector(R, X, w, 0, nrows, pr, &bc[0]);
  __syncthreads();
  for (int j = 0; j < w; ++j) {
    const Bcast b = bc[j & 1];
    const bool owns_next = j + 1 < w && warp == (j + 1) % kWarps;
    int k = j + 1 + ((warp - (j + 1) % kWarps) % kWarps + kWarps) % kWarps;
    if (b.active) {
      if (owns_next) {  // look-ahead column first, then its reflector
        reflect_col_next(b, R, X, j, k, nrows, pr, lane, &bc[(j + 1) & 1]);
        k += kWarps;
      }
      for (; k + kWarps < w; k += 2 * kWarps) reflect_col2(b, R, X, j, k, k + kWarps, nrows, pr, lane);
      if (k < w) reflect_col(b, R, X, j, k, nrows, pr, lane);
    } else if (owns_next) {
      panel_reflector(R, X, w, j + 1, nrows, pr, &bc[(j + 1) & 1]);
    }
    hook(j, owns_next);
    __syncthreads();
  }
}

// NT threads: 256, or 512 for wide IDs (w > 32, one CTA per SM by shared
// memory) so each column step spreads over 16 warps
// DIAG (timing diagnostics only, OIOBF_PANEL_DIAG): 1 = entry generation
// alone (no absorb), 2 = absorb alone (cheap synthetic entries)
// PIPE (Green kernel, one thread per panel row, register-cached absorb): the
// entries of panel p + 1 are generated inside the column steps of panel p --
// a thread produces its row's entry of column c once that column of X is dead
// (step c's barrier has passed), up to two per step, skipping the steps in
// which its warp builds the next reflector -- so the FP64-heavy generation
// fills the latency bubbles of the barrier-bound absorb instead of running
// between absorbs.  Same entries, same absorb order: bit-identical R.
template <int NT, int RPL, int MINB = (NT >= 512 ? 1 : (RPL >= 8 ? 2 : 3)), int DIAG = 0, int PIPE = 0>  // RPL: panel rows / 32
__global__ void __launch_bounds__(NT, MINB) k_panel(LevelDesc L, KSpec ks, const int* __restrict__ proxies,
                                                    const int* __restrict__ targets, const int* __restrict__ width,
                                                    double2* __restrict__ rpart) {
  extern __shared__ __align__(16) unsigned char smem[];
  const i64 slot = blockIdx.x / L.nparts;
  const i64 part = blockIdx.x % L.nparts;
  const int w = width[slot];
  const int pr = L.pr;
  double2* R = reinterpret_cast<double2*>(smem);  // packed upper triangle
  double2* X = R + L.wmax * (L.wmax + 1) / 2;
  Bcast* bc = reinterpret_cast<Bcast*>(X + static_cast<i64>(pr) * L.wmax);
  int* sprox = reinterpret_cast<int*>(bc + 2);
  int* stgt = sprox + L.psize;
  // Radon 2D, columns over a target mode: sin / cos(2 pi x) of each candidate
  double* csin = reinterpret_cast<double*>(reinterpret_cast<uintptr_t>(stgt + L.wmax + 1) & ~uintptr_t{7});
  double* ccos = csin + L.wmax;
  const int sk_k = static_cast<int>((slot / L.nj) % L.d);  // unfolded mode k of the slot (decode_slot)
  const int sk = (L.side == 0 ? L.d : 0) + sk_k;
  const int D = 2 * L.d;
  for (int i = threadIdx.x; i < L.psize; i += NT) sprox[i] = proxies[slot * L.psize + i];
  for (int i = threadIdx.x; i < w; i += NT) {
    const int t = targets[slot * L.wmax + i];
    stgt[i] = t;
    if (ks.kind == OIOBF_KERNEL_RADON2D && sk < L.d) {
      double sn, cs;
      sincos(__dmul_rn(2.0 * M_PI, __ddiv_rn(static_cast<double>(t - 1), static_cast<double>(ks.n))), &sn, &cs);
      csin[i] = sn;
      ccos[i] = cs;
    } else if (ks.kind == OIOBF_KERNEL_GREEN) {  // the candidate's coordinate along the unfolded mode
      csin[i] = sk < L.d ? green_x(ks, t) : green_y(ks, sk - L.d, t);
    }
  }
  for (int i = threadIdx.x; i < w * (w + 1) / 2; i += NT) R[i] = make_double2(0, 0);
  int cnt[kMaxModes], off[kMaxModes];
  for (int p = 0; p < D; ++p) {
    cnt[p] = L.counts[sk_k][p];
    off[p] = L.poff[sk_k][p];
  }
  __syncthreads();
  if (w == 0) return;
  const i64 r_begin = part * L.rpp;
  i64 r_end = r_begin + L.rpp;
  if (r_end > L.m) r_end = L.m;
  const int ncg = NT / pr;  // column groups per row
  const int my_row = threadIdx.x % pr, my_cg = threadIdx.x / pr;
  double diag_acc = 0;
  if constexpr (PIPE && RPL > 0 && DIAG == 0) {
    // (host: Green kernel, pr == NT -- thread = panel row, all w columns)
    const bool tgt = sk < L.d;
    const int q = tgt ? sk : sk - L.d;
    // row-invariant coordinates of panel row `row` (kernel_entry's operations)
    auto row_coords = [&](i64 row, double* xs, double* ys) {
      int ii[kMaxD], jj[kMaxD];
      i64 rem = row;
      for (int p = 0; p < D; ++p) {
        if (p == sk) continue;
        const int c = cnt[p];
        const int v = sprox[off[p] + static_cast<int>(rem % c)];
        rem /= c;
        if (p < L.d) ii[p] = v;
        else jj[p - L.d] = v;
      }
      xs[0] = xs[1] = xs[2] = 0;
      ys[0] = ks.off0;
      ys[1] = ks.off1;
      ys[2] = ks.off2;
#pragma unroll
      for (int p = 0; p < 3; ++p)
        if (p < L.d) {
          if (p != sk) xs[p] = green_x(ks, ii[p]);
          if (p + L.d != sk) ys[p] = green_y(ks, p, jj[p]);
        }
    };
    auto entry = [&](int c, const double* xs, const double* ys) {
      const double v = csin[c];  // green_x / green_y of the candidate (hoisted per column)
      double xc[3], yc[3];
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        xc[p] = (tgt && p == q) ? v : xs[p];
        yc[p] = (!tgt && p == q) ? v : ys[p];
      }
      return green_from_coords_rcp(ks, xc, yc);
    };
    const int row_t = threadIdx.x;  // pr == NT
    double xs[3], ys[3];
    {  // first panel: all columns up front
      const bool valid = r_begin + row_t < r_end;
      if (valid) row_coords(r_begin + row_t, xs, ys);
      for (int c = 0; c < w; ++c) X[row_t + c * pr] = valid ? entry(c, xs, ys) : make_double2(0, 0);
    }
    __syncthreads();
    for (i64 r0 = r_begin; r0 < r_end; r0 += pr) {
      const i64 rn = r0 + pr + row_t;  // this thread's row of the next panel
      const bool more = r0 + pr < r_end;
      const bool valid = more && rn < r_end;
      if (valid) row_coords(rn, xs, ys);
      int g = more ? 0 : w;  // next column of the next panel this thread generates
      auto hook = [&](int j, bool owns_next) {
        if (owns_next) return;  // this warp is on the step's critical path
        // one entry per step (about one reflector chain's worth of FP64 work
        // per SM sub-partition), two when a skipped owner step left it behind
        const int nmax = g + 1 < j ? 2 : 1;
#pragma unroll 1
        for (int n = 0; n < nmax && g < j && g < w; ++n, ++g)
          X[row_t + g * pr] = valid ? entry(g, xs, ys) : make_double2(0, 0);
      };
      absorb_panel_r<NT / 32, RPL>(R, X, w, pr, pr, bc, hook);
      // (the last step's barrier has passed: every column is dead)
      for (; g < w; ++g) X[row_t + g * pr] = valid ? entry(g, xs, ys) : make_double2(0, 0);
      __syncthreads();
    }
  } else
  for (i64 r0 = r_begin; r0 < r_end; r0 += pr) {
    const int nrows = static_cast<int>((r_end - r0) < pr ? (r_end - r0) : pr);
    if (DIAG == 2) {
      for (int i = threadIdx.x; i < pr * w; i += NT) {
        const int rr = i % pr, c = i / pr;
        const unsigned hsh = static_cast<unsigned>((r0 + rr) * 2654435761u) ^ static_cast<unsigned>(c * 40503u + 17u);
        X[rr + c * pr] = rr < nrows ? make_double2(static_cast<double>(hsh & 0xffff) * 1.5e-5 - 0.5,
                                                   static_cast<double>(hsh >> 16) * 1.5e-5 - 0.5)
                                    : make_double2(0, 0);
      }
    } else if (my_cg < ncg) {
      int ii[kMaxD], jj[kMaxD];
      const i64 row = r0 + my_row;
      const bool valid = my_row < nrows;
      if (valid) {
        i64 rem = row;
        for (int p = 0; p < D; ++p) {
          if (p == sk) continue;
          const int c = cnt[p];
          const int v = sprox[off[p] + static_cast<int>(rem % c)];
          rem /= c;
          if (p < L.d) ii[p] = v;
          else jj[p - L.d] = v;
        }
      }
      if (ks.kind == OIOBF_KERNEL_GREEN) {
        // row-invariant coordinates once per row; per column only the
        // unfolded mode's coordinate (same operations as kernel_entry)
        double xs[3] = {0, 0, 0}, ys[3] = {ks.off0, ks.off1, ks.off2};
        if (valid) {
#pragma unroll
          for (int p = 0; p < 3; ++p)
            if (p < L.d) {
              if (p != sk) xs[p] = green_x(ks, ii[p]);
              if (p + L.d != sk) ys[p] = green_y(ks, p, jj[p]);
            }
        }
        for (int c = my_cg; c < w; c += ncg) {
          double2 e = make_double2(0, 0);
          if (valid) {
            const bool tgt = sk < L.d;
            const int q = tgt ? sk : sk - L.d;
            const double v = csin[c];  // green_x / green_y of the candidate (hoisted per column)
            double xc[3], yc[3];
#pragma unroll
            for (int p = 0; p < 3; ++p) {
              xc[p] = (tgt && p == q) ? v : xs[p];
              yc[p] = (!tgt && p == q) ? v : ys[p];
            }
            e = green_from_coords_rcp(ks, xc, yc);
          }
          X[my_row + c * pr] = e;
        }
      } else if (ks.kind == OIOBF_KERNEL_RADON2D) {
        // radon2d_entry with sin / cos(2 pi x_p) hoisted: per row for the row's
        // target modes, per candidate column (csin / ccos) for an unfolded
        // target mode -- the same operations as kernel_entry, so bit-identical
        double sx[2] = {0, 0}, cx[2] = {0, 0};
        if (valid)
          for (int p = 0; p < 2; ++p)
            if (p != sk)
              sincos(__dmul_rn(2.0 * M_PI, __ddiv_rn(static_cast<double>(ii[p] - 1), static_cast<double>(ks.n))), &sx[p],
                     &cx[p]);
        for (int c = my_cg; c < w; c += ncg) {
          double2 e = make_double2(0, 0);
          if (valid) {
            const int t = stgt[c];
            if (sk < 2) {
              ii[sk] = t;
              sx[sk] = csin[c];
              cx[sk] = ccos[c];
            } else {
              jj[sk - 2] = t;
            }
            e = radon2d_entry_sc(ks, ii, jj, sx[0], cx[0], sx[1], cx[1]);
          }
          X[my_row + c * pr] = e;
        }
      } else {
        for (int c = my_cg; c < w; c += ncg) {
          double2 e = make_double2(0, 0);
          if (valid) {
            const int t = stgt[c];
            if (sk < L.d) ii[sk] = t;
            else jj[sk - L.d] = t;
            e = kernel_entry(ks, ii, jj);
          }
          X[my_row + c * pr] = e;
        }
      }
    }
    __syncthreads();
    // rows nrows..pr-1 of the panel were generated as zeros, so the
    // register-cached absorb folds all pr rows unconditionally (no per-element
    // row predicates; zero rows leave R unchanged)
    if constexpr (DIAG == 1) {
      for (int i = threadIdx.x; i < pr * w; i += NT) diag_acc += X[i].x;
      __syncthreads();
    } else if constexpr (RPL > 0) {
      absorb_panel_r<NT / 32, RPL>(R, X, w, pr, pr, bc, [](int, bool) {});
    } else {
      absorb_panel<NT / 32>(R, X, w, nrows, pr, bc, [](int, bool) {});
    }
  }
  if (DIAG == 1 && diag_acc == 12345.678) R[0].x += 1;  // keeps the generation live
  double2* out = rpart + (slot * L.nparts + part) * L.wmax * L.wmax;
  for (int i = threadIdx.x; i < w * w; i += NT) {  // unpack to w x w column-major
    const int r = i % w, c = i / w;
    out[i] = r <= c ? R[rpk(r, c)] : make_double2(0, 0);
  }
}

// ---------------------------------------------------------------- finish
constexpr int kFinThreads = 128;

__device__ __forceinline__ double block_max(double v, double* red) {
  v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 16));
  v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 8));
  v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 4));
  v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 2));
  v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 1));
  const int warp = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[warp] = v;
  __syncthreads();
  double m = red[0];
  for (int q = 1; q < kFinThreads / 32; ++q) m = fmax(m, red[q]);
  return m;
}
__device__ __forceinline__ int block_min_int(int v, int* red) {
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[warp] = v;
  __syncthreads();
  int m = red[0];
  for (int q = 1; q < kFinThreads / 32; ++q) m = min(m, red[q]);
  return m;
}

// Outputs per slot (scratch, stride wmax / wmax^2): rank, saturated, perm[w],
// skeleton (global, sorted) [r], interp (r x w col-major, ld r), gap diagnostics.
__global__ void __launch_bounds__(kFinThreads) k_finish(LevelDesc L, double tol, double tie_eps, i64 max_rank,
                                                        const i64* __restrict__ mrows,
                                                        const i64* __restrict__ max_rank_arr,
                                                        const double2* __restrict__ rpart,
                                                        const int* __restrict__ targets,
                                                        const int* __restrict__ width, int* __restrict__ rank_out,
                                                        int* __restrict__ sat_out, int* __restrict__ perm_out,
                                                        int* __restrict__ skel_tmp, double2* __restrict__ interp_tmp,
                                                        double* __restrict__ gap_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const i64 slot = blockIdx.x;
  const int w = width[slot];
  const int ld = w | 1;  // odd leading dimension: conflict-free column walks
  double2* A = reinterpret_cast<double2*>(smem);           // w x w, ld
  double2* X = A + static_cast<i64>(ld) * (L.wmax | 1);    // partition panel w x w, ld w
  double2* v = X + L.wmax * L.wmax;                        // Householder vector
  Bcast* bc = reinterpret_cast<Bcast*>(v + L.wmax);
  double* red = reinterpret_cast<double*>(bc + 2);
  int* ired = reinterpret_cast<int*>(red + 8);
  int* perm = ired + 8;
  __shared__ double s_ref, s_xnorm, s_beta, s_mingap;
  __shared__ double2 s_sign;
  __shared__ int s_stop, s_jmax, s_rank, s_sat;
  const int t = threadIdx.x;
  if (w == 0) {
    if (t == 0) {
      rank_out[slot] = 0;
      sat_out[slot] = 0;
    }
    return;
  }
  // ---- combine partition factors: A = R_0, then absorb R_1..R_{P-1}
  // (absorb_panel uses kWarps warps; here only kFinThreads/32 exist, so use a
  // simple column-serial Householder with thread-per-column updates instead)
  for (int i = t; i < w * w; i += kFinThreads) {
    const int r = i % w, c = i / w;
    A[r + c * ld] = rpart[(slot * L.nparts) * L.wmax * L.wmax + i];
  }
  __syncthreads();
  for (i64 part = 1; part < L.nparts; ++part) {
    const double2* src = rpart + (slot * L.nparts + part) * L.wmax * L.wmax;
    for (int i = t; i < w * w; i += kFinThreads) X[i] = src[i];
    __syncthreads();
    for (int j = 0; j < w; ++j) {
      // sigma over panel column j (rows 0..j suffice: upper triangular)
      if (t == 0) {
        double sig = 0;
        for (int i = 0; i <= j; ++i) sig += cnorm2(X[i + j * w]);
        bc[0] = make_reflector(A[j + j * ld], sig, &A[j + j * ld]);
      }
      __syncthreads();
      if (bc[0].active) {
        const Bcast b = bc[0];
        for (int k = j + 1 + t; k < w; k += kFinThreads) {
          double2 dot = make_double2(0, 0);
          for (int i = 0; i <= j; ++i) cfmac(dot, X[i + j * w], X[i + k * w]);
          const double2 ws = reflect_coeff(b, A[j + k * ld], dot);
          const double2 tt = cmul(b.scale, ws);
          A[j + k * ld] = csub(A[j + k * ld], ws);
          for (int i = 0; i <= j; ++i) X[i + k * w] = csub(X[i + k * w], cmul(X[i + j * w], tt));
        }
      }
      __syncthreads();
    }
  }
  // ---- reference qrcp (id.cpp:24-85) on A (w x w); A rows >= w are zero
  const i64 mm = mrows ? mrows[slot] : L.m;
  i64 limit = mm < w ? mm : w;
  const i64 mr = max_rank_arr ? max_rank_arr[slot] : max_rank;
  if (mr >= 0 && mr < limit) limit = mr;
  for (int j = t; j < w; j += kFinThreads) perm[j] = j;
  if (t == 0) {
    s_mingap = INFINITY;
    s_sat = 0;
  }
  __syncthreads();
  int k = 0;
  for (;; ++k) {
    // residual norms of trailing columns
    double c = -1;
    if (t >= k && t < w) {
      c = 0;
      for (int i = k; i < w; ++i) c += cnorm2(A[i + t * ld]);
    }
    const double cmax = block_max(c, red);
    const double best = sqrt(cmax > 0 ? cmax : 0);
    if (k == 0 && t == 0) s_ref = best;
    __syncthreads();
    const double ref = s_ref;
    // first (lowest current position) column within tie_eps*ref of the best
    const bool cand = (t >= k && t < w) && (sqrt(c) >= best - tie_eps * ref);
    const int jmax = block_min_int(cand ? t : 0x7fffffff, ired);
    // runner-up gap (diagnostic)
    const double c2 = (t >= k && t < w && t != jmax) ? c : -1;
    const double second = block_max(c2, red);
    if (t == 0) {
      if (second >= 0 && ref > 0) s_mingap = fmin(s_mingap, (best - sqrt(second)) / ref);
      int stop = 0;
      if (k == 0) {
        stop = (ref == 0);
      } else {
        stop = (best <= tol * ref);
      }
      if (!stop && k == limit) {
        s_sat = (best > tol * ref) && (limit < w);
        stop = 1;
      }
      if (k >= w) stop = 1;
      s_stop = stop;
      s_jmax = jmax;
    }
    __syncthreads();
    if (s_stop) break;
    const int jm = s_jmax;
    // swap columns k <-> jm
    if (jm != k) {
      for (int i = t; i < w; i += kFinThreads) {
        const double2 a = A[i + k * ld];
        A[i + k * ld] = A[i + jm * ld];
        A[i + jm * ld] = a;
      }
      if (t == 0) {
        const int q = perm[k];
        perm[k] = perm[jm];
        perm[jm] = q;
      }
    }
    __syncthreads();
    // Householder reflector zeroing A(k+1:w, k)
    if (t == 0) {
      double xs = 0;
      for (int i = k; i < w; ++i) xs += cnorm2(A[i + k * ld]);
      const double xnorm = sqrt(xs);
      s_xnorm = xnorm;
      const double2 alpha = A[k + k * ld];
      const double aa = sqrt(cnorm2(alpha));
      const double2 sign = (alpha.x == 0 && alpha.y == 0) ? make_double2(1, 0)
                                                          : make_double2(alpha.x / aa, alpha.y / aa);
      s_sign = sign;
      double vn2 = 0;
      for (int i = k; i < w; ++i) {
        double2 vi = A[i + k * ld];
        if (i == k) vi = make_double2(vi.x + sign.x * xnorm, vi.y + sign.y * xnorm);
        v[i] = vi;
        vn2 += cnorm2(vi);
      }
      s_beta = (xnorm > 0 && vn2 > 0) ? 2.0 / vn2 : 0.0;
    }
    __syncthreads();
    if (s_xnorm > 0) {
      const double beta = s_beta;
      if (beta > 0) {
        for (int j = k + 1 + t; j < w; j += kFinThreads) {
          double2 s = make_double2(0, 0);
          for (int i = k; i < w; ++i) cfmac(s, v[i], A[i + j * ld]);
          const double2 ws = cscale(beta, s);
          for (int i = k; i < w; ++i) A[i + j * ld] = csub(A[i + j * ld], cmul(v[i], ws));
        }
      }
      __syncthreads();
      if (t == 0) {
        for (int i = k + 1; i < w; ++i) A[i + k * ld] = make_double2(0, 0);
        A[k + k * ld] = make_double2(-s_sign.x * s_xnorm, -s_sign.y * s_xnorm);
      }
    }
    __syncthreads();
  }
  const int r = k;
  // ---- id_from_qrcp (id.cpp:87-120): T = R11^{-1} R12 in place in A(:, r:)
  for (int cidx = t; cidx < w - r; cidx += kFinThreads) {
    const int col = r + cidx;
    for (int i = r - 1; i >= 0; --i) {
      double2 s = A[i + col * ld];
      for (int q = i + 1; q < r; ++q) s = csub(s, cmul(A[i + q * ld], A[q + col * ld]));
      A[i + col * ld] = cdiv(s, A[i + i * ld]);
    }
  }
  __syncthreads();
  // sorted position of pivot p among the first r pivots
  double2* interp = interp_tmp + slot * L.wmax * L.wmax;
  int* skel = skel_tmp + slot * L.wmax;
  const int* tg = targets + slot * L.wmax;
  for (int p = t; p < r; p += kFinThreads) {
    int pos = 0;
    for (int q = 0; q < r; ++q) pos += perm[q] < perm[p];
    skel[pos] = tg[perm[p]];
    interp[pos + perm[p] * r] = make_double2(1, 0);
    for (int j = 0; j < r; ++j)
      if (j != p) interp[pos + perm[j] * r] = make_double2(0, 0);
    for (int j = r; j < w; ++j) interp[pos + perm[j] * r] = A[p + j * ld];
  }
  for (int j = t; j < w; j += kFinThreads) perm_out[slot * L.wmax + j] = perm[j];
  if (t == 0) {
    rank_out[slot] = r;
    sat_out[slot] = s_sat;
    gap_out[slot] = s_mingap;
  }
}

__global__ void k_compact(i64 nslots, i64 wmax, const int* __restrict__ rank, const int* __restrict__ width,
                          const i64* __restrict__ skel_off, const i64* __restrict__ interp_off,
                          const int* __restrict__ skel_tmp, const double2* __restrict__ interp_tmp,
                          int* __restrict__ skel, double2* __restrict__ interp) {
  const i64 slot = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (slot >= nslots) return;
  const int r = rank[slot], w = width[slot];
  for (int i = lane; i < r; i += 32) skel[skel_off[slot] + i] = skel_tmp[slot * wmax + i];
  for (int i = lane; i < r * w; i += 32) interp[interp_off[slot] + i] = interp_tmp[slot * wmax * wmax + i];
}


// column_id of explicit device matrices: same TSQR, rows read from HBM
__global__ void __launch_bounds__(kThreads) k_matrix_panel(i64 nparts, i64 rpp, int pr, i64 wmax,
                                                           const i64* __restrict__ a_off, const i64* __restrict__ mrows,
                                                           const int* __restrict__ ncols,
                                                           const double2* __restrict__ A,
                                                           double2* __restrict__ rpart) {
  extern __shared__ __align__(16) unsigned char smem[];
  const i64 slot = blockIdx.x / nparts;
  const i64 part = blockIdx.x % nparts;
  const int w = ncols[slot];
  const i64 m = mrows[slot];
  double2* R = reinterpret_cast<double2*>(smem);  // packed upper triangle
  double2* X = R + wmax * (wmax + 1) / 2;
  Bcast* bc = reinterpret_cast<Bcast*>(X + static_cast<i64>(pr) * wmax);
  for (int i = threadIdx.x; i < w * (w + 1) / 2; i += kThreads) R[i] = make_double2(0, 0);
  __syncthreads();
  const i64 r_begin = part * rpp;
  i64 r_end = r_begin + rpp;
  if (r_end > m) r_end = m;
  const double2* a = A + a_off[slot];
  for (i64 r0 = r_begin; r0 < r_end; r0 += pr) {
    const int nrows = static_cast<int>((r_end - r0) < pr ? (r_end - r0) : pr);
    for (int e = threadIdx.x; e < pr * w; e += kThreads) {
      const int i = e % pr, c = e / pr;
      X[i + c * pr] = i < nrows ? a[r0 + i + static_cast<i64>(c) * m] : make_double2(0, 0);
    }
    __syncthreads();
    absorb_panel<kWarps>(R, X, w, nrows, pr, bc, [](int, bool) {});
  }
  double2* out = rpart + (slot * nparts + part) * wmax * wmax;
  for (int i = threadIdx.x; i < w * w; i += kThreads) {  // unpack to w x w column-major
    const int r = i % w, c = i / w;
    out[i] = r <= c ? R[rpk(r, c)] : make_double2(0, 0);
  }
}


}  // namespace

size_t panel_smem_bytes(const LevelDesc& L) {
  return sizeof(double2) * (L.wmax * (L.wmax + 1) / 2 + static_cast<size_t>(L.pr) * L.wmax) + 2 * sizeof(Bcast) +
         sizeof(int) * (L.psize + L.wmax + 1) + sizeof(double) * (2 * L.wmax + 1) + 16;
}

size_t finish_smem_bytes(const LevelDesc& L) {
  return sizeof(double2) * ((L.wmax | 1) * (L.wmax | 1) + L.wmax * L.wmax + L.wmax) + 2 * sizeof(Bcast) +
         8 * sizeof(double) + 8 * sizeof(int) + sizeof(int) * L.wmax + 16;
}

void launch_gen_proxies(const LevelDesc& L, int* proxies, cudaStream_t st) {
  const i64 total = L.nslots * 2 * L.d;
  k_gen_proxies<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(L, proxies);
  TBF_CUDA(cudaGetLastError());
  int big = 0;
  for (int k = 0; k < L.d; ++k)
    for (int p = 0; p < 2 * L.d; ++p) big |= L.counts[k][p] > kMaxProxy;
  if (big && L.proxy_mode == OIOBF_PROXY_UNIFORM_RANDOM) {
    const size_t smem = static_cast<size_t>(L.n) * (sizeof(int) + 1) + 16;
    TBF_CUDA(cudaFuncSetAttribute(k_gen_proxies_big, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    k_gen_proxies_big<<<static_cast<unsigned>(total), 32, smem, st>>>(L, proxies);
    TBF_CUDA(cudaGetLastError());
  }
}

void launch_targets(const LevelDesc& L, const int* crank, const i64* cskel_off, const int* cskel, int* targets,
                    int* width, cudaStream_t st) {
  const i64 threads = L.nslots * 32;
  k_targets<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(L, crank, cskel_off, cskel, targets, width);
  TBF_CUDA(cudaGetLastError());
}

template <int NT, int RPL, int DIAG = 0, int PIPE = 0, int MINB = (NT >= 512 ? 1 : (RPL >= 8 ? 2 : 3))>
void launch_panel_t(const LevelDesc& L, const KSpec& ks, const int* proxies, const int* targets, const int* width,
                    double2* rpart, size_t smem, i64 grid, cudaStream_t st) {
  TBF_CUDA(cudaFuncSetAttribute(k_panel<NT, RPL, MINB, DIAG, PIPE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kMaxDynSmem));
  k_panel<NT, RPL, MINB, DIAG, PIPE><<<static_cast<unsigned>(grid), NT, smem, st>>>(L, ks, proxies, targets, width,
                                                                                   rpart);
}

// Panel rows and resident CTAs per SM for a level of width wmax.  The column
// sweep is latency-bound (one CTA barrier and one look-ahead reflector per
// column), so a step should carry as many rows as shared memory holds:
// w <= 32: 256-thread CTAs, 256- / 128-row panels, up to 3 CTAs per SM;
// w > 32: one 512-thread CTA per SM with the tallest panel (multiple of 32
// rows, at most 192) next to the packed R.
void panel_shape(i64 wmax, i64 psize, int* pr, int* ctas_per_sm) {
  static const int over = std::getenv("OIOBF_PANEL_PR") ? std::atoi(std::getenv("OIOBF_PANEL_PR")) : 0;  // sweeps
  LevelDesc t{};
  t.wmax = wmax;
  t.psize = psize;
  if (wmax <= 32) {
    t.pr = over > 0 ? over : wmax <= 24 ? 256 : 128;
    *pr = t.pr;
    *ctas_per_sm = static_cast<int>(std::max<size_t>(1, std::min<size_t>(3, 227 * 1024 / (panel_smem_bytes(t) + 1024))));
    return;
  }
  int best = 64;
  for (int p = 64; p <= 192; p += 32) {
    t.pr = p;
    if (panel_smem_bytes(t) <= static_cast<size_t>(kMaxDynSmem)) best = p;
  }
  *pr = over > 0 ? over : best;
  *ctas_per_sm = 1;
}

template <int DIAG>
void launch_panel_mode(const LevelDesc& L, const KSpec& ks, const int* proxies, const int* targets,
                       const int* width, double2* rpart, cudaStream_t st) {
  const size_t smem = panel_smem_bytes(L);
  const i64 grid = L.nslots * L.nparts;
  static const bool generic = std::getenv("OIOBF_PANEL_GENERIC") != nullptr;  // A/B switch
  if (L.wmax > 32) {
    if (!generic && L.pr == 192) launch_panel_t<512, 6, DIAG>(L, ks, proxies, targets, width, rpart, smem, grid, st);
    else if (!generic && L.pr == 160) launch_panel_t<512, 5, DIAG>(L, ks, proxies, targets, width, rpart, smem, grid, st);
    else if (!generic && L.pr == 128) launch_panel_t<512, 4, DIAG>(L, ks, proxies, targets, width, rpart, smem, grid, st);
    else if (!generic && L.pr == 96) launch_panel_t<512, 3, DIAG>(L, ks, proxies, targets, width, rpart, smem, grid, st);
    else if (!generic && L.pr == 64) launch_panel_t<512, 2, DIAG>(L, ks, proxies, targets, width, rpart, smem, grid, st);
    else launch_panel_t<512, 0, DIAG>(L, ks, proxies, targets, width, rpart, smem, grid, st);
  } else {
    // (the register-cached absorb spills at the 3-CTA/SM budget of these CTAs)
    // register-cached absorb on 256-row panels at 2 CTAs/SM (128 registers,
    // one column update at a time): bit-identical to the generic absorb,
    // config 2 panel 20.4 -> 17.2 ms, config 3 unchanged
    static const int rc = std::getenv("OIOBF_PANEL_NARROW_RC") ? std::atoi(std::getenv("OIOBF_PANEL_NARROW_RC")) : 1;
    // (Green entries of the next panel generated inside the column steps: OIOBF_PANEL_PIPE=0 disables)
    static const bool pipe = !(std::getenv("OIOBF_PANEL_PIPE") && std::getenv("OIOBF_PANEL_PIPE")[0] == '0');
    if (rc && !generic && L.pr == 256 && DIAG == 0 && pipe && ks.kind == OIOBF_KERNEL_GREEN)
      launch_panel_t<kThreads, 8, 0, 1>(L, ks, proxies, targets, width, rpart, smem, grid, st);
    else if (rc && !generic && L.pr == 256) launch_panel_t<kThreads, 8, DIAG>(L, ks, proxies, targets, width, rpart, smem, grid, st);
    else launch_panel_t<kThreads, 0, DIAG>(L, ks, proxies, targets, width, rpart, smem, grid, st);
  }
  TBF_CUDA(cudaGetLastError());
}

void launch_panel(const LevelDesc& L, const KSpec& ks, const int* proxies, const int* targets, const int* width,
                  double2* rpart, cudaStream_t st) {
  launch_panel_mode<0>(L, ks, proxies, targets, width, rpart, st);
  static const bool diag = std::getenv("OIOBF_PANEL_DIAG") != nullptr;  // timing split (tools)
  if (!diag) return;
  cudaEvent_t e[4];
  for (auto& x : e) TBF_CUDA(cudaEventCreate(&x));
  double2* scratch = nullptr;
  const size_t bytes = sizeof(double2) * static_cast<size_t>(L.nslots * L.nparts * L.wmax * L.wmax);
  TBF_CUDA(cudaMallocAsync(&scratch, bytes, st));
  TBF_CUDA(cudaEventRecord(e[0], st));
  launch_panel_mode<0>(L, ks, proxies, targets, width, scratch, st);
  TBF_CUDA(cudaEventRecord(e[1], st));
  launch_panel_mode<1>(L, ks, proxies, targets, width, scratch, st);
  TBF_CUDA(cudaEventRecord(e[2], st));
  launch_panel_mode<2>(L, ks, proxies, targets, width, scratch, st);
  TBF_CUDA(cudaEventRecord(e[3], st));
  TBF_CUDA(cudaEventSynchronize(e[3]));
  float t[3];
  for (int i = 0; i < 3; ++i) TBF_CUDA(cudaEventElapsedTime(&t[i], e[i], e[i + 1]));
  std::fprintf(stderr, "panel-diag side %d l %d nslots %lld w %lld pr %d nparts %lld m %lld: full %.3f gen %.3f absorb %.3f ms\n",
               static_cast<int>(L.side), static_cast<int>(L.l), static_cast<long long>(L.nslots),
               static_cast<long long>(L.wmax), L.pr, static_cast<long long>(L.nparts), static_cast<long long>(L.m),
               t[0], t[1], t[2]);
  TBF_CUDA(cudaFreeAsync(scratch, st));
  for (auto& x : e) TBF_CUDA(cudaEventDestroy(x));
}

void launch_finish(const LevelDesc& L, double tol, double tie_eps, i64 max_rank, const double2* rpart,
                   const int* targets, const int* width, int* rank, int* sat, int* perm, int* skel_tmp,
                   double2* interp_tmp, double* gaps, cudaStream_t st) {
  const size_t smem = finish_smem_bytes(L);
  TBF_CUDA(cudaFuncSetAttribute(k_finish, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
  k_finish<<<static_cast<unsigned>(L.nslots), kFinThreads, smem, st>>>(L, tol, tie_eps, max_rank, nullptr, nullptr,
                                                                      rpart, targets,
                                                                      width, rank, sat, perm, skel_tmp, interp_tmp,
                                                                      gaps);
  TBF_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// Narrow column IDs of the separable DFT kernel (config 4: every candidate set
// has w <= 2 columns over m = 131,072 proxy rows).  The DFT entry is
// K = exp(-2 pi i/n * sum_p (a_p - 1)(b_p - 1 - n/2)) with a, b the
// (bit-reversed) target / source indices, so the two candidate columns of a
// slot differ only in the factor of the unfolded mode k, and over the
// Cartesian-product proxy rows
//   |a_0|^2 = |a_1|^2 = m,   a_0^H a_1 = (m / cnt) * S,   S = sum_x w^(-e_x)
// with x running over the cnt proxies of the mode paired with k and
// e_x = (phase of column 1 - phase of column 0) mod n.  The reference QRCP on
// the explicit m x 2 matrix (id.cpp:24-85) therefore reduces to: first pivot
// a tie (column norms equal; gap 0 reported, oracle replay),
// residual^2 = m (1 - |S|^2 / cnt^2) against (tol |R11|)^2 = tol^2 m, and
// T = R11^-1 R12 = S / cnt.  When every e_x is equal (the two-sided
// bit-reversed DFT, where all ranks are exactly 1) the residual is exactly 0
// and T = w^(-e) is computed with the entry formula itself.  One thread per
// slot; only the paired mode's proxy list is regenerated (same seeds as
// k_gen_proxies), so no proxy, panel or R buffers are needed.
__global__ void k_narrow_dft(LevelDesc L, KSpec ks, double tol, const int* __restrict__ crank,
                             const i64* __restrict__ cskel_off, const int* __restrict__ cskel,
                             int* __restrict__ width_out, int* __restrict__ rank_out, int* __restrict__ sat_out,
                             int* __restrict__ perm_out, int* __restrict__ skel_tmp, double2* __restrict__ interp_tmp,
                             double* __restrict__ gap_out) {
  const i64 slot = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (slot >= L.nslots) return;
  const SlotPos s = decode_slot(L, slot);
  sat_out[slot] = 0;
  if (!owns_outer(L, s.outer)) {
    width_out[slot] = 0;
    rank_out[slot] = 0;
    return;
  }
  int tg[2];
  int w = 0;
  if (L.l == 0) {
    for (i64 c = 0; c < s.sz[s.skip] && w < 2; ++c) tg[w++] = static_cast<int>(s.lo[s.skip] + c);
  } else {
    const i64 c0 = child_slot(L, s, 0), c1 = child_slot(L, s, 1);
    for (int c = 0; c < crank[c0]; ++c) tg[w++] = cskel[cskel_off[c0] + c];
    for (int c = 0; c < crank[c1]; ++c) tg[w++] = cskel[cskel_off[c1] + c];
  }
  width_out[slot] = w;
  int* perm = perm_out + slot * L.wmax;
  int* skel = skel_tmp + slot * L.wmax;
  double2* interp = interp_tmp + slot * L.wmax * L.wmax;
  if (w == 0) {
    rank_out[slot] = 0;
    return;
  }
  if (w == 1) {  // |K| = 1: the column norm is sqrt(m) > 0, rank 1
    perm[0] = 0;
    skel[0] = tg[0];
    interp[0] = make_double2(1, 0);
    rank_out[slot] = 1;
    gap_out[slot] = INFINITY;
    return;
  }
  // paired mode: V side (columns = source mode k) pairs with target mode k;
  // U side (columns = target mode k) pairs with source mode k
  const int pm = L.side == 0 ? static_cast<int>(s.k) : L.d + static_cast<int>(s.k);
  const i64 cnt = L.counts[s.k][pm];
  const u64 tags[7] = {L.side_tag, static_cast<u64>(L.l), static_cast<u64>(s.outer), static_cast<u64>(s.inner),
                       static_cast<u64>(s.k), static_cast<u64>(s.j), 0ULL};
  const u64 sseed = derive_seed(L.seed, tags, 7);
  const u64 ptags[2] = {0x70ULL, static_cast<u64>(pm)};
  const u64 pseed = derive_seed(sseed, ptags, 2);
  int px[kMaxProxy];
  const i64 np = L.proxy_mode == OIOBF_PROXY_ALL ? s.sz[pm] : select_proxies(s.sz[pm], cnt, L.proxy_mode, pseed, px);
  const i64 n = ks.n;
  auto br = [&](i64 idx) { return ks.bitrev ? bitrev1(idx, n) : idx; };
  const i64 t0 = br(tg[0]), t1 = br(tg[1]);
  int e_first = -1;
  bool all_equal = true;
  double2 S = make_double2(0, 0);
  for (i64 q = 0; q < np; ++q) {
    const i64 x = (L.proxy_mode == OIOBF_PROXY_ALL ? q + 1 : px[q]) + s.lo[pm] - 1;
    const i64 bx = br(x);
    i64 e = L.side == 0 ? (bx - 1) * (t1 - t0) : (t1 - t0) * (bx - 1 - n / 2);
    e %= n;
    if (e < 0) e += n;
    if (e_first < 0) e_first = static_cast<int>(e);
    all_equal &= (e == e_first);
    double sn, cs;
    sincos(__dmul_rn(M_PI, __ddiv_rn(2.0 * static_cast<double>(e), static_cast<double>(n))), &sn, &cs);
    S = make_double2(S.x + cs, S.y - sn);
  }
  const double dn = static_cast<double>(np);
  const double def = all_equal ? 0.0 : fmax(0.0, 1.0 - (S.x * S.x + S.y * S.y) / (dn * dn));
  perm[0] = 0;  // exact tie: first column in current order (reference strict >)
  perm[1] = 1;
  gap_out[slot] = 0.0;
  if (def <= tol * tol) {
    double2 T;
    if (all_equal) {
      double sn, cs;
      sincos(__dmul_rn(M_PI, __ddiv_rn(2.0 * static_cast<double>(e_first), static_cast<double>(n))), &sn, &cs);
      T = make_double2(cs, -sn);
    } else {
      T = make_double2(S.x / dn, S.y / dn);
    }
    skel[0] = tg[0];
    interp[0] = make_double2(1, 0);  // r x w col-major, ld 1
    interp[1] = T;
    rank_out[slot] = 1;
  } else {  // full rank: skeleton = both candidates (already in order), interp = I
    skel[0] = tg[0];
    skel[1] = tg[1];
    interp[0] = make_double2(1, 0);
    interp[1] = make_double2(0, 0);
    interp[2] = make_double2(0, 0);
    interp[3] = make_double2(1, 0);
    rank_out[slot] = 2;
  }
}

void launch_narrow_dft(const LevelDesc& L, const KSpec& ks, double tol, const int* crank, const i64* cskel_off,
                       const int* cskel, int* width, int* rank, int* sat, int* perm, int* skel_tmp, double2* interp_tmp,
                       double* gaps, cudaStream_t st) {
  if (L.nslots == 0) return;
  k_narrow_dft<<<static_cast<unsigned>((L.nslots + 127) / 128), 128, 0, st>>>(L, ks, tol, crank, cskel_off, cskel, width,
                                                                             rank, sat, perm, skel_tmp, interp_tmp,
                                                                             gaps);
  TBF_CUDA(cudaGetLastError());
}

void launch_compact(i64 nslots, i64 wmax, const int* rank, const int* width, const i64* skel_off,
                    const i64* interp_off, const int* skel_tmp, const double2* interp_tmp, int* skel, double2* interp,
                    cudaStream_t st) {
  const i64 threads = nslots * 32;
  k_compact<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(nslots, wmax, rank, width, skel_off,
                                                                         interp_off, skel_tmp, interp_tmp, skel,
                                                                         interp);
  TBF_CUDA(cudaGetLastError());
}

void launch_matrix_ids(i64 njobs, const i64* a_off, const i64* m, const int* n, const double2* A, i64 nparts, i64 rpp,
                       int pr, i64 wmax, double2* rpart, cudaStream_t st) {
  const size_t smem = sizeof(double2) * (wmax * (wmax + 1) / 2 + static_cast<size_t>(pr) * wmax) + 2 * sizeof(Bcast) + 16;
  TBF_CUDA(cudaFuncSetAttribute(k_matrix_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
  k_matrix_panel<<<static_cast<unsigned>(njobs * nparts), kThreads, smem, st>>>(nparts, rpp, pr, wmax, a_off, m, n, A,
                                                                               rpart);
  TBF_CUDA(cudaGetLastError());
}

void launch_finish_var(const LevelDesc& L, const i64* mrows, double tol, double tie_eps, const i64* max_rank,
                       const double2* rpart, const int* targets, const int* width, int* rank, int* sat, int* perm,
                       int* skel_tmp, double2* interp_tmp, double* gaps, cudaStream_t st) {
  const size_t smem = finish_smem_bytes(L);
  TBF_CUDA(cudaFuncSetAttribute(k_finish, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
  k_finish<<<static_cast<unsigned>(L.nslots), kFinThreads, smem, st>>>(L, tol, tie_eps, -1, mrows, max_rank, rpart,
                                                                      targets, width, rank, sat, perm, skel_tmp,
                                                                      interp_tmp, gaps);
  TBF_CUDA(cudaGetLastError());
}

}  // namespace tbf
