// column_id of explicit matrices with more columns than the shared-memory ID
// kernels hold (n > kMaxW = 96): the reference's column-pivoted Householder QR
// (ref: proj/src/id.cpp:24-85) and its interpolation step (id.cpp:87-120)
// restated directly on a work copy of the matrix in global memory, one CTA per
// matrix.  This is the drop-in's completeness path (column_id / row_id /
// hybrid_id of arbitrary size), not a hot path: the butterfly's own IDs have at
// most 2 r_max candidate columns and run in k_panel / k_finish.
//
// Per step k (pivot rule as the reference: exact squared norms of the trailing
// columns over rows k.., first maximum wins):
//   norms (a warp per column) -> argmax -> stop tests (tolerance against the
//   first pivot, rank limit / saturation) -> column swap -> reflector
//   v = x + sign |x| e_1 -> trailing update a_j -= v (2 / v^H v) v^H a_j (a
//   warp per column) -> a_kk = -sign |x|.
// Then T = R11^{-1} R12 by back substitution (a warp per column), the skeleton
// in ascending column order and the interpolation matrix in that row order.
#include "kernels.h"

namespace tbf {

namespace {

constexpr int kWideThreads = 256;
constexpr int kWideWarps = kWideThreads / 32;

__global__ void __launch_bounds__(kWideThreads) k_qrcp_wide(const WideIdJob* __restrict__ jobs, double2* __restrict__ A,
                                                            double* __restrict__ nrm_all, int* __restrict__ perm_all,
                                                            int* __restrict__ pos_all, double tol,
                                                            int* __restrict__ rank_out, int* __restrict__ sat_out,
                                                            int* __restrict__ skel_all, double2* __restrict__ interp_all) {
  const WideIdJob J = jobs[blockIdx.x];
  const i64 m = J.m;
  const int n = J.n;
  double2* a = A + J.a_off;
  double* nrm = nrm_all + J.n_off;
  int* perm = perm_all + J.n_off;
  int* pos = pos_all + J.n_off;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ double s_best[kWideWarps];
  __shared__ int s_j[kWideWarps];
  __shared__ double s_ref, s_pivot2, s_beta;
  __shared__ int s_stop, s_jmax, s_sat;
  __shared__ double2 s_v0, s_rkk;
  for (int i = tid; i < n; i += kWideThreads) perm[i] = i;
  if (tid == 0) s_sat = 0;
  const i64 lim0 = m < n ? m : n;
  const i64 limit = J.max_rank >= 0 && J.max_rank < lim0 ? J.max_rank : lim0;
  int k = 0;
  __syncthreads();
  for (;; ++k) {
    // squared norms of the trailing columns over rows k..m-1
    for (int j = k + warp; j < n; j += kWideWarps) {
      const double2* c = a + static_cast<i64>(j) * m;
      double s = 0;
      for (i64 i = k + lane; i < m; i += 32) s += cnorm2(c[i]);
      s = warp_sum(s);
      if (lane == 0) nrm[j] = s;
    }
    __syncthreads();
    // first maximum (strictly greater wins; equal norms keep the lowest index)
    double best = -1;
    int jb = -1;
    for (int j = k + tid; j < n; j += kWideThreads) {
      const double c = nrm[j];
      if (c > best) {
        best = c;
        jb = j;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oj = __shfl_xor_sync(0xffffffffu, jb, o);
      if (oj >= 0 && (jb < 0 || ob > best || (ob == best && oj < jb))) {
        best = ob;
        jb = oj;
      }
    }
    if (lane == 0) {
      s_best[warp] = best;
      s_j[warp] = jb;
    }
    __syncthreads();
    if (tid == 0) {
      for (int q = 0; q < kWideWarps; ++q)
        if (s_j[q] >= 0 && (jb < 0 || s_best[q] > best || (s_best[q] == best && s_j[q] < jb))) {
          best = s_best[q];
          jb = s_j[q];
        }
      const double eta = jb >= 0 ? sqrt(best) : 0.0;
      int stop = 0;
      if (k == 0) {
        s_ref = eta;
        stop = eta == 0;
      } else {
        stop = jb < 0 || eta <= tol * s_ref;
      }
      if (!stop && k == limit) {
        s_sat = (eta > tol * s_ref) && (limit < n);
        stop = 1;
      }
      s_stop = stop;
      s_jmax = jb;
      s_pivot2 = best;
    }
    __syncthreads();
    if (s_stop) break;
    const int jmax = s_jmax;
    if (jmax != k) {
      double2* ck = a + static_cast<i64>(k) * m;
      double2* cj = a + static_cast<i64>(jmax) * m;
      for (i64 i = tid; i < m; i += kWideThreads) {
        const double2 t = ck[i];
        ck[i] = cj[i];
        cj[i] = t;
      }
      if (tid == 0) {
        const int t = perm[k];
        perm[k] = perm[jmax];
        perm[jmax] = t;
      }
    }
    __syncthreads();
    double2* ck = a + static_cast<i64>(k) * m;
    if (tid == 0) {
      const double2 alpha = ck[k];
      const double x2 = s_pivot2, xnorm = sqrt(x2);
      double beta = 0;
      double2 v0 = alpha, rkk = alpha;
      if (xnorm > 0) {
        const double aa = sqrt(cnorm2(alpha));
        const double2 sign = aa == 0 ? make_double2(1, 0) : make_double2(alpha.x / aa, alpha.y / aa);
        v0 = make_double2(alpha.x + sign.x * xnorm, alpha.y + sign.y * xnorm);
        double tail2 = x2 - cnorm2(alpha);  // sum over the rows below the diagonal
        if (tail2 < 0) tail2 = 0;
        const double vnorm2 = cnorm2(v0) + tail2;
        if (vnorm2 > 0) beta = 2.0 / vnorm2;
        rkk = make_double2(-sign.x * xnorm, -sign.y * xnorm);
      }
      s_v0 = v0;
      s_beta = beta;
      s_rkk = rkk;
    }
    __syncthreads();
    const double beta = s_beta;
    const double2 v0 = s_v0;
    if (beta > 0) {
      for (int j = k + 1 + warp; j < n; j += kWideWarps) {
        double2* cj = a + static_cast<i64>(j) * m;
        double2 dot = make_double2(0, 0);
        for (i64 i = k + 1 + lane; i < m; i += 32) cfmac(dot, ck[i], cj[i]);
        dot = warp_sum2(dot);
        cfmac(dot, v0, cj[k]);
        const double2 w = cscale(beta, dot);
        for (i64 i = k + 1 + lane; i < m; i += 32) cj[i] = csub(cj[i], cmul(ck[i], w));
        if (lane == 0) cj[k] = csub(cj[k], cmul(v0, w));
      }
    }
    __syncthreads();
    if (tid == 0) ck[k] = s_rkk;
    __syncthreads();
  }
  const int r = k;
  if (tid == 0) {
    rank_out[blockIdx.x] = r;
    sat_out[blockIdx.x] = s_sat;
  }
  // T = R11^{-1} R12 in place (rows 0..r-1 of columns r..n-1), a warp per column
  for (int j = r + warp; j < n; j += kWideWarps) {
    double2* cj = a + static_cast<i64>(j) * m;
    for (int i = r - 1; i >= 0; --i) {
      double2 s = make_double2(0, 0);
      for (int l = i + 1 + lane; l < r; l += 32) cfma(s, a[i + static_cast<i64>(l) * m], cj[l]);
      s = warp_sum2(s);
      if (lane == 0) cj[i] = cdiv(csub(cj[i], s), a[i + static_cast<i64>(i) * m]);
      __syncwarp();
    }
  }
  // skeleton in ascending column order: position of pivot p among the first r
  for (int p = tid; p < r; p += kWideThreads) {
    int c = 0;
    for (int q = 0; q < r; ++q) c += perm[q] < perm[p];
    pos[p] = c;
    skel_all[J.n_off + c] = perm[p] + 1;
  }
  double2* interp = interp_all + J.i_off;  // r x n column-major
  for (i64 e = tid; e < static_cast<i64>(r) * n; e += kWideThreads) interp[e] = make_double2(0, 0);
  __syncthreads();
  for (int p = tid; p < r; p += kWideThreads) interp[pos[p] + static_cast<i64>(perm[p]) * r] = make_double2(1, 0);
  for (i64 e = tid; e < static_cast<i64>(r) * (n - r); e += kWideThreads) {
    const int p = static_cast<int>(e % r), j = r + static_cast<int>(e / r);
    interp[pos[p] + static_cast<i64>(perm[j]) * r] = a[p + static_cast<i64>(j) * m];
  }
}

}  // namespace

void launch_wide_ids(i64 njobs, const WideIdJob* jobs, double2* A, double* nrm, int* perm, int* pos, double tol,
                     int* rank, int* sat, int* skel, double2* interp, cudaStream_t st) {
  if (njobs == 0) return;
  k_qrcp_wide<<<static_cast<unsigned>(njobs), kWideThreads, 0, st>>>(jobs, A, nrm, perm, pos, tol, rank, sat, skel,
                                                                    interp);
  TBF_CUDA(cudaGetLastError());
}

}  // namespace tbf
