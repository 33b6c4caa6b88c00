// Middle-level core generation (Alg. 1 step 3, lines 155-160;
// id.cpp:285 subtensor_at at the skeleton multi-sets) and the K-check direct
// dense sums used for the accuracy gate.
//
// Cores are stored ROW-major (one contiguous row per target skeleton
// multi-index), i.e. the transpose of the reference's column-major
// matricization, so the apply GEMV streams each row with coalesced 16-B loads.
#include <cub/cub.cuh>

#include "kernels.h"

namespace tbf {

namespace {

__global__ void k_cores(KSpec ks, i64 npairs, const PairDesc* __restrict__ pairs, i64 total,
                        const int* __restrict__ uskel, const int* __restrict__ vskel, double2* __restrict__ cores) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= total) return;
  i64 lo = 0, hi = npairs - 1;
  while (lo < hi) {
    const i64 mid = (lo + hi + 1) >> 1;
    if (pairs[mid].work_off <= e) lo = mid;
    else hi = mid - 1;
  }
  const PairDesc& P = pairs[lo];
  const i64 q = e - P.work_off;
  const int col = static_cast<int>(q % P.C);
  const int row = static_cast<int>(q / P.C);
  int ii[kMaxD], jj[kMaxD];
  int rem = row;
  for (int k = 0; k < ks.d; ++k) {
    ii[k] = uskel[P.rs_off[k] + rem % P.rr[k]];
    rem /= P.rr[k];
  }
  rem = col;
  for (int k = 0; k < ks.d; ++k) {
    jj[k] = vskel[P.cs_off[k] + rem % P.rc[k]];
    rem /= P.rc[k];
  }
  cores[P.core_off + q] = kernel_entry(ks, ii, jj);
}

// one CTA per sampled output row; Neumaier-compensated sums
__global__ void __launch_bounds__(512) k_dense_rows(KSpec ks, const i64* __restrict__ rows, const double2* __restrict__ F, int nv,
                             i64 N, double2* __restrict__ out, i64 nrows) {
  __shared__ double red[4][32];
  const i64 r = blockIdx.x;
  int ii[kMaxD], jj[kMaxD];
  i64 rem = rows[r];
  for (int p = 0; p < ks.d; ++p) {
    ii[p] = static_cast<int>(rem % ks.n) + 1;
    rem /= ks.n;
  }
  for (int v = 0; v < nv; ++v) {
    double sr = 0, si = 0, cr = 0, ci = 0;
    for (i64 f = threadIdx.x; f < N; f += blockDim.x) {
      i64 rr = f;
      for (int p = 0; p < ks.d; ++p) {
        jj[p] = static_cast<int>(rr % ks.n) + 1;
        rr /= ks.n;
      }
      const double2 k = kernel_entry(ks, ii, jj);
      const double2 pr = cmul(k, F[f + v * N]);
      double t = sr + pr.x;
      cr += fabs(sr) >= fabs(pr.x) ? (sr - t) + pr.x : (pr.x - t) + sr;
      sr = t;
      t = si + pr.y;
      ci += fabs(si) >= fabs(pr.y) ? (si - t) + pr.y : (pr.y - t) + si;
      si = t;
    }
    double a = sr + cr, b = si + ci;
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
      red[0][warp] = a;
      red[1][warp] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double A = 0, B = 0;
      for (int q = 0; q < static_cast<int>(blockDim.x / 32); ++q) {
        A += red[0][q];
        B += red[1][q];
      }
      out[r + v * nrows] = make_double2(A, B);
    }
    __syncthreads();
  }
}

struct Counts12 {
  i64 c[kMaxModes];
  i64 off[kMaxModes];
};
__global__ void k_subtensor(KSpec ks, Counts12 cn, const int* __restrict__ lists, i64 total, double2* __restrict__ out) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= total) return;
  int ii[kMaxD], jj[kMaxD];
  i64 rem = e;
  for (int p = 0; p < 2 * ks.d; ++p) {
    const int v = lists[cn.off[p] + rem % cn.c[p]];
    rem /= cn.c[p];
    if (p < ks.d) ii[p] = v;
    else jj[p - ks.d] = v;
  }
  out[e] = kernel_entry(ks, ii, jj);
}

__global__ void k_count_nonfinite(const double2* __restrict__ x, long long n, unsigned long long* out) {
  unsigned long long c = 0;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double2 v = x[i];
    c += !(isfinite(v.x) && isfinite(v.y));
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

}  // namespace

unsigned long long count_nonfinite(const double2* x, i64 n, cudaStream_t st) {
  unsigned long long* d = nullptr;
  TBF_CUDA(cudaMallocAsync(&d, sizeof(unsigned long long), st));
  TBF_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), st));
  if (n > 0) k_count_nonfinite<<<148 * 8, 256, 0, st>>>(x, n, d);
  unsigned long long h = 0;
  TBF_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
  TBF_CUDA(cudaStreamSynchronize(st));
  TBF_CUDA(cudaFreeAsync(d, st));
  return h;
}

void launch_subtensor(const KSpec& ks, const i64* counts_h, const int* lists, i64 total, double2* out,
                      cudaStream_t st) {
  if (total == 0) return;
  Counts12 cn{};
  i64 off = 0;
  for (int p = 0; p < 2 * ks.d; ++p) {
    cn.c[p] = counts_h[p];
    cn.off[p] = off;
    off += counts_h[p];
  }
  k_subtensor<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(ks, cn, lists, total, out);
  TBF_CUDA(cudaGetLastError());
}

void launch_cores(const KSpec& ks, i64 npairs, const PairDesc* pairs, i64 total_entries, const int* uskel,
                  const int* vskel, double2* cores, cudaStream_t st) {
  if (total_entries == 0) return;
  k_cores<<<static_cast<unsigned>((total_entries + 255) / 256), 256, 0, st>>>(ks, npairs, pairs, total_entries, uskel,
                                                                             vskel, cores);
  TBF_CUDA(cudaGetLastError());
}

void launch_dense_rows(const KSpec& ks, i64 nrows, const i64* rows, const double2* F, int nv, double2* out,
                       cudaStream_t st) {
  i64 N = 1;
  for (int p = 0; p < ks.d; ++p) N *= ks.n;
  k_dense_rows<<<static_cast<unsigned>(nrows), 512, 0, st>>>(ks, rows, F, nv, N, out, nrows);
  TBF_CUDA(cudaGetLastError());
}


// ---- device-side bookkeeping (construction at config-4 scale: 1e8 slots /
// 1.7e7 pairs per level would otherwise be uploaded from host mirrors)
namespace {
__global__ void k_slot_sizes(i64 n, const int* __restrict__ rank, const int* __restrict__ width, i64* __restrict__ a,
                             i64* __restrict__ b) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  a[i] = rank[i];
  b[i] = static_cast<i64>(rank[i]) * width[i];
}
__global__ void k_layout_pairs(int d, i64 nmid, const int* __restrict__ urank, const i64* __restrict__ uskel_off,
                               const int* __restrict__ vrank, const i64* __restrict__ vskel_off,
                               PairDesc* __restrict__ pairs, i64* __restrict__ work) {
  const i64 p = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= nmid * nmid) return;
  const i64 s = p / nmid, t = p % nmid;
  PairDesc pd;
  pd.R = 1;
  pd.C = 1;
  for (int k = 0; k < kMaxD; ++k) {
    pd.rr[k] = pd.rc[k] = 0;
    pd.rs_off[k] = pd.cs_off[k] = 0;
  }
  for (int k = 0; k < d; ++k) {
    const i64 us = (t * nmid + s) * d + k;  // U slot (Lc, t, nu=s, k, j=0)
    const i64 vs = (s * nmid + t) * d + k;  // V slot (Lc, s, tau=t, k, j=0)
    pd.rr[k] = urank[us];
    pd.rc[k] = vrank[vs];
    pd.rs_off[k] = uskel_off[us];
    pd.cs_off[k] = vskel_off[vs];
    pd.R *= pd.rr[k];
    pd.C *= pd.rc[k];
  }
  pd.core_off = 0;
  pd.work_off = 0;
  pairs[p] = pd;
  work[p] = static_cast<i64>(pd.R) * pd.C;
}
__global__ void k_pair_offsets(i64 np, const i64* __restrict__ off, PairDesc* __restrict__ pairs) {
  const i64 p = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= np) return;
  pairs[p].core_off = off[p];
  pairs[p].work_off = off[p];
}
template <class T>
void exclusive_sum(const i64* in, i64* out, i64 n, cudaStream_t st, T) {
  size_t bytes = 0;
  TBF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, st));
  void* tmp = nullptr;
  TBF_CUDA(cudaMallocAsync(&tmp, std::max<size_t>(bytes, 16), st));
  TBF_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, n, st));
  TBF_CUDA(cudaFreeAsync(tmp, st));
}
}  // namespace

void scan_slot_offsets(i64 n, const int* rank, const int* width, i64* skel_off, i64* interp_off, cudaStream_t st) {
  if (n == 0) return;
  i64* a = nullptr;
  TBF_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&a), sizeof(i64) * 2 * n, st));
  k_slot_sizes<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(n, rank, width, a, a + n);
  TBF_CUDA(cudaGetLastError());
  exclusive_sum(a, skel_off, n, st, 0);
  exclusive_sum(a + n, interp_off, n, st, 0);
  TBF_CUDA(cudaFreeAsync(a, st));
}

void layout_pairs_device(int d, i64 nmid, const int* urank, const i64* uskel_off, const int* vrank,
                         const i64* vskel_off, PairDesc* pairs, cudaStream_t st) {
  const i64 np = nmid * nmid;
  i64* w = nullptr;
  TBF_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&w), sizeof(i64) * 2 * np, st));
  k_layout_pairs<<<static_cast<unsigned>((np + 255) / 256), 256, 0, st>>>(d, nmid, urank, uskel_off, vrank, vskel_off,
                                                                          pairs, w);
  TBF_CUDA(cudaGetLastError());
  exclusive_sum(w, w + np, np, st, 0);
  k_pair_offsets<<<static_cast<unsigned>((np + 255) / 256), 256, 0, st>>>(np, w + np, pairs);
  TBF_CUDA(cudaGetLastError());
  TBF_CUDA(cudaFreeAsync(w, st));
}

}  // namespace tbf
