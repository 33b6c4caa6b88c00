// Contraction kernels (Alg. 2).
//   k_mode_product  batched block-diagonal mode-j products: the V-bar / W / P /
//                   U-bar steps (tensor.cpp:136-166 semantics, one launch per
//                   (level, mode) covering every (tau, s) or (t, nu) item)
//   k_gemv          middle-level core contraction G_{t,s} = K(tbar,sbar) F_{t,s}
//                   (id.cpp:321 pattern): HBM-bound stream of the cores, one
//                   warp per core row, 16-B loads, F_{t,s} staged in SMEM
//   k_sum_children  ordered accumulation G_{t,p_nu} = sum_nu (...) (Alg. 2 l. 203)
#include "kernels.h"

namespace tbf {

namespace {

__device__ __forceinline__ i64 find_item(const i64* __restrict__ work_off_base, size_t stride_bytes, i64 n,
                                         i64 e) {
  // binary search over item work offsets (monotone), returns item with off <= e
  i64 lo = 0, hi = n - 1;
  while (lo < hi) {
    const i64 mid = (lo + hi + 1) >> 1;
    const i64 off = *reinterpret_cast<const i64*>(reinterpret_cast<const char*>(work_off_base) + mid * stride_bytes);
    if (off <= e) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void k_mode_product(i64 nitems, const MPStep* __restrict__ steps, i64 total_out,
                               const Blk* __restrict__ blks, const double2* __restrict__ mats,
                               const double2* __restrict__ in, double2* __restrict__ out) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= total_out) return;
  const i64 it = find_item(&steps[0].work_off, sizeof(MPStep), nitems, e);
  const MPStep& S = steps[it];
  i64 rem = e - S.work_off;
  i64 in_addr = S.in_off, out_addr = S.out_off;
  int o = 0;
  for (int p = 0; p < S.nd; ++p) {
    const int x = static_cast<int>(rem % S.ext[p]);
    rem /= S.ext[p];
    out_addr += x * S.out_stride[p];
    if (p == S.mode) o = x;
    else in_addr += x * S.in_stride[p];
  }
  // block containing output index o
  int b = 0;
  for (; b + 1 < S.nblk; ++b) {
    const Blk& nb = blks[S.blk_off + b + 1];
    if (o < nb.out_start) break;
  }
  const Blk B = blks[S.blk_off + b];
  const int ol = o - B.out_start;
  const int bin = S.transpose ? B.rows : B.cols;
  const i64 sk = S.in_stride[S.mode];
  const double2* M = mats + B.mat_off;
  const double2* X = in + in_addr + static_cast<i64>(B.in_start) * sk;
  double2 acc = make_double2(0, 0);
  if (S.transpose) {  // out_o = sum_i B(i, o) x_i
    const double2* col = M + static_cast<i64>(ol) * B.rows;
    for (int i = 0; i < bin; ++i) cfma(acc, X[i * sk], col[i]);
  } else {  // out_o = sum_i B(o, i) x_i
    for (int i = 0; i < bin; ++i) cfma(acc, X[i * sk], M[ol + static_cast<i64>(i) * B.rows]);
  }
  out[out_addr] = acc;
}

constexpr int kGemvThreads = 256;
constexpr int kGemvRowsPerCta = 32;

__device__ __forceinline__ double4 ld_stream(const double4* p) {
  double4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2+16];" : "=d"(r.z), "=d"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_stream2(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

// grid: one CTA per (pair, 32-row chunk); each warp walks 4 rows
__global__ void __launch_bounds__(kGemvThreads) k_gemv(const int* __restrict__ cta_pair,
                                                       const GemvDesc* __restrict__ ds, int nv,
                                                       const double2* __restrict__ cores,
                                                       const double2* __restrict__ x, double2* __restrict__ y) {
  extern __shared__ __align__(16) double2 sx[];
  const i64 cta = blockIdx.x;
  const GemvDesc D = ds[cta_pair[cta]];
  const int chunk = static_cast<int>(cta - D.cta_off);
  for (int i = threadIdx.x; i < D.C * nv; i += kGemvThreads) sx[i] = x[D.x_off + i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = chunk * kGemvRowsPerCta;
  for (int rr = warp; rr < kGemvRowsPerCta; rr += kGemvThreads / 32) {
    const int r = r0 + rr;
    if (r >= D.R) break;
    const double2* row = cores + D.core_off + static_cast<i64>(r) * D.C;
    for (int v = 0; v < nv; ++v) {
      double2 acc0 = make_double2(0, 0), acc1 = make_double2(0, 0);
      const double2* xv = sx + v * D.C;
      int c = lane;
      for (; c + 96 < D.C; c += 128) {
        const double2 a0 = ld_stream2(row + c), a1 = ld_stream2(row + c + 32);
        const double2 a2 = ld_stream2(row + c + 64), a3 = ld_stream2(row + c + 96);
        cfma(acc0, a0, xv[c]);
        cfma(acc1, a1, xv[c + 32]);
        cfma(acc0, a2, xv[c + 64]);
        cfma(acc1, a3, xv[c + 96]);
      }
      for (; c < D.C; c += 32) cfma(acc0, ld_stream2(row + c), xv[c]);
      acc0 = cadd(acc0, acc1);
      acc0 = warp_sum2(acc0);
      if (lane == 0) y[D.y_off + r + static_cast<i64>(v) * D.R] = acc0;
    }
  }
}

__global__ void k_sum_children(i64 n, const SumDesc* __restrict__ ds, i64 total, const double2* __restrict__ in,
                               double2* __restrict__ out) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const i64 it = find_item(&ds[0].work_off, sizeof(SumDesc), n, e);
  const SumDesc& D = ds[it];
  const i64 q = e - D.work_off;
  double2 acc = in[D.child_off[0] + q];
  for (int c = 1; c < D.nchild; ++c) acc = cadd(acc, in[D.child_off[c] + q]);
  out[D.out_off + q] = acc;
}

}  // namespace

void launch_mode_product(i64 nitems, const MPStep* steps, i64 total_out, const Blk* blks, const double2* mats,
                         const double2* in, double2* out, cudaStream_t st) {
  if (total_out == 0) return;
  k_mode_product<<<static_cast<unsigned>((total_out + 255) / 256), 256, 0, st>>>(nitems, steps, total_out, blks, mats,
                                                                                in, out);
  TBF_CUDA(cudaGetLastError());
}

void launch_gemv(const int* cta_pair, const GemvDesc* d, i64 nctas, int nv, const double2* cores, const double2* x,
                 double2* y, int max_c, cudaStream_t st) {
  if (nctas == 0) return;
  const size_t smem = sizeof(double2) * static_cast<size_t>(max_c) * nv;
  TBF_CUDA(cudaFuncSetAttribute(k_gemv, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
  k_gemv<<<static_cast<unsigned>(nctas), kGemvThreads, smem, st>>>(cta_pair, d, nv, cores, x, y);
  TBF_CUDA(cudaGetLastError());
}

void launch_sum_children(i64 n, const SumDesc* d, i64 total, const double2* in, double2* out, cudaStream_t st) {
  if (total == 0) return;
  k_sum_children<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(n, d, total, in, out);
  TBF_CUDA(cudaGetLastError());
}

int gemv_rows_per_cta() { return kGemvRowsPerCta; }

}  // namespace tbf
