// Fused level contractions for the apply (Alg. 2, 185,
// 201, 203; reference mode_product_blockdiag tensor.cpp:136-166 semantics).
//
// The block-diagonal factor of every level splits the level into independent
// boxes: out_box = in_box x_1 M_1 x_2 M_2 ... x_d M_d.  One CTA per box:
//   phase 0  the box descriptor is copied to shared memory by the whole CTA
//   phase 1  the d factor blocks AND the input box are staged into shared
//            memory in a single round trip (all loads independent)
//   phase 2  the d mode products run back to back in shared memory
//   phase 3  the last mode writes the output box (global strides: the V-bar
//            input slab / U-bar output slab are views of F and G)
// P levels (l >= 1) write per-child contributions; k_sum_parent then adds the
// 2^d children of every parent in ascending order (deterministic, no atomics).
// All index arithmetic is 32-bit (box sizes are far below 2^31).
#include "kernels.h"

namespace tbf {

namespace {

constexpr int kBoxThreads = 1024;

// M(a, x): transpose = 0: B(r x w)(a, x);  transpose = 1: B(x, a)
__device__ __forceinline__ int mat_idx(int mrows, int transpose, int a, int x) {
  return transpose ? x + a * mrows : a + x * mrows;
}

// n / d and n % d for 0 <= n < 2^24, 1 <= d < 2^16 with one 64-bit multiply:
// q = (n * ceil(2^40 / d)) >> 40 is exact in that range (error < 2^-16 < 1/d).
struct FastDiv {
  unsigned long long m;
  int d;
  __device__ __forceinline__ void init(int dd) {
    d = dd;
    m = ((1ULL << 40) + static_cast<unsigned long long>(dd) - 1) / static_cast<unsigned long long>(dd);
  }
  __device__ __forceinline__ int div(int n) const {
    return static_cast<int>((static_cast<unsigned long long>(n) * m) >> 40);
  }
};

template <class T>
__device__ __forceinline__ void copy_desc(T* dst, const T* src) {
  static_assert(sizeof(T) % 8 == 0, "descriptor must be 8-byte sized");
  const long long* s = reinterpret_cast<const long long*>(src);
  long long* d = reinterpret_cast<long long*>(dst);
  for (int i = threadIdx.x; i < static_cast<int>(sizeof(T) / 8); i += blockDim.x) d[i] = s[i];
}

// DD = d (modes per side) is a template parameter so every per-mode array
// lives in registers and every loop over modes is unrolled.
template <int DD>
__global__ void __launch_bounds__(kBoxThreads) k_box(const BoxItem* __restrict__ items,
                                                     const BoxTerm* __restrict__ terms, BoxLaunchInfo info,
                                                     const double2* __restrict__ mats,
                                                     const double2* __restrict__ in, double2* __restrict__ out) {
  constexpr int D = DD + 1;  // + nv mode (never contracted)
  extern __shared__ __align__(16) double2 sm[];
  __shared__ BoxItem it;
  __shared__ BoxTerm tm;
  const int tid = threadIdx.x;
  copy_desc(&it, items + blockIdx.x);  // items and terms are 1:1 (same index)
  copy_desc(&tm, terms + blockIdx.x);
  __syncthreads();
  int ext[D];
  long long istr[D];
  int isize = 1;
#pragma unroll
  for (int p = 0; p < DD; ++p) {
    ext[p] = tm.in_ext[p];
    isize *= ext[p];
  }
  ext[DD] = info.nv;
  isize *= info.nv;
#pragma unroll
  for (int p = 0; p < D; ++p) istr[p] = tm.in_stride[p];
  // shared layout: [input box (leading dim e0+1) | factors | ping | pong]
  double2* xin = sm;
  double2* smat = xin + info.smem_elems_in;
  double2* bufA = smat + info.smem_elems_mat;
  double2* bufB = bufA + info.smem_elems_a;
  int moff[DD + 1];
  moff[0] = 0;
#pragma unroll
  for (int k = 0; k < DD; ++k) moff[k + 1] = moff[k] + tm.mrows[k] * tm.mcols[k];
  const int msize = moff[DD];
  const int ld0 = ext[0] + 1;
  // ---- stage the factor blocks (linear copy) and the input box (one row =
  // one mode-0 fibre per thread: the row base is decoded once, then the
  // fibre is fetched with independent loads)
  for (int q = tid; q < msize; q += kBoxThreads) {
    int k = 0;
#pragma unroll
    for (int kk = 1; kk < DD; ++kk)
      if (q >= moff[kk]) k = kk;
    smat[q] = __ldg(mats + tm.mat_off[k] + (q - moff[k]));
  }
  {
    const int e0 = ext[0];
    const int nrows = isize / e0;
    for (int row = tid; row < nrows; row += kBoxThreads) {
      long long addr = tm.in_off;
      int rem = row;
#pragma unroll
      for (int p = 1; p < D; ++p) {
        const int q = rem / ext[p];
        addr += static_cast<long long>(rem - q * ext[p]) * istr[p];
        rem = q;
      }
      const double2* srcp = in + addr;
      double2* dstp = xin + ld0 * row;
      constexpr int kU = 8;
      for (int x0 = 0; x0 < e0; x0 += kU) {
        double2 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u)
          if (x0 + u < e0) v[u] = __ldg(srcp + static_cast<long long>(x0 + u) * istr[0]);
#pragma unroll
        for (int u = 0; u < kU; ++u)
          if (x0 + u < e0) dstp[x0 + u] = v[u];
      }
    }
  }
  __syncthreads();
  // ---- mode products, one output element per thread-iteration
  const double2* src = xin;
  double2* dst = bufA;
#pragma unroll
  for (int k = 0; k < DD; ++k) {
    const double2* M = smat + moff[k];
    const int mrows = tm.mrows[k];
    const int ein = ext[k];
    const int eout = info.transpose ? tm.mcols[k] : tm.mrows[k];
    // M(a, x) = M[a * sa + x * sx]
    const int sa = info.transpose ? mrows : 1;
    const int sx = info.transpose ? 1 : mrows;
    int below = 1, above = 1;
#pragma unroll
    for (int p = 0; p < D; ++p) {
      if (p < k) below *= ext[p];
      if (p > k) above *= ext[p];
    }
    // source element (b, x, c) at b + sb * x + sc * c
    const int sb = (k == 0) ? 1 : below;
    const int sc = (k == 0) ? ld0 : below * ein;
    const int total = below * eout * above;
    FastDiv fb, fa;
    fb.init(below);
    fa.init(eout > 0 ? eout : 1);
    FastDiv fe[D];
    if (k == DD - 1) {
#pragma unroll
      for (int p = 0; p < D; ++p) fe[p].init(ext[p] > 0 ? ext[p] : 1);
    }
    for (int e = tid; e < total; e += kBoxThreads) {
      const int r2 = fb.div(e);
      const int b = e - r2 * below;
      const int c = fa.div(r2);
      const int a = r2 - c * eout;
      const double2* xs = src + b + sc * c;
      const double2* Ma = M + a * sa;
      double2 s0 = make_double2(0, 0), s1 = make_double2(0, 0), s2 = make_double2(0, 0), s3 = make_double2(0, 0);
      int x = 0;
      for (; x + 3 < ein; x += 4) {
        cfma(s0, xs[sb * x], Ma[sx * x]);
        cfma(s1, xs[sb * (x + 1)], Ma[sx * (x + 1)]);
        cfma(s2, xs[sb * (x + 2)], Ma[sx * (x + 2)]);
        cfma(s3, xs[sb * (x + 3)], Ma[sx * (x + 3)]);
      }
      for (; x < ein; ++x) cfma(s0, xs[sb * x], Ma[sx * x]);
      const double2 sum = cadd(cadd(s0, s1), cadd(s2, s3));
      if (k < DD - 1) {
        dst[e] = sum;
      } else {
        // output box element (b; a; c) -> global address
        long long addr = it.out_off + static_cast<long long>(a) * it.out_stride[k];
        int rb = b;
#pragma unroll
        for (int p = 0; p < D; ++p)
          if (p < k) {
            const int q = fe[p].div(rb);
            addr += static_cast<long long>(rb - q * ext[p]) * it.out_stride[p];
            rb = q;
          }
        int rc = c;
#pragma unroll
        for (int p = 0; p < D; ++p)
          if (p > k) {
            const int q = fe[p].div(rc);
            addr += static_cast<long long>(rc - q * ext[p]) * it.out_stride[p];
            rc = q;
          }
        out[addr] = sum;
      }
    }
    if (k < DD - 1) {
      ext[k] = eout;
      __syncthreads();
      src = dst;
      dst = (dst == bufA) ? bufB : bufA;
    }
  }
}

// ordered child sums: CTAs map to (parent, 1024-element chunk); children are
// added in ascending nu (deterministic)
__global__ void __launch_bounds__(256) k_sum_parent(const SumDesc* __restrict__ ds, const int* __restrict__ cta_map,
                                                    const double2* __restrict__ in, double2* __restrict__ out) {
  const int pidx = cta_map[2 * blockIdx.x], chunk = cta_map[2 * blockIdx.x + 1];
  const SumDesc* D = ds + pidx;
  const int nchild = D->nchild;
  const long long total = D->total, out_off = D->out_off;
  long long coff[1 << kMaxD];
  for (int c = 0; c < nchild; ++c) coff[c] = D->child_off[c];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const long long q = static_cast<long long>(chunk) * 1024 + u * 256 + threadIdx.x;
    if (q >= total) break;
    double2 acc = in[coff[0] + q];
    for (int c = 1; c < nchild; ++c) acc = cadd(acc, in[coff[c] + q]);
    out[out_off + q] = acc;
  }
}

}  // namespace

size_t box_smem_bytes(const BoxLaunchInfo& info) {
  return sizeof(double2) *
         static_cast<size_t>(info.smem_elems_in + info.smem_elems_mat + info.smem_elems_a + info.smem_elems_b);
  // smem_elems_in includes the padding of the leading dimension (host adds it)
}

void launch_box(i64 nitems, const BoxItem* items, const BoxTerm* terms, const BoxLaunchInfo& info,
                const double2* mats, const double2* in, double2* out, cudaStream_t st) {
  if (nitems == 0) return;
  const size_t smem = box_smem_bytes(info);
  switch (info.d) {
#define TBF_BOX_CASE(DD)                                                                                     \
  case DD:                                                                                                    \
    TBF_CUDA(cudaFuncSetAttribute(k_box<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));      \
    k_box<DD><<<static_cast<unsigned>(nitems), kBoxThreads, smem, st>>>(items, terms, info, mats, in, out); \
    break;
    TBF_BOX_CASE(1)
    TBF_BOX_CASE(2)
    TBF_BOX_CASE(3)
    TBF_BOX_CASE(4)
    TBF_BOX_CASE(5)
    TBF_BOX_CASE(6)
#undef TBF_BOX_CASE
    default:
      throw std::runtime_error("launch_box: d out of range");
  }
  TBF_CUDA(cudaGetLastError());
}

void launch_sum_parent(i64 nctas, const SumDesc* d, const int* cta_map, const double2* in, double2* out,
                       cudaStream_t st) {
  if (nctas == 0) return;
  k_sum_parent<<<static_cast<unsigned>(nctas), 256, 0, st>>>(d, cta_map, in, out);
  TBF_CUDA(cudaGetLastError());
}

}  // namespace tbf
