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
#include <cooperative_groups.h>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace tbf {

namespace {

constexpr int kBoxThreads = 256;

// debug tracing (OIOBF_BOX_TRACE): per-CTA %globaltimer stamps at phase
// boundaries; never enabled in the product path
__device__ unsigned long long* g_box_trace = nullptr;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define BOX_STAMP(slot)                                                      \
  do {                                                                       \
    if (g_box_trace && threadIdx.x == 0) {                                   \
      g_box_trace[blockIdx.x * 8 + (slot)] = gtime();                        \
      if ((slot) == 0) g_box_trace[blockIdx.x * 8 + 5] = clock64();          \
      if ((slot) == 4) g_box_trace[blockIdx.x * 8 + 6] = clock64();          \
    }                                                                        \
  } while (0)

// M(a, x): transpose = 0: B(r x w)(a, x);  transpose = 1: B(x, a)
__device__ __forceinline__ int mat_idx(int mrows, int transpose, int a, int x) {
  return transpose ? x + a * mrows : a + x * mrows;
}

// n / d for 0 <= n < 2^24, d >= 1: float reciprocal estimate (off by at most
// one in that range) plus one integer correction; no division subroutine.
__device__ __forceinline__ int qdiv(int n, int d) {
  int q = __float2int_rz(__fdividef(static_cast<float>(n), static_cast<float>(d)));
  const int r = n - q * d;
  q += (r >= d) - (r < 0);
  return q;
}

template <class T>
__device__ __forceinline__ void copy_desc(T* dst, const T* src) {
  static_assert(sizeof(T) % 8 == 0, "descriptor must be 8-byte sized");
  const long long* s = reinterpret_cast<const long long*>(src);
  long long* d = reinterpret_cast<long long*>(dst);
  for (int i = threadIdx.x; i < static_cast<int>(sizeof(T) / 8); i += blockDim.x) d[i] = s[i];
}

// Compact on purpose: this kernel does little work per CTA, so its cost is
// dominated by latency and by cold instruction fetch; the mode loop is a
// runtime loop (per-mode state in shared memory), divisions use qdiv().
__global__ void __launch_bounds__(kBoxThreads) k_box(const BoxItem* __restrict__ items,
                                                     const BoxTerm* __restrict__ terms, BoxLaunchInfo info,
                                                     const double2* __restrict__ mats,
                                                     const double2* __restrict__ in, double2* __restrict__ out) {
  extern __shared__ __align__(16) double2 sm[];
  __shared__ BoxItem it;
  __shared__ BoxTerm tm;
  __shared__ int s_ext[kMaxTM];
  __shared__ int s_moff[kMaxD + 1];
  __shared__ int s_z0, s_isize;
  __shared__ long long s_inoff;
  BOX_STAMP(0);
  const int tid = threadIdx.x;
  const int cs = info.cs;
  const int crank = cs > 1 ? static_cast<int>(blockIdx.x % cs) : 0;
  const int item = cs > 1 ? static_cast<int>(blockIdx.x / cs) : static_cast<int>(blockIdx.x);
  copy_desc(&it, items + item);  // items and terms are 1:1 (same index)
  copy_desc(&tm, terms + item);
  __syncthreads();
  const int d = info.d, D = d + 1;  // + nv mode (never contracted)
  if (tid == 0) {
    // cluster split: this CTA contracts the slab [z0, z1) of the last input mode
    const int elast = tm.in_ext[d - 1];
    const int z0 = qdiv(crank * elast, cs), z1 = qdiv((crank + 1) * elast, cs);
    int isize = 1;
    for (int p = 0; p < d; ++p) {
      s_ext[p] = p == d - 1 ? z1 - z0 : tm.in_ext[p];
      isize *= s_ext[p];
    }
    s_ext[d] = info.nv;
    s_isize = isize * info.nv;
    s_z0 = z0;
    s_inoff = tm.in_off + static_cast<long long>(z0) * tm.in_stride[d - 1];
    s_moff[0] = 0;
    for (int k = 0; k < d; ++k) s_moff[k + 1] = s_moff[k] + tm.mrows[k] * tm.mcols[k];
  }
  __syncthreads();
  BOX_STAMP(1);
  const int e0 = s_ext[0];
  const int ld0 = e0 + 1;
  double2* xin = sm;  // input slab, leading dimension e0 + 1
  double2* smat = xin + info.smem_elems_in;
  double2* bufA = smat + info.smem_elems_mat;
  double2* bufB = bufA + info.smem_elems_a;
  double2* acc = bufB + info.smem_elems_b;
  // ---- stage the factor blocks (linear) and the input slab (one mode-0
  // fibre per thread-iteration, up to 4 independent loads in flight)
  const int msize = s_moff[d];
  for (int q = tid; q < msize; q += kBoxThreads) {
    int k = 0;
    while (k + 1 < d && q >= s_moff[k + 1]) ++k;
    smat[q] = __ldg(mats + tm.mat_off[k] + (q - s_moff[k]));
  }
  const int nrows = e0 > 0 ? s_isize / e0 : 0;
  const long long st0 = tm.in_stride[0];
  for (int row = tid; row < nrows; row += kBoxThreads) {
    long long addr = s_inoff;
    int rem = row;
    for (int p = 1; p < D; ++p) {
      const int q = qdiv(rem, s_ext[p]);
      addr += static_cast<long long>(rem - q * s_ext[p]) * tm.in_stride[p];
      rem = q;
    }
    const double2* srcp = in + addr;
    double2* dstp = xin + ld0 * row;
    for (int x0 = 0; x0 < e0; x0 += 4) {
      double2 v0, v1, v2, v3;
      v0 = __ldg(srcp + x0 * st0);
      if (x0 + 1 < e0) v1 = __ldg(srcp + (x0 + 1) * st0);
      if (x0 + 2 < e0) v2 = __ldg(srcp + (x0 + 2) * st0);
      if (x0 + 3 < e0) v3 = __ldg(srcp + (x0 + 3) * st0);
      dstp[x0] = v0;
      if (x0 + 1 < e0) dstp[x0 + 1] = v1;
      if (x0 + 2 < e0) dstp[x0 + 2] = v2;
      if (x0 + 3 < e0) dstp[x0 + 3] = v3;
    }
  }
  __syncthreads();
  BOX_STAMP(2);
  // ---- mode products, one output element per thread-iteration
  const int reps = (g_box_trace && info.nv < 0) ? 2 : 1;  // never true (nv >= 1): keeps layout
  int ext[kMaxTM];
  for (int rep = 0; rep < (g_box_trace ? 2 : 1); ++rep) {
  if (rep == 1) { __syncthreads(); BOX_STAMP(7); }
  (void)reps;
    const double2* src = xin;
    double2* dst = bufA;
    for (int p = 0; p < D; ++p) ext[p] = s_ext[p];
    for (int k = 0; k < d; ++k) {
      const bool last = (k == d - 1);
      const int mrows = tm.mrows[k];
      const int ein = ext[k];
      const int eout = info.transpose ? tm.mcols[k] : tm.mrows[k];
      const int sa = info.transpose ? mrows : 1;  // M(a, x) = M[a * sa + x * sx]
      const int sx = info.transpose ? 1 : mrows;
      const double2* M = smat + s_moff[k] + (last ? s_z0 * sx : 0);
      int below = 1, above = 1;
      for (int p = 0; p < D; ++p) {
        if (p < k) below *= ext[p];
        if (p > k) above *= ext[p];
      }
      const int sb = k == 0 ? 1 : below;  // source element (b, x, c) at b + sb*x + sc*c
      const int sc = k == 0 ? ld0 : below * ein;
      const int total = below * eout * above;
      double2* o = last ? (cs > 1 ? acc : nullptr) : dst;
      for (int e = tid; e < total; e += kBoxThreads) {
        const int r2 = qdiv(e, below);
        const int b = e - r2 * below;
        const int c = qdiv(r2, eout);
        const int a = r2 - c * eout;
        const double2* xs = src + b + sc * c;
        const double2* Ma = M + a * sa;
        double2 s0 = make_double2(0, 0), s1 = make_double2(0, 0);
        int x = 0;
        for (; x + 1 < ein; x += 2) {
          cfma(s0, xs[sb * x], Ma[sx * x]);
          cfma(s1, xs[sb * (x + 1)], Ma[sx * (x + 1)]);
        }
        if (x < ein) cfma(s0, xs[sb * x], Ma[sx * x]);
        const double2 sum = cadd(s0, s1);
        if (o) {
          o[e] = sum;
        } else {  // single-CTA box: write the output element straight to global
          long long addr = it.out_off + static_cast<long long>(a) * it.out_stride[k];
          int rb = b;
          for (int p = 0; p < k; ++p) {
            const int q = qdiv(rb, ext[p]);
            addr += static_cast<long long>(rb - q * ext[p]) * it.out_stride[p];
            rb = q;
          }
          int rc = c;
          for (int p = k + 1; p < D; ++p) {
            const int q = qdiv(rc, ext[p]);
            addr += static_cast<long long>(rc - q * ext[p]) * it.out_stride[p];
            rc = q;
          }
          out[addr] = sum;
        }
      }
      if (!last) {
        ext[k] = eout;
        __syncthreads();
        src = dst;
        dst = (dst == bufA) ? bufB : bufA;
      } else {
        ext[k] = eout;
      }
    }
  }
  BOX_STAMP(3);
  if (cs > 1) {
    // deterministic cluster reduction: CTA r sums its share of the output box
    // over ranks 0..cs-1 (in order) through distributed shared memory
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();
    int osize = 1;
    for (int p = 0; p < D; ++p) osize *= ext[p];
    const int e_begin = qdiv(crank * osize, cs);
    const int e_end = qdiv((crank + 1) * osize, cs);
    for (int e = e_begin + tid; e < e_end; e += kBoxThreads) {
      double2 sum = make_double2(0, 0);
      for (int q = 0; q < cs; ++q) sum = cadd(sum, cluster.map_shared_rank(acc, q)[e]);
      long long addr = it.out_off;
      int rem = e;
      for (int p = 0; p < D; ++p) {
        const int qd = qdiv(rem, ext[p]);
        addr += static_cast<long long>(rem - qd * ext[p]) * it.out_stride[p];
        rem = qd;
      }
      out[addr] = sum;
    }
    cluster.sync();  // keep every CTA's shared memory alive until all reads are done
  }
  BOX_STAMP(4);
}

// ordered child sums: CTAs map to (parent, 1024-element chunk); children are
// added in ascending nu (deterministic)
__global__ void __launch_bounds__(256) k_sum_parent(const SumDesc* __restrict__ ds, const int* __restrict__ cta_map,
                                                    const double2* __restrict__ in, double2* __restrict__ out) {
  __shared__ SumDesc D;
  const int pidx = cta_map[2 * blockIdx.x], chunk = cta_map[2 * blockIdx.x + 1];
  copy_desc(&D, ds + pidx);
  __syncthreads();
  const int nchild = D.nchild;
  // each thread owns 4 elements; all children's loads for a group of 8 are
  // issued before any add (no serialized load -> add chains)
  for (int u = 0; u < 4; ++u) {
    const long long q = static_cast<long long>(chunk) * 1024 + u * 256 + threadIdx.x;
    if (q >= D.total) break;
    double2 acc = make_double2(0, 0);
    for (int c0 = 0; c0 < nchild; c0 += 8) {
      double2 v[8];
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c0 + c < nchild) v[c] = in[D.child_off[c0 + c] + q];
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c0 + c < nchild) acc = cadd(acc, v[c]);
    }
    out[D.out_off + q] = acc;
  }
}

}  // namespace

size_t box_smem_bytes(const BoxLaunchInfo& info) {
  return sizeof(double2) * static_cast<size_t>(info.smem_elems_in + info.smem_elems_mat + info.smem_elems_a +
                                               info.smem_elems_b + info.smem_elems_acc);
  // smem_elems_in includes the padding of the leading dimension (host adds it)
}

void launch_box(i64 nitems, const BoxItem* items, const BoxTerm* terms, const BoxLaunchInfo& info,
                const double2* mats, const double2* in, double2* out, cudaStream_t st) {
  if (nitems == 0) return;
  const size_t smem = box_smem_bytes(info);
  if (info.d < 1 || info.d > kMaxD) throw std::runtime_error("launch_box: d out of range");
  TBF_CUDA(cudaFuncSetAttribute(k_box, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(nitems * info.cs));
  cfg.blockDim = dim3(kBoxThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(info.cs);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TBF_CUDA(cudaLaunchKernelEx(&cfg, k_box, items, terms, info, mats, in, out));
  TBF_CUDA(cudaGetLastError());
}

// largest number of co-resident clusters of size cs for a given smem footprint
int box_max_active_clusters(int cs, size_t smem) {
  TBF_CUDA(cudaFuncSetAttribute(k_box, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(cs * 148));
  cfg.blockDim = dim3(kBoxThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(cs);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  TBF_CUDA(cudaOccupancyMaxActiveClusters(&n, k_box, &cfg));
  return n;
}

void box_trace_enable(unsigned long long* buf) {
  TBF_CUDA(cudaMemcpyToSymbol(g_box_trace, &buf, sizeof(buf)));
}

void launch_sum_parent(i64 nctas, const SumDesc* d, const int* cta_map, const double2* in, double2* out,
                       cudaStream_t st) {
  if (nctas == 0) return;
  k_sum_parent<<<static_cast<unsigned>(nctas), 256, 0, st>>>(d, cta_map, in, out);
  TBF_CUDA(cudaGetLastError());
}

}  // namespace tbf
