// d = 2 boxes as two register-tiled complex GEMMs (Alg. 2 lines
// 183-203; reference mode_product_blockdiag tensor.cpp:136-166 semantics).
//
// One box (one CTA):  out = M0 . in . M1^T  per vector (M_k^T on the P/U side),
//   phase 1  T(x0, a1) = sum_x1 in(x0, x1) M1(a1, x1)     k-chunks of x1 staged
//   phase 2  out(a0, a1) = sum_x0 M0(a0, x0) T(x0, a1)    k-chunks of x0 staged
// Every thread owns a 4 x 4 output tile (rows / columns strided by the tile
// count, so the lanes of a warp read consecutive shared-memory rows and the
// other operand is a broadcast): 8 shared loads per 16 complex FMAs instead of
// k_box's one-column-per-thread chains.  The P-level child contributions are
// summed (ascending child) while the input chunks are staged.  Config 5's
// boxes (Radon, d = 2, ~76 x 76 -> ~48 x 48, 4,096 per level) are ~35% of its
// apply on k_box at ~20% of their FP64 floor.
#include "kernels.h"

namespace tbf {

namespace {

constexpr int kB2Threads = 256;
constexpr int kB2K = 16;  // contracted columns per staged chunk

__device__ __forceinline__ void b2_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void b2_pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

__global__ void __launch_bounds__(kB2Threads, 2) k_box2(const BoxDesc* __restrict__ descs, BoxLaunchInfo info,
                                                        const double2* __restrict__ mats,
                                                        const double2* __restrict__ in, double2* __restrict__ out) {
  extern __shared__ __align__(16) double2 sm[];
  __shared__ BoxDesc D;
  b2_pdl_trigger();
  {
    const long long* s = reinterpret_cast<const long long*>(descs + blockIdx.x);
    long long* d = reinterpret_cast<long long*>(&D);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(BoxDesc) / 8); i += kB2Threads) d[i] = s[i];
  }
  __syncthreads();
  const int e0 = D.ein[0], e1 = D.ein[1], o0 = D.eout[0], o1 = D.eout[1];
  const int tr = info.transpose, nv = info.nv, nsum = D.nsum;
  const double2* M0 = mats + D.mat_off[0];
  const double2* M1 = mats + D.mat_off[1];
  // element (a, x) of the o x e operator of mode k (stored r x w column-major)
  auto m0 = [&](int a, int x) { return __ldg(tr ? M0 + x + static_cast<long long>(e0) * a : M0 + a + static_cast<long long>(o0) * x); };
  auto m1 = [&](int a, int x) { return __ldg(tr ? M1 + x + static_cast<long long>(e1) * a : M1 + a + static_cast<long long>(o1) * x); };
  const int LT = e0 | 1;                  // T stored [a1][x0], odd leading dimension
  double2* Ts = sm;                       // o1 x LT
  double2* ch = Ts + static_cast<long long>(o1) * LT;  // staged chunks
  const int R1 = (e0 + 3) >> 2, C1 = (o1 + 3) >> 2;   // phase-1 tiles
  const int R2 = (o0 + 3) >> 2, C2 = (o1 + 3) >> 2;   // phase-2 tiles
  b2_pdl_wait();  // the input box is produced by the previous launch
  for (int v = 0; v < nv; ++v) {
    const long long ibase = D.in_off + static_cast<long long>(v) * D.in_stride[2];
    // ---------------- phase 1: T = in . M1^T
    for (int tb = 0; tb < R1 * C1; tb += kB2Threads) {
      const int t = tb + threadIdx.x;
      const bool act = t < R1 * C1;
      const int r = act ? t % R1 : 0, c = act ? t / R1 : 0;
      double2 acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = make_double2(0, 0);
      for (int k0 = 0; k0 < e1; k0 += kB2K) {
        const int kn = min(kB2K, e1 - k0);
        double2* xin = ch;                                   // [k][x0]
        double2* mk = ch + kB2K * e0;                        // [k][a1]
        for (int q = threadIdx.x; q < kn * e0; q += kB2Threads) {
          const int k = q / e0, x0 = q - k * e0;
          const long long a = ibase + x0 * D.in_stride[0] + static_cast<long long>(k0 + k) * D.in_stride[1];
          double2 s = in[a];
          for (int cc = 1; cc < nsum; ++cc) s = cadd(s, in[a + cc * D.sum_stride]);  // ascending child
          xin[q] = s;
        }
        for (int q = threadIdx.x; q < kn * o1; q += kB2Threads) {
          const int k = q / o1, a1 = q - k * o1;
          mk[q] = m1(a1, k0 + k);
        }
        __syncthreads();
        if (act) {
          for (int k = 0; k < kn; ++k) {
            double2 xv[4], mv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int x0 = r + R1 * i;
              xv[i] = x0 < e0 ? xin[k * e0 + x0] : make_double2(0, 0);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int a1 = c + C1 * j;
              mv[j] = a1 < o1 ? mk[k * o1 + a1] : make_double2(0, 0);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) cfma(acc[i][j], xv[i], mv[j]);
          }
        }
        __syncthreads();
      }
      if (act) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int x0 = r + R1 * i, a1 = c + C1 * j;
            if (x0 < e0 && a1 < o1) Ts[a1 * LT + x0] = acc[i][j];
          }
      }
    }
    __syncthreads();
    // ---------------- phase 2: out = M0 . T
    const long long obase = D.out_off + static_cast<long long>(v) * D.out_stride[2];
    for (int tb = 0; tb < R2 * C2; tb += kB2Threads) {
      const int t = tb + threadIdx.x;
      const bool act = t < R2 * C2;
      const int r = act ? t % R2 : 0, c = act ? t / R2 : 0;
      double2 acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = make_double2(0, 0);
      for (int k0 = 0; k0 < e0; k0 += kB2K) {
        const int kn = min(kB2K, e0 - k0);
        double2* mk = ch;  // [k][a0]
        for (int q = threadIdx.x; q < kn * o0; q += kB2Threads) {
          const int k = q / o0, a0 = q - k * o0;
          mk[q] = m0(a0, k0 + k);
        }
        __syncthreads();
        if (act) {
          for (int k = 0; k < kn; ++k) {
            double2 mv[4], tv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int a0 = r + R2 * i;
              mv[i] = a0 < o0 ? mk[k * o0 + a0] : make_double2(0, 0);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int a1 = c + C2 * j;
              tv[j] = a1 < o1 ? Ts[a1 * LT + k0 + k] : make_double2(0, 0);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j) cfma(acc[i][j], mv[i], tv[j]);
          }
        }
        __syncthreads();
      }
      if (act) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int a0 = r + R2 * i, a1 = c + C2 * j;
            if (a0 < o0 && a1 < o1)
              out[obase + a0 * D.out_stride[0] + static_cast<long long>(a1) * D.out_stride[1]] = acc[i][j];
          }
      }
    }
    __syncthreads();
  }
}

}  // namespace

size_t box2_smem_bytes(int e0, int o0, int o1) {
  const size_t chunks = std::max<size_t>(static_cast<size_t>(kB2K) * (e0 + o1), static_cast<size_t>(kB2K) * o0);
  return sizeof(double2) * (static_cast<size_t>(o1) * (e0 | 1) + chunks);
}

void launch_box2(i64 nitems, const BoxDesc* descs, const BoxLaunchInfo& info, size_t smem, const double2* mats,
                 const double2* in, double2* out, cudaStream_t st) {
  if (nitems == 0) return;
  if (info.d != 2) throw std::runtime_error("launch_box2: d must be 2");
  TBF_CUDA(cudaFuncSetAttribute(k_box2, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(nitems));
  cfg.blockDim = dim3(kB2Threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  TBF_CUDA(cudaLaunchKernelEx(&cfg, k_box2, descs, info, mats, in, out));
  TBF_CUDA(cudaGetLastError());
}

}  // namespace tbf
