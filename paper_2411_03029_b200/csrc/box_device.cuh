// Device code of one fused box contraction (Alg. 2, 185,
// 201, 203; reference mode_product_blockdiag tensor.cpp:136-166 semantics),
// run by the per-level kernel k_box (box_kernels.cu).
//
// One box is
//   out = in x_{d-1} M_{d-1} ... x_1 M_1 x_0 M_0      (M_k^T on the P/U side)
// handled by cs CTAs that split the OUTPUT rows of mode d-1 (the first mode
// contracted): every CTA needs the whole input box but no partial sums are
// exchanged.  Per CTA:
//   prologue  this CTA's factor rows -> shared memory, stored [x][a] (a
//             fastest); independent of the producer of the input, so it runs
//             before the dependency wait (programmatic dependent launch)
//   stage     input box -> shared memory: one cp.async.bulk per contiguous
//             mode-0 row (mbarrier completion); for the ordered sum of P-level
//             child contributions, batched register loads (8 children in
//             flight) summed in ascending child order
//   mode d-1  thread per input column, this CTA's A output rows in registers
//             (few columns: a column's rows split over threads in groups of 4)
//   modes d-2..1  smem -> smem, 4 output rows per thread-task
//   mode 0    4 columns per thread-task, written straight to global memory
//             (consecutive threads = consecutive rows of mode 0: coalesced)
// On the V / W side (unstaged input, <= 16 input rows and <= 8 output rows per
// mode) the three mode phases run on the FP64 tensor core instead
// (mma.sync.m8n8k4.f64: first_mode_global_mma, middle_mode_mma, last_mode_mma).
// The code is latency/issue bound (boxes are small) and sensitive to occupancy
// and code size: k_box is instantiated per register budget (CTAs per SM that
// shared memory allows) and per PATH (variants compiled out), see box_body.
// 32-bit index math inside a box.
#pragma once

#include "kernels.h"

namespace tbf {
namespace {

constexpr int kBoxThreads = 256;  // default CTA size (k_box<128, .> for small boxes)
__device__ __forceinline__ int box_nt() { return static_cast<int>(blockDim.x); }

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

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}


// address of mode-0 row `row` of the box (row = index over modes 1..d-1, nv)
__device__ __forceinline__ long long row_addr(const BoxDesc& D, int d, int row) {
  int rem = row;
  long long a = D.in_off;
  for (int p = 1; p < d; ++p) {
    const int q = qdiv(rem, D.ein[p]);
    a += static_cast<long long>(rem - q * D.ein[p]) * D.in_stride[p];
    rem = q;
  }
  return a + static_cast<long long>(rem) * D.in_stride[d];
}

// mode d-1 from the staged input: t0[rs + Rs (i + A v)] = sum_x X(rs, x, v) M(i, x)
// (AM = register bucket >= A; the code is kept small on purpose: these CTAs
// are short and a cold instruction cache is their largest stall)
template <int AM>
__device__ __forceinline__ void first_mode_smem(const double2* __restrict__ xs, const double2* __restrict__ Mf,
                                                double2* __restrict__ t0, int A, int Rs, int ein_f, int nv) {
  const int R = Rs * nv;
  for (int r = threadIdx.x; r < R; r += box_nt()) {
    const int v = qdiv(r, Rs), rs = r - v * Rs;
    double2 acc[AM];
#pragma unroll
    for (int i = 0; i < AM; ++i) acc[i] = make_double2(0, 0);
    const double2* col = xs + rs + Rs * ein_f * v;
#pragma unroll 4
    for (int x = 0; x < ein_f; ++x) {
      const double2 v0 = col[x * Rs];
#pragma unroll
      for (int i = 0; i < AM; ++i)
        if (i < A) cfma(acc[i], v0, Mf[x * A + i]);
    }
#pragma unroll
    for (int i = 0; i < AM; ++i)
      if (i < A) t0[rs + Rs * (i + A * v)] = acc[i];
  }
}

// the same for boxes with few columns (R <= half the CTA: the P / U side's
// small inputs, e.g. 7 x 7 columns on 128 threads): a task is (column, group of
// 4 output rows), so 2-4x as many threads work; every output is still summed
// over x in order (bit-identical to first_mode_smem)
__device__ __forceinline__ void first_mode_smem_split(const double2* __restrict__ xs, const double2* __restrict__ Mf,
                                                      double2* __restrict__ t0, int A, int Rs, int ein_f, int nv) {
  const int R = Rs * nv;
  const int G = (A + 3) >> 2;
  for (int t = threadIdx.x; t < R * G; t += box_nt()) {
    const int g = qdiv(t, R), r = t - g * R;
    const int v = qdiv(r, Rs), rs = r - v * Rs;
    const int i0 = g * 4, na = min(4, A - i0);
    double2 acc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = make_double2(0, 0);
    const double2* col = xs + rs + Rs * ein_f * v;
#pragma unroll 4
    for (int x = 0; x < ein_f; ++x) {
      const double2 v0 = col[x * Rs];
      const double2* m = Mf + x * A + i0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i < na) cfma(acc[i], v0, m[i]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i < na) t0[rs + Rs * (i0 + i + A * v)] = acc[i];
  }
}

// mode d-1 streamed from global memory (input box too large to stage)
template <int AM, int LD>  // LD: loads in flight per thread (8 where the register budget allows)
__device__ __forceinline__ void first_mode_global(const BoxDesc& D, int d, const double2* in,
                                                  const double2* __restrict__ Mf, double2* __restrict__ t0, int A,
                                                  int Rs, int ein_f, int nv) {
  const int f = d - 1;
  const int R = Rs * nv;
  const long long sf = D.in_stride[f];
  for (int r = threadIdx.x; r < R; r += box_nt()) {
    const int v = qdiv(r, Rs), rs = r - v * Rs;
    int rem = rs;
    long long addr = D.in_off + static_cast<long long>(v) * D.in_stride[d];
    for (int p = 0; p < f; ++p) {
      const int q = qdiv(rem, D.ein[p]);
      addr += static_cast<long long>(rem - q * D.ein[p]) * D.in_stride[p];
      rem = q;
    }
    double2 acc[AM];
#pragma unroll
    for (int i = 0; i < AM; ++i) acc[i] = make_double2(0, 0);
    // LD loads in flight per thread (the input streams from HBM: config 3's
    // first V level reads 268 MB this way)
#pragma unroll 1
    for (int x0 = 0; x0 < ein_f; x0 += LD) {
      double2 val[LD];
#pragma unroll
      for (int u = 0; u < LD; ++u)
        if (x0 + u < ein_f) val[u] = __ldcs(reinterpret_cast<const double2*>(in + addr + (x0 + u) * sf));
#pragma unroll
      for (int u = 0; u < LD; ++u)
        if (x0 + u < ein_f)
#pragma unroll
          for (int i = 0; i < AM; ++i)
            if (i < A) cfma(acc[i], val[u], Mf[(x0 + u) * A + i]);
    }
#pragma unroll
    for (int i = 0; i < AM; ++i)
      if (i < A) t0[rs + Rs * (i + A * v)] = acc[i];
  }
}

__device__ __forceinline__ void box_mma_f64(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// mode d-1 streamed from global memory on the FP64 tensor core (ein_f <= 16):
//   T(i, col) = sum_z M(i, z) X(col, z)   as m8n8k4 MMAs with
//   A = M (rows i: this CTA's <= 8 output rows, zero beyond; k = z),
//   B = 8 input columns of the box (lane l: column 8 tile + l / 4, z = 4 ks + l % 4:
//       8 consecutive columns are 128 contiguous bytes per z),
//   D = T(l / 4, 8 tile + 2 (l % 4) + {0, 1});  complex = four real MMAs.
// A warp takes two column tiles per step and has all their loads (8 per lane)
// in flight before the first MMA.  Against the CUDA-core loop this is 16
// MMAs instead of ~100 DFMAs + their shared-memory operand loads per tile
// (config 3 first V level: ncu issue slots 40% busy with the FP64 pipe at 31%).
template <int TP>  // column tiles per step (TP * 4 loads in flight per lane)
__device__ __forceinline__ void first_mode_global_mma(const BoxDesc& D, int d, const double2* in,
                                                      const double2* __restrict__ Mf, double2* __restrict__ t0,
                                                      int A, int Rs, int ein_f, int nv) {
  const int f = d - 1;
  const int R = Rs * nv;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = box_nt() >> 5;
  const int li = lane >> 2, lk = lane & 3;
  const long long sf = D.in_stride[f];
  double mr[4], mi[4], mn[4];
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int z = 4 * ks + lk;
    double2 m = make_double2(0, 0);
    if (li < A && z < ein_f) m = Mf[z * A + li];
    mr[ks] = m.x;
    mi[ks] = m.y;
    mn[ks] = -m.y;
  }
  const int ntiles = (R + 7) >> 3;
#pragma unroll 1
  for (int t = warp * TP; t < ntiles; t += nw * TP) {
    double2 xv[TP][4];
#pragma unroll
    for (int u = 0; u < TP; ++u) {
      const int col = (t + u) * 8 + li;
      const bool okc = col < R;
      long long addr = 0;
      if (okc) {
        const int v = qdiv(col, Rs);
        int rem = col - v * Rs;
        addr = D.in_off + static_cast<long long>(v) * D.in_stride[d];
        for (int p = 0; p < f; ++p) {
          const int q = qdiv(rem, D.ein[p]);
          addr += static_cast<long long>(rem - q * D.ein[p]) * D.in_stride[p];
          rem = q;
        }
      }
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int z = 4 * ks + lk;
        xv[u][ks] = okc && z < ein_f ? __ldcs(reinterpret_cast<const double2*>(in + addr + z * sf))
                                     : make_double2(0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < TP; ++u) {
      double cr0 = 0, cr1 = 0, ci0 = 0, ci1 = 0;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
        if (4 * ks < ein_f) {
          box_mma_f64(cr0, cr1, mr[ks], xv[u][ks].x);
          box_mma_f64(ci0, ci1, mr[ks], xv[u][ks].y);
          box_mma_f64(cr0, cr1, mn[ks], xv[u][ks].y);
          box_mma_f64(ci0, ci1, mi[ks], xv[u][ks].x);
        }
      if (li < A) {
        const int c0 = (t + u) * 8 + 2 * lk;
        if (c0 < R) {
          const int v = qdiv(c0, Rs);
          t0[c0 - v * Rs + Rs * (li + A * v)] = make_double2(cr0, ci0);
        }
        if (c0 + 1 < R) {
          const int v = qdiv(c0 + 1, Rs);
          t0[c0 + 1 - v * Rs + Rs * (li + A * v)] = make_double2(cr1, ci1);
        }
      }
    }
  }
}

// middle mode k: dst(b, a, c) = sum_x M(a, x) src(b, x, c), 4 output rows per task
__device__ __forceinline__ void middle_mode(const double2* __restrict__ src, double2* __restrict__ dst,
                                            const double2* __restrict__ Mk, int B, int ein, int eo, int Cc) {
  const int ng = (eo + 3) >> 2;
  const int ntask = B * ng * Cc;
  for (int t = threadIdx.x; t < ntask; t += box_nt()) {
    const int q1 = qdiv(t, B), b = t - q1 * B;
    const int c = qdiv(q1, ng), ag = q1 - c * ng;
    const int a0 = ag * 4;
    const int na = min(4, eo - a0);
    double2 acc[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) acc[g] = make_double2(0, 0);
    const double2* s = src + b + B * ein * c;
#pragma unroll 4
    for (int x = 0; x < ein; ++x) {
      const double2 val = s[B * x];
      const double2* m = Mk + x * eo + a0;
#pragma unroll
      for (int g = 0; g < 4; ++g)
        if (g < na) cfma(acc[g], val, m[g]);
    }
    double2* o = dst + b + B * (a0 + eo * c);
#pragma unroll
    for (int g = 0; g < 4; ++g)
      if (g < na) o[B * g] = acc[g];
  }
}

// middle mode k on the FP64 tensor core (eo <= 8 output rows, ein <= 16):
// per slice c, dst(b, a) = sum_x M(a, x) src(b, x) with A = M (rows a, k = x;
// fragments in registers), B = 8 consecutive b of the slice (lane l: b = 8
// tile + l / 4, x = 4 ks + l % 4), D = dst(8 tile + 2 (l % 4) + {0, 1}, a = l / 4).
__device__ __forceinline__ void middle_mode_mma(const double2* __restrict__ src, double2* __restrict__ dst,
                                                const double2* __restrict__ Mk, int B, int ein, int eo, int Cc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = box_nt() >> 5;
  const int li = lane >> 2, lk = lane & 3;
  double mr[4], mi[4], mn[4];
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int x = 4 * ks + lk;
    double2 m = make_double2(0, 0);
    if (li < eo && x < ein) m = Mk[x * eo + li];
    mr[ks] = m.x;
    mi[ks] = m.y;
    mn[ks] = -m.y;
  }
  const int nbt = (B + 7) >> 3;
#pragma unroll 1
  for (int t = warp; t < nbt * Cc; t += nw) {
    const int c = qdiv(t, nbt), b0 = (t - c * nbt) * 8;
    const double2* s = src + B * ein * c;
    const int b = b0 + li;
    double2 xv[4];
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int x = 4 * ks + lk;
      xv[ks] = b < B && x < ein ? s[b + B * x] : make_double2(0, 0);
    }
    double cr0 = 0, cr1 = 0, ci0 = 0, ci1 = 0;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
      if (4 * ks < ein) {
        box_mma_f64(cr0, cr1, mr[ks], xv[ks].x);
        box_mma_f64(ci0, ci1, mr[ks], xv[ks].y);
        box_mma_f64(cr0, cr1, mn[ks], xv[ks].y);
        box_mma_f64(ci0, ci1, mi[ks], xv[ks].x);
      }
    if (li < eo) {
      double2* o = dst + B * (li + eo * c);
      const int bb = b0 + 2 * lk;
      if (bb < B) o[bb] = make_double2(cr0, ci0);
      if (bb + 1 < B) o[bb + 1] = make_double2(cr1, ci1);
    }
  }
}

// global offset (modes 1..d-1, nv) of output column c = (a_1 .. a_{d-2}, i, v)
__device__ __forceinline__ long long col_offset(const BoxDesc& D, int d, int lo, int A, int c) {
  const int f = d - 1;
  int rem = c;
  long long addr = 0;
  for (int p = 1; p < f; ++p) {
    const int q = qdiv(rem, D.eout[p]);
    addr += static_cast<long long>(rem - q * D.eout[p]) * D.out_stride[p];
    rem = q;
  }
  const int v = qdiv(rem, A), i = rem - v * A;
  return addr + static_cast<long long>(lo + i) * D.out_stride[f] + static_cast<long long>(v) * D.out_stride[d];
}

constexpr int kColTab = 512;  // output columns whose offsets are tabulated in shared memory

// mode 0 -> global: task (a, 4 consecutive columns); column c = (a_1 .. a_{d-2}, i, v)
// tab: per-column offsets (Cc <= kColTab), or null (computed per store)
template <int CPT, bool STREAM = false>  // columns per task; streaming stores
__device__ __forceinline__ void last_mode(const BoxDesc& D, int d, int lo, int A, const double2* __restrict__ src,
                                          const double2* __restrict__ M0, int Cc, const int* tab,
                                          double2* __restrict__ out) {
  const int ein = D.ein[0], eo = D.eout[0];
  const int ncg = (Cc + CPT - 1) / CPT;
  const int ntask = eo * ncg;
  for (int t = threadIdx.x; t < ntask; t += box_nt()) {
    const int cg = qdiv(t, eo), a = t - cg * eo;
    const int c0 = cg * CPT;
    const int nc = min(CPT, Cc - c0);
    double2 acc[CPT];
#pragma unroll
    for (int g = 0; g < CPT; ++g) acc[g] = make_double2(0, 0);
    const double2* s = src + ein * c0;
#pragma unroll 4
    for (int x = 0; x < ein; ++x) {
      const double2 m = M0[x * eo + a];
#pragma unroll
      for (int g = 0; g < CPT; ++g)
        if (g < nc) cfma(acc[g], s[x + ein * g], m);
    }
    const long long base = D.out_off + static_cast<long long>(a) * D.out_stride[0];
    if (tab) {
#pragma unroll
      for (int g = 0; g < CPT; ++g)
        if (g < nc) {
          if (STREAM) __stcs(out + base + tab[c0 + g], acc[g]);  // the result tensor G: written once, never re-read
          else out[base + tab[c0 + g]] = acc[g];
        }
    } else {
#pragma unroll 1
      for (int g = 0; g < nc; ++g)
      {
        double2 v = acc[0];  // (static indexing keeps the accumulators in registers)
#pragma unroll
        for (int q = 1; q < CPT; ++q)
          if (g == q) v = acc[q];
        out[base + col_offset(D, d, lo, A, c0 + g)] = v;
      }
    }
  }
}

// mode 0 -> global on the FP64 tensor core (ein <= 16, eout <= 16, tabulated
// columns):  out(a, c) = sum_x M0(a, x) src(x, c)  as m8n8k4 MMAs with
//   A = M0 (rows a of one 8-row tile, k = x; fragments in registers for the
//       whole phase), B = 8 columns of the staged intermediate (lane l: column
//       8 tile + l / 4, x = 4 ks + l % 4: one 16-byte shared-memory load per
//       k-step), D = out(8 mt + l / 4, 8 tile + 2 (l % 4) + {0, 1}) stored
//       straight to global memory (8 consecutive a per column = 128 contiguous
//       bytes); complex = four real MMAs.
// A column tile costs ein / 4 loads and 4 ein / 4 MMAs per row tile instead
// of five shared-memory operands per four complex FMAs.  Measured (config 3):
// on the V / W side (one row tile, 14-16 input rows) 1.028 -> 1.020 ms; on the
// P / U side (two row tiles, 5-8 input rows padded to 8: the same FP64 pipe
// time as the CUDA-core loop) 22 us slower, so the default uses it for V / W
// only (info.mma == 2; 3 = both sides).
__device__ __forceinline__ void last_mode_mma(const BoxDesc& D, const double2* __restrict__ src,
                                              const double2* __restrict__ M0, int Cc, const int* tab,
                                              double2* __restrict__ out) {
  const int ein = D.ein[0], eo = D.eout[0];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = box_nt() >> 5;
  const int li = lane >> 2, lk = lane & 3;
  const int ntiles = (Cc + 7) >> 3;
  const long long s0 = D.out_stride[0];
#pragma unroll 1
  for (int mt = 0; mt * 8 < eo; ++mt) {
    const int a = mt * 8 + li;
    double mr[4], mi[4], mn[4];
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int x = 4 * ks + lk;
      double2 m = make_double2(0, 0);
      if (a < eo && x < ein) m = M0[x * eo + a];
      mr[ks] = m.x;
      mi[ks] = m.y;
      mn[ks] = -m.y;
    }
    const long long base = D.out_off + static_cast<long long>(a) * s0;
#pragma unroll 1
    for (int t = warp; t < ntiles; t += nw) {
      const int c = t * 8 + li;
      double2 xv[4];
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int x = 4 * ks + lk;
        xv[ks] = c < Cc && x < ein ? src[x + ein * c] : make_double2(0, 0);
      }
      double cr0 = 0, cr1 = 0, ci0 = 0, ci1 = 0;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
        if (4 * ks < ein) {
          box_mma_f64(cr0, cr1, mr[ks], xv[ks].x);
          box_mma_f64(ci0, ci1, mr[ks], xv[ks].y);
          box_mma_f64(cr0, cr1, mn[ks], xv[ks].y);
          box_mma_f64(ci0, ci1, mi[ks], xv[ks].x);
        }
      if (a < eo) {
        const int c0 = t * 8 + 2 * lk;
        if (c0 < Cc) out[base + tab[c0]] = make_double2(cr0, ci0);
        if (c0 + 1 < Cc) out[base + tab[c0 + 1]] = make_double2(cr1, ci1);
      }
    }
  }
}

// Shared-memory state of one box CTA besides the dynamic buffer.
struct BoxSmem {
  BoxDesc D;
  int coltab[kColTab];  // output column offsets of mode 0's stores, relative to the box origin (32 bits: the
                        // host enables the table only when every box's span fits, info.tab_ok)
  int mo[kMaxD + 1];
  unsigned long long bar;  // staging mbarrier (initialised once per CTA)
};

// One CTA's share (crank of info.cs) of the box whose descriptor is already
// in S.D (all threads synchronised after the copy).  `wait` blocks until the
// input is produced (all threads call it; it ends with a CTA barrier).
// `phase` is the staging mbarrier's parity, flipped on each bulk staging.
// PATH (compile time; the host picks it per launch, info.path): 0 = every
// variant behind run-time branches; 1 = the V / W side's tensor-core box
// (unstaged first mode, middle modes and mode 0 by MMA; the launch's boxes all
// meet the MMA size limits); 2 = staged CUDA-core box (child sums / copied
// rows, row-split first mode): the same code paths with the other variants
// compiled out and d fixed to 3 -- these 80-register kernels are sensitive to
// code size.
constexpr int kPathAny = 0, kPathVmma = 1, kPathStaged = 2;
template <int LD, int TP, int PATH, class Wait>  // TP: column tiles per step of the tensor-core first mode
__device__ __forceinline__ void box_body(BoxSmem& S, const BoxLaunchInfo& info, int crank,
                                         const double2* __restrict__ mats, const double2* in, double2* out,
                                         double2* sm, unsigned& phase, Wait wait) {
  const BoxDesc& D = S.D;
  const int tid = threadIdx.x;
  const int cs = info.cs;
  // (the specialised variants are built for d = 3 -- the host selects them only then -- so the
  // mode loops and the index decompositions below unroll)
  const int d = PATH != kPathAny ? 3 : info.d;
  const int f = d - 1, nv = info.nv, tr = PATH == kPathVmma ? 0 : info.transpose;
  const int ef = D.eout[f];
  const int lo = qdiv(crank * ef, cs), hi = qdiv((crank + 1) * ef, cs);
  const int A = hi - lo;  // 0 <= A <= 8 (host)
  if (A <= 0) {           // narrow box: nothing left for this CTA (k_flow never issues one)
    wait();
    return;
  }
  int Rs = 1;  // columns of mode d-1 (modes 0..d-2); times nv below
  for (int p = 0; p < f; ++p) Rs *= D.ein[p];
  const int ein_f = D.ein[f];
  const int e0n = D.ein[0];
  const int total_in = Rs * ein_f * nv;
  // bulk staging needs contiguous 16-B rows (every double2 row qualifies)
  const bool bulk = PATH != kPathVmma && info.stage && D.nsum == 1 && D.in_stride[0] == 1;
  if (tid == 0) {
    S.mo[0] = 0;
    for (int k = 0; k < d; ++k) S.mo[k + 1] = S.mo[k] + D.ein[k] * (k == f ? A : D.eout[k]);
    if (bulk) mbar_expect_tx(&S.bar, static_cast<unsigned>(total_in) * 16u);
  }
  __syncthreads();
  double2* smat = sm;
  double2* xs = smat + info.smem_mat;
  double2* t0 = xs + info.smem_in;
  double2* t1 = t0 + info.smem_t;
  // ---- prologue: factor rows, [x][a] with a fastest (mode d-1: rows lo..hi)
  for (int k = 0; k < d; ++k) {
    const int ein = D.ein[k], eo = k == f ? A : D.eout[k], a0 = k == f ? lo : 0;
    const int mrows = tr ? ein : D.eout[k];  // stored matrix: r x w column-major
    const double2* M = mats + D.mat_off[k];
    double2* Sm = smat + S.mo[k];
    for (int q = tid; q < ein * eo; q += box_nt()) {
      const int x = qdiv(q, eo), a = q - x * eo + a0;
      const double2* src = M + (tr ? x + mrows * a : a + mrows * x);
      // asynchronous copies: the staging loads below are issued behind them
      // without waiting for the factor rows to land (one memory latency less
      // on every CTA's critical path)
      if (info.afac) cp_async16(Sm + q, src);
      else Sm[q] = __ldg(src);
    }
  }
  // ---- the input box is produced by an earlier launch / item
  wait();
  if (PATH != kPathVmma && (PATH == kPathStaged || info.stage)) {
    const int nrows = total_in / e0n;
    if (bulk) {
      const unsigned rbytes = static_cast<unsigned>(e0n) * 16u;
      for (int row = tid; row < nrows; row += box_nt())
        bulk_g2s(xs + row * e0n, in + row_addr(D, d, row), rbytes, &S.bar);
      mbar_wait(&S.bar, phase);
      phase ^= 1u;
    } else if (D.nsum == 1) {
      const long long s0 = D.in_stride[0];
      for (int row = tid; row < nrows; row += box_nt()) {
        const long long ra = row_addr(D, d, row);
        for (int x = 0; x < e0n; ++x) cp_async16(xs + row * e0n + x, in + ra + x * s0);
      }
      cp_async_wait_all();
    } else {
      // ordered child sums (ascending child), 8 children of loads in flight
      const long long s0 = D.in_stride[0];
      const long long cstr = D.sum_stride;
#pragma unroll 1
      for (int e = tid; e < total_in; e += box_nt()) {
        const int row = qdiv(e, e0n);
        const double2* p = in + row_addr(D, d, row) + (e - row * e0n) * s0;
        double2 acc = make_double2(0, 0);
#pragma unroll 1
        for (int c0 = 0; c0 < D.nsum; c0 += 8) {
          double2 v[8];
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (c0 + c < D.nsum) v[c] = p[(c0 + c) * cstr];
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (c0 + c < D.nsum) acc = (c0 + c == 0) ? v[c] : cadd(acc, v[c]);
        }
        xs[e] = acc;
      }
    }
  }
  if (info.afac) cp_async_wait_all();
  __syncthreads();
  // ---- mode d-1: column r = rs + Rs * v  ->  t0[rs + Rs * (i + A * v)]
  {
    // (the row count is dispatched to its register bucket: no predicated-off
    // FMAs; one bucket is hot per launch, so the i-cache footprint stays)
    const double2* Mf = smat + S.mo[f];
    if constexpr (PATH == kPathVmma) {
      first_mode_global_mma<TP>(D, d, in, Mf, t0, A, Rs, ein_f, nv);
    } else if constexpr (PATH == kPathStaged) {
      if (info.split1 && A > 4 && 2 * Rs * nv <= box_nt()) first_mode_smem_split(xs, Mf, t0, A, Rs, ein_f, nv);
      else if (info.amax <= 2) first_mode_smem<2>(xs, Mf, t0, A, Rs, ein_f, nv);
      else if (info.amax <= 4) first_mode_smem<4>(xs, Mf, t0, A, Rs, ein_f, nv);
      else first_mode_smem<8>(xs, Mf, t0, A, Rs, ein_f, nv);
    } else if (info.stage && info.split1 && A > 4 && 2 * Rs * nv <= box_nt()) {
      first_mode_smem_split(xs, Mf, t0, A, Rs, ein_f, nv);
    } else if (info.stage) {
      if (info.amax <= 2) first_mode_smem<2>(xs, Mf, t0, A, Rs, ein_f, nv);
      else if (info.amax <= 4) first_mode_smem<4>(xs, Mf, t0, A, Rs, ein_f, nv);
      else first_mode_smem<8>(xs, Mf, t0, A, Rs, ein_f, nv);
    } else if (info.mma && ein_f <= 16) {
      first_mode_global_mma<TP>(D, d, in, Mf, t0, A, Rs, ein_f, nv);
    } else {
      first_mode_global<8, LD>(D, d, in, Mf, t0, A, Rs, ein_f, nv);
    }
  }
  __syncthreads();
  // ---- modes d-2 .. 1 (smem -> smem); extents: e[p] = ein (p <= k), eout (k < p < f), A (f), nv
  double2* src = t0;
  double2* dst = t1;
  int Cc = A * nv;  // product of the extents above the current mode
  for (int k = f - 1; k >= 1; --k) {
    const int ein = D.ein[k], eo = D.eout[k];
    int B = 1;
    for (int p = 0; p < k; ++p) B *= D.ein[p];
    if constexpr (PATH == kPathVmma) middle_mode_mma(src, dst, smat + S.mo[k], B, ein, eo, Cc);
    else if constexpr (PATH == kPathStaged) middle_mode(src, dst, smat + S.mo[k], B, ein, eo, Cc);
    else if (info.mma >= 4 && !info.transpose && eo <= 8 && ein <= 16) middle_mode_mma(src, dst, smat + S.mo[k], B, ein, eo, Cc);
    else middle_mode(src, dst, smat + S.mo[k], B, ein, eo, Cc);
    __syncthreads();
    Cc *= eo;
    double2* tmp = src;
    src = dst;
    dst = tmp;
  }
  // output column offsets of mode 0's stores (computed once, not per store)
  const bool tab = Cc <= kColTab && info.tab_ok;
  if (tab)
    for (int c = tid; c < Cc; c += box_nt()) S.coltab[c] = static_cast<int>(col_offset(D, d, lo, A, c));
  __syncthreads();
  // ---- mode 0 -> global
  if constexpr (PATH == kPathVmma) {
    last_mode_mma(D, src, smat + S.mo[0], Cc, S.coltab, out);
  } else if constexpr (PATH == kPathStaged) {
    if (info.stream_out) last_mode<4, true>(D, d, lo, A, src, smat + S.mo[0], Cc, tab ? S.coltab : nullptr, out);
    else last_mode<4>(D, d, lo, A, src, smat + S.mo[0], Cc, tab ? S.coltab : nullptr, out);
  } else if (tab && D.ein[0] <= 16 && D.eout[0] <= 16 && (info.mma == 3 || ((info.mma == 2 || info.mma >= 4) && !info.transpose)))
    last_mode_mma(D, src, smat + S.mo[0], Cc, S.coltab, out);
  else if (info.stream_out)
    last_mode<4, true>(D, d, lo, A, src, smat + S.mo[0], Cc, tab ? S.coltab : nullptr, out);
  else
    last_mode<4>(D, d, lo, A, src, smat + S.mo[0], Cc, tab ? S.coltab : nullptr, out);
  __syncthreads();
}

}  // namespace
}  // namespace tbf
