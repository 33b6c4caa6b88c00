// Contraction kernels (Alg. 2).
//   k_mode_product  batched block-diagonal mode-j products: the V-bar / W / P /
//                   U-bar steps (tensor.cpp:136-166 semantics, one launch per
//                   (level, mode) covering every (tau, s) or (t, nu) item)
//   k_gemv          middle-level core contraction G_{t,s} = K(tbar,sbar) F_{t,s}
//                   (id.cpp:321 pattern): HBM-bound stream of the cores; a
//                   persistent grid whose CTA row ranges come from a cost
//                   model (row length + per-row overhead), one warp per core
//                   row with 8 independent 16-B streaming loads per lane,
//                   F_{t,s} staged in SMEM (vectors in chunks of 4 for n_v > 1);
//                   programmatic dependent launch: each warp's first row is
//                   prefetched into L2 before waiting for the W boxes
//   k_gemv_tma      variant for long rows: cp.async.bulk ring, producer warp
//                   streams cores before the dependency wait
//   k_sum_children  ordered accumulation G_{t,p_nu} = sum_nu (...) (Alg. 2 l. 203),
//                   fallback path only (box plans fold it into staging)
#include <cstdlib>

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

__device__ __forceinline__ void pdl_wait_dep() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger_dep() { asm volatile("griddepcontrol.launch_dependents;" :::); }

constexpr int kGemvThreads = 256;

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

// Persistent, balanced core GEMV: CTA i owns the contiguous global row range
// [row_begin[i], row_begin[i+1]) over all pairs, split so every CTA streams
// the same number of core BYTES (row lengths differ per pair; rows of a pair are
// contiguous in the core arena), so every SM streams the same number of
// bytes.  Per pair segment the CTA stages x = F_{t,s} in shared memory, then
// each warp walks whole rows with 8 independent 16-B streaming loads per lane
// in flight; a row is read once and applied to all nv vectors.
template <int NV>  // NV = 1: single-vector fast path; NV = 0: generic nv
__global__ void __launch_bounds__(kGemvThreads, NV == 1 ? 4 : 2) k_gemv(const int* __restrict__ cta_pair,
                                                       const GemvDesc* __restrict__ ds, int nv_rt, long long total_rows,
                                                       const long long* __restrict__ row_begin,
                                                       const double2* __restrict__ cores,
                                                       const double2* __restrict__ x, double2* __restrict__ y) {
  extern __shared__ __align__(16) double2 sx[];
  const int nv = NV == 1 ? 1 : nv_rt;
  constexpr int kAcc = NV == 1 ? 1 : 4;
  pdl_trigger_dep();  // the P/U boxes behind may start their prologue on freed SMs
  const long long g0 = row_begin[blockIdx.x];
  const long long g1 = min(total_rows, row_begin[blockIdx.x + 1]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int p = cta_pair[blockIdx.x];
  long long g = g0;
  if (g0 + warp < g1) {  // this warp's first core row into L2 while the previous kernel drains
    const GemvDesc D0 = ds[p];
    if (g0 + warp < D0.cta_off + D0.R) {
      const char* r0 = reinterpret_cast<const char*>(cores + D0.core_off + (g0 + warp - D0.cta_off) * D0.C);
      for (int o = lane * 128; o < D0.C * 16; o += 32 * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(r0 + o));
    }
  }
  pdl_wait_dep();  // x (the W outputs) comes from the previous kernel
  // vectors in chunks of kAcc: x of one chunk staged at a time (shared memory
  // bounded by C_max * kAcc for any nv); a row is read once per chunk
  for (int v0 = 0; v0 < nv; v0 += kAcc) {
    const int nvc = min(kAcc, nv - v0);
    g = g0;
    p = cta_pair[blockIdx.x];
    while (g < g1) {
      const GemvDesc D = ds[p];
      const long long pend = min(g1, D.cta_off + D.R);  // cta_off holds the pair's first global row
      const int C = D.C;
      const double2* xs = x + D.x_off + static_cast<long long>(v0) * C;
      // stage x (C * nvc) with independent loads
      for (int i = threadIdx.x; i < C * nvc; i += kGemvThreads * 4) {
        double2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i + u * kGemvThreads < C * nvc) v[u] = xs[i + u * kGemvThreads];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i + u * kGemvThreads < C * nvc) sx[i + u * kGemvThreads] = v[u];
      }
      __syncthreads();
      for (long long gr = g + warp; gr < pend; gr += kGemvThreads / 32) {
        const int r = static_cast<int>(gr - D.cta_off);
        const double2* row = cores + D.core_off + static_cast<long long>(r) * C;
        double2 acc[kAcc];
#pragma unroll
        for (int v = 0; v < kAcc; ++v) acc[v] = make_double2(0, 0);
        int c = lane;
        for (; c + 7 * 32 < C; c += 8 * 32) {
          double2 a[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) a[u] = ld_stream2(row + c + u * 32);
#pragma unroll
          for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int v = 0; v < kAcc; ++v)
              if (v < nvc) cfma(acc[v], a[u], sx[v * C + c + u * 32]);
        }
        if (c < C) {  // row tail (< 8 x 32 elements): its loads in batches of 4, not one round trip each
#pragma unroll
          for (int h = 0; h < 8; h += 4) {
            double2 a[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (c + (h + u) * 32 < C) a[u] = ld_stream2(row + c + (h + u) * 32);
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (c + (h + u) * 32 < C)
#pragma unroll
                for (int v = 0; v < kAcc; ++v)
                  if (v < nvc) cfma(acc[v], a[u], sx[v * C + c + (h + u) * 32]);
          }
        }
#pragma unroll
        for (int v = 0; v < kAcc; ++v)
          if (v < nvc) {
            const double2 t = warp_sum2(acc[v]);
            if (lane == 0) y[D.y_off + r + static_cast<long long>(v0 + v) * D.R] = t;
          }
      }
      __syncthreads();
      g = pend;
      ++p;
    }
  }
}

// Short rows (C <= 32 * RL, n_v = 1): a warp issues every load of its row at
// once (RL 16-B streaming loads per lane, predicated on C) before any FMA, so
// a row is one DRAM round trip instead of a loop of 8-load batches and tails;
// config 3's rows (C = 343-448) kept too few bytes in flight for HBM with the
// batched loop (ncu: long-scoreboard stalls, DRAM 61% of peak).
template <int RL>
__global__ void __launch_bounds__(kGemvThreads, 2) k_gemv_short(const int* __restrict__ cta_pair,
                                                              const GemvDesc* __restrict__ ds, long long total_rows,
                                                              const long long* __restrict__ row_begin,
                                                              const double2* __restrict__ cores,
                                                              const double2* __restrict__ x, double2* __restrict__ y,
                                                              int l2_ahead) {
  extern __shared__ __align__(16) double2 sx[];
  pdl_trigger_dep();
  const long long g0 = row_begin[blockIdx.x];
  const long long g1 = min(total_rows, row_begin[blockIdx.x + 1]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int p = cta_pair[blockIdx.x];
  if (g0 + warp < g1) {  // this warp's first core row into L2 while the previous kernel drains
    const GemvDesc D0 = ds[p];
    if (g0 + warp < D0.cta_off + D0.R) {
      const char* r0 = reinterpret_cast<const char*>(cores + D0.core_off + (g0 + warp - D0.cta_off) * D0.C);
      for (int o = lane * 128; o < D0.C * 16; o += 32 * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(r0 + o));
    }
  }
  pdl_wait_dep();
  long long g = g0;
  while (g < g1) {
    const GemvDesc D = ds[p];
    const long long pend = min(g1, D.cta_off + D.R);
    const int C = D.C;
    const double2* xs = x + D.x_off;
    for (int i = threadIdx.x; i < C; i += kGemvThreads) sx[i] = xs[i];
    __syncthreads();
    for (long long gr = g + warp; gr < pend; gr += kGemvThreads / 32) {
      const int r = static_cast<int>(gr - D.cta_off);
      const double2* row = cores + D.core_off + static_cast<long long>(r) * C;
      if (l2_ahead && gr + kGemvThreads / 32 < pend) {  // this warp's next row into L2 behind this one
        const char* nx = reinterpret_cast<const char*>(row + static_cast<long long>(kGemvThreads / 32) * C);
        for (int o = lane * 128; o < C * 16; o += 32 * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(nx + o));
      }
      double2 a[RL];
#pragma unroll
      for (int u = 0; u < RL; ++u)
        if (lane + u * 32 < C) a[u] = ld_stream2(row + lane + u * 32);
      double2 acc0 = make_double2(0, 0), acc1 = make_double2(0, 0);
#pragma unroll
      for (int u = 0; u < RL; ++u)
        if (lane + u * 32 < C) cfma((u & 1) ? acc1 : acc0, a[u], sx[lane + u * 32]);
      const double2 t = warp_sum2(cadd(acc0, acc1));
      if (lane == 0) y[D.y_off + r] = t;
    }
    __syncthreads();
    g = pend;
    ++p;
  }
}

// ---- compressed cores (the role ZFP plays in PAPER.md Alg. 2: "ZFP
// decompress K(tbar, sbar)"): block floating point, fixed rate.  Each core
// row is cut into blocks of 32 complex entries; a block stores one 16-bit
// exponent e (every |component| < 2^e) and, per component, the 32-bit integer
// round(x 2^(31 - e)), so a decoded entry is within 2^(e - 32) <= 2^-31 max|block|
// of the FP64 value (~5e-10 relative) and a core takes 8.06 instead of 16
// bytes per entry.  The core GEMV is HBM-bound, so it reads half the bytes.
// Layout: pair p's rows padded to nb = ceil(C / 32) blocks, row r at
// q_off[p] + r nb 32 (int2 = re, im), its exponents at (q_off[p] + r nb 32) / 32.
__global__ void k_bfp_compress(const long long* __restrict__ blk_prefix, long long npairs,
                               const GemvDesc* __restrict__ raw, const long long* __restrict__ q_off,
                               long long total_blocks, const double2* __restrict__ cores, int2* __restrict__ q,
                               short* __restrict__ ex) {
  const long long gb = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gb >= total_blocks) return;
  long long lo = 0, hi = npairs - 1;  // pair holding block gb
  while (lo < hi) {
    const long long mid = (lo + hi + 1) >> 1;
    if (blk_prefix[mid] <= gb) lo = mid;
    else hi = mid - 1;
  }
  const GemvDesc D = raw[lo];
  const int nb = (D.C + 31) / 32;
  const long long local = gb - blk_prefix[lo];
  const long long r = local / nb;
  const int b = static_cast<int>(local - r * nb);
  const int c = b * 32 + lane;
  const double2 v = c < D.C ? cores[D.core_off + r * D.C + c] : make_double2(0, 0);
  double m = fmax(fabs(v.x), fabs(v.y));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  const int e = m > 0 ? ilogb(m) + 1 : -1000;  // |component| < 2^e
  const double sc = ldexp(1.0, 31 - e);
  const long long base = q_off[lo] + (r * nb + b) * 32;
  const double qx = fmin(fmax(rint(v.x * sc), -2147483647.0), 2147483647.0);
  const double qy = fmin(fmax(rint(v.y * sc), -2147483647.0), 2147483647.0);
  q[base + lane] = make_int2(static_cast<int>(qx), static_cast<int>(qy));
  if (lane == 0) ex[base / 32] = static_cast<short>(e);
}

__device__ __forceinline__ int4 ld_stream_i4(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Core GEMV on block-floating-point cores (n_v = 1): k_gemv_short's schedule
// (persistent byte-balanced CTAs, a warp per row, every load of a row chunk
// in flight at once, the warp's next row prefetched into L2), rows decoded in
// registers.  Each lane loads 16 B = two consecutive entries per instruction
// (a warp instruction covers two 32-entry blocks: lanes 0-15 the first, 16-31
// the second); the blocks' exponents are loaded once per chunk (lane b holds
// block b's) and shuffled to the lanes that decode them.
template <int NBC>  // blocks per chunk of a row (16: rows up to 512 entries in one chunk)
__global__ void __launch_bounds__(kGemvThreads, 3) k_gemv_bfp(const int* __restrict__ cta_pair,
                                                            const GemvDesc* __restrict__ ds, long long total_rows,
                                                            const long long* __restrict__ row_begin,
                                                            const int2* __restrict__ q, const short* __restrict__ ex,
                                                            const double2* __restrict__ x, double2* __restrict__ y) {
  extern __shared__ __align__(16) double2 sx[];
  constexpr int NL = NBC / 2;  // 16-byte loads per lane per chunk
  pdl_trigger_dep();
  const long long g0 = row_begin[blockIdx.x];
  const long long g1 = min(total_rows, row_begin[blockIdx.x + 1]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, hl = lane & 15;
  int p = cta_pair[blockIdx.x];
  pdl_wait_dep();
  long long g = g0;
  while (g < g1) {
    const GemvDesc D = ds[p];
    const long long pend = min(g1, D.cta_off + D.R);
    const int C = D.C, nb = (C + 31) / 32;
    const int nb2 = (nb + 1) & ~1;  // x padded to whole block pairs
    const double2* xs = x + D.x_off;
    for (int i = threadIdx.x; i < nb2 * 32; i += kGemvThreads) sx[i] = i < C ? xs[i] : make_double2(0, 0);
    __syncthreads();
    for (long long gr = g + warp; gr < pend; gr += kGemvThreads / 32) {
      const int r = static_cast<int>(gr - D.cta_off);
      const long long rq = D.core_off + static_cast<long long>(r) * nb * 32;  // this row's first entry
      if (gr + kGemvThreads / 32 < pend) {  // the warp's next row into L2
        const char* nx = reinterpret_cast<const char*>(q + rq + static_cast<long long>(kGemvThreads / 32) * nb * 32);
        for (int o = lane * 128; o < nb * 256; o += 32 * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(nx + o));
      }
      double2 acc0 = make_double2(0, 0), acc1 = make_double2(0, 0);
      for (int b0 = 0; b0 < nb; b0 += NBC) {
        int4 a[NL];
#pragma unroll
        for (int u = 0; u < NL; ++u)
          if (b0 + 2 * u + half < nb)
            a[u] = ld_stream_i4(reinterpret_cast<const int4*>(q + rq + (b0 + 2 * u + half) * 32 + 2 * hl));
        const int ev = b0 + lane < nb ? ex[rq / 32 + b0 + lane] : 0;
#pragma unroll
        for (int u = 0; u < NL; ++u) {
          const int bb = 2 * u + half;  // this lane's block in the chunk
          const int e = __shfl_sync(0xffffffffu, ev, bb & 31);
          if (b0 + bb < nb) {
            const double sc = __longlong_as_double(static_cast<long long>(e - 31 + 1023) << 52);  // 2^(e - 31)
            const int c = (b0 + bb) * 32 + 2 * hl;
            cfma(acc0, make_double2(static_cast<double>(a[u].x) * sc, static_cast<double>(a[u].y) * sc), sx[c]);
            cfma(acc1, make_double2(static_cast<double>(a[u].z) * sc, static_cast<double>(a[u].w) * sc), sx[c + 1]);
          }
        }
      }
      const double2 t = warp_sum2(cadd(acc0, acc1));
      if (lane == 0) y[D.y_off + r] = t;
    }
    __syncthreads();
    g = pend;
    ++p;
  }
}

// Multi-vector core contraction on the FP64 tensor core: Y (R x nv) = K (R x C) X
// (C x nv) per pair, nv <= 8 padded to one 8-wide N tile.  Same CTA row ranges
// and x staging as k_gemv; a warp takes 8-row tiles of a pair and walks the
// columns in k-steps of 4 with mma.sync.m8n8k4.f64 (lane l: A = K[r0 + l/4][k + l%4],
// B = X[k + l%4][l/4], D = Y[r0 + l/4][2 (l%4) + i]); complex = four real
// MMAs.  The generic CUDA-core path spends ~22 us per vector on config 2's
// cores (FP64 issue / shared-memory bound); this one streams them once per
// 8 vectors.
__device__ __forceinline__ void mma_f64(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(kGemvThreads, 3) k_gemv_mma(const int* __restrict__ cta_pair,
                                                            const GemvDesc* __restrict__ ds, int nv,
                                                            long long total_rows,
                                                            const long long* __restrict__ row_begin,
                                                            const double2* __restrict__ cores,
                                                            const double2* __restrict__ x, double2* __restrict__ y) {
  extern __shared__ __align__(16) double2 sx[];  // [v][c], the nv vectors (the N tile's rest reads 0)
  pdl_trigger_dep();
  const long long g0 = row_begin[blockIdx.x];
  const long long g1 = min(total_rows, row_begin[blockIdx.x + 1]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lr = lane >> 2, lk = lane & 3;
  pdl_wait_dep();
  int p = cta_pair[blockIdx.x];
  long long g = g0;
  while (g < g1) {
    const GemvDesc D = ds[p];
    const long long pend = min(g1, D.cta_off + D.R);
    const int C = D.C;
    const int ldx = C | 1;  // odd row stride: the 8 vectors of a B fragment hit distinct banks
    const double2* xs = x + D.x_off;
    for (int i = threadIdx.x; i < C * nv; i += kGemvThreads) {
      const int v = i / C, c = i - v * C;
      sx[v * ldx + c] = xs[i];  // x is C x nv, vector stride C
    }
    __syncthreads();
    const int r_begin = static_cast<int>(g - D.cta_off), r_end = static_cast<int>(pend - D.cta_off);
    for (int r0 = r_begin + 8 * warp; r0 < r_end; r0 += 8 * (kGemvThreads / 32)) {
      const int r = r0 + lr;
      const bool rok = r < r_end;
      const double2* row = cores + D.core_off + static_cast<long long>(rok ? r : r0) * C;
      // two accumulator sets (even / odd k-steps): independent MMA chains
      double cr0 = 0, cr1 = 0, ci0 = 0, ci1 = 0, dr0 = 0, dr1 = 0, di0 = 0, di1 = 0;
      int k = 0;
      const bool vok = lr < nv;  // B rows of vectors >= nv are zero
      for (; k + 32 <= C; k += 32) {  // 8 k-steps: the 8 core loads in flight, x from shared memory per step
        double2 a[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = rok ? __ldg(row + k + 4 * u + lk) : make_double2(0, 0);
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
          const double2 b0 = vok ? sx[lr * ldx + k + 4 * u + lk] : make_double2(0, 0);
          const double2 b1 = vok ? sx[lr * ldx + k + 4 * u + 4 + lk] : make_double2(0, 0);
          mma_f64(cr0, cr1, a[u].x, b0.x);
          mma_f64(dr0, dr1, a[u + 1].x, b1.x);
          mma_f64(ci0, ci1, a[u].x, b0.y);
          mma_f64(di0, di1, a[u + 1].x, b1.y);
          mma_f64(cr0, cr1, -a[u].y, b0.y);
          mma_f64(dr0, dr1, -a[u + 1].y, b1.y);
          mma_f64(ci0, ci1, a[u].y, b0.x);
          mma_f64(di0, di1, a[u + 1].y, b1.x);
        }
      }
      cr0 += dr0;
      cr1 += dr1;
      ci0 += di0;
      ci1 += di1;
      for (; k < C; k += 4) {  // column tail
        const int kk = k + lk;
        const double2 a = (rok && kk < C) ? __ldg(row + kk) : make_double2(0, 0);
        const double2 b = (kk < C && lr < nv) ? sx[lr * ldx + kk] : make_double2(0, 0);
        mma_f64(cr0, cr1, a.x, b.x);
        mma_f64(cr0, cr1, -a.y, b.y);
        mma_f64(ci0, ci1, a.x, b.y);
        mma_f64(ci0, ci1, a.y, b.x);
      }
      // D fragment: row r0 + lr, vectors 2 lk and 2 lk + 1
      if (rok) {
        const int v0 = 2 * lk;
        if (v0 < nv) y[D.y_off + r + static_cast<long long>(v0) * D.R] = make_double2(cr0, ci0);
        if (v0 + 1 < nv) y[D.y_off + r + static_cast<long long>(v0 + 1) * D.R] = make_double2(cr1, ci1);
      }
    }
    __syncthreads();
    g = pend;
    ++p;
  }
}

// ---------------------------------------------------------------------------
// Core GEMV with a TMA bulk-copy pipeline (sm_90+/sm_100a): one producer warp
// streams whole core rows (contiguous C*16 bytes) into a shared-memory ring
// with cp.async.bulk + mbarrier complete_tx; 8 consumer warps compute the
// row . x dot products from shared memory.  Bytes in flight are bounded by
// the ring (not by registers), which is what an HBM stream needs.  Each CTA
// owns a balanced contiguous row range; the x vectors of the (<= kTmaMaxPairs)
// pairs it touches are staged up front.
constexpr int kTmaConsumers = 8;
constexpr int kTmaThreads = 32 * (kTmaConsumers + 1);
constexpr int kTmaMaxPairs = 4;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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

__global__ void __launch_bounds__(kTmaThreads) k_gemv_tma(const int* __restrict__ cta_pair,
                                                              const GemvDesc* __restrict__ ds, int nv,
                                                              long long total_rows,
                                                              const long long* __restrict__ row_begin,
                                                              int stages, int stage_elems, int xcap,
                                                              const double2* __restrict__ cores,
                                                              const double2* __restrict__ x,
                                                              double2* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem_raw);
  unsigned long long* empty = full + stages;
  double2* ring = reinterpret_cast<double2*>(smem_raw + 128 * ((2 * stages * 8 + 127) / 128));
  double2* sxs = ring + static_cast<long long>(stages) * stage_elems;  // kTmaMaxPairs x-slots of xcap
  __shared__ GemvDesc pd[kTmaMaxPairs];
  __shared__ int npairs_s;
  const long long g0 = row_begin[blockIdx.x];
  const long long g1 = min(total_rows, row_begin[blockIdx.x + 1]);
  const int p0 = cta_pair[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_trigger_dep();
  if (threadIdx.x == 0) {
    int np = 0;
    while (np < kTmaMaxPairs) {
      const GemvDesc D = ds[p0 + np];
      pd[np] = D;
      ++np;
      if (D.cta_off + D.R >= g1) break;
    }
    npairs_s = np;
    for (int i = 0; i < stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int np = npairs_s;
  const long long nrows = g1 - g0;
  if (warp != kTmaConsumers) {
    // consumers stage x (the previous kernel's output) while the producer
    // already streams core rows (independent of the previous kernel)
    pdl_wait_dep();
    for (int q = 0; q < np; ++q)
      for (int i = threadIdx.x; i < pd[q].C * nv; i += 32 * kTmaConsumers) sxs[q * xcap + i] = x[pd[q].x_off + i];
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kTmaConsumers) : "memory");
  }
  if (warp == kTmaConsumers) {  // producer
    if (lane == 0) {
      int q = 0;
      for (long long i = 0; i < nrows; ++i) {
        const long long gr = g0 + i;
        while (gr >= pd[q].cta_off + pd[q].R) ++q;
        const int st = static_cast<int>(i % stages);
        const long long round = i / stages;
        if (round > 0) mbar_wait(&empty[st], static_cast<unsigned>((round - 1) & 1));
        const unsigned bytes = static_cast<unsigned>(pd[q].C) * 16u;
        mbar_expect_tx(&full[st], bytes);
        bulk_g2s(ring + static_cast<long long>(st) * stage_elems,
                 cores + pd[q].core_off + (gr - pd[q].cta_off) * pd[q].C, bytes, &full[st]);
      }
    }
    return;
  }
  int q = 0;
  for (long long i = warp; i < nrows; i += kTmaConsumers) {
    const long long gr = g0 + i;
    while (gr >= pd[q].cta_off + pd[q].R) ++q;
    const int st = static_cast<int>(i % stages);
    mbar_wait(&full[st], static_cast<unsigned>((i / stages) & 1));
    const double2* row = ring + static_cast<long long>(st) * stage_elems;
    const double2* xv = sxs + q * xcap;
    const int C = pd[q].C;
    const int r = static_cast<int>(gr - pd[q].cta_off);
    for (int v = 0; v < nv; ++v) {
      double2 a0 = make_double2(0, 0), a1 = make_double2(0, 0);
      int c = lane;
      for (; c + 32 < C; c += 64) {
        cfma(a0, row[c], xv[v * C + c]);
        cfma(a1, row[c + 32], xv[v * C + c + 32]);
      }
      if (c < C) cfma(a0, row[c], xv[v * C + c]);
      const double2 t = warp_sum2(cadd(a0, a1));
      if (lane == 0) y[pd[q].y_off + r + static_cast<long long>(v) * pd[q].R] = t;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
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

// n_v in [2, 8] with the vectors' x on chip: the FP64 tensor-core kernel
bool gemv_uses_mma(int nv, int max_c) {
  static const bool no_mma = std::getenv("OIOBF_GEMV_NO_MMA") != nullptr;
  return !no_mma && nv >= 2 && nv <= 8 && static_cast<size_t>(max_c | 1) * nv * sizeof(double2) <= 96 * 1024;
}

void launch_bfp_compress(const long long* blk_prefix, i64 npairs, const GemvDesc* raw, const long long* q_off,
                         i64 total_blocks, const double2* cores, int2* q, short* ex, cudaStream_t st) {
  if (total_blocks == 0) return;
  const i64 threads = total_blocks * 32;
  k_bfp_compress<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(blk_prefix, npairs, raw, q_off,
                                                                              total_blocks, cores, q, ex);
  TBF_CUDA(cudaGetLastError());
}

int gemv_bfp_ctas_per_sm(int max_c) {
  int n = 0;
  const size_t smem = sizeof(double2) * static_cast<size_t>((max_c + 63) / 64 * 64);
  TBF_CUDA(cudaFuncSetAttribute(k_gemv_bfp<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
  TBF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_gemv_bfp<16>, kGemvThreads, smem));
  return n < 1 ? 1 : n;
}

void launch_gemv_bfp(const int* cta_pair, const GemvDesc* d, i64 nctas, i64 total_rows, const i64* row_begin,
                     const int2* q, const short* ex, const double2* x, double2* y, int max_c, cudaStream_t st) {
  if (nctas == 0) return;
  const size_t smem = sizeof(double2) * static_cast<size_t>((max_c + 63) / 64 * 64);
  TBF_CUDA(cudaFuncSetAttribute(k_gemv_bfp<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(nctas));
  cfg.blockDim = dim3(kGemvThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  TBF_CUDA(cudaLaunchKernelEx(&cfg, k_gemv_bfp<16>, cta_pair, d, static_cast<long long>(total_rows), row_begin, q, ex,
                              x, y));
  TBF_CUDA(cudaGetLastError());
}

constexpr int kShortRL = 16;  // k_gemv_short: rows up to 512 elements
bool gemv_uses_short(int nv, int max_c) {
  static const bool off = std::getenv("OIOBF_GEMV_SHORT") && std::getenv("OIOBF_GEMV_SHORT")[0] == '0';
  return !off && nv == 1 && max_c >= 128 && max_c <= 32 * kShortRL;
}

void launch_gemv(const int* cta_pair, const GemvDesc* d, i64 nctas, i64 total_rows, const i64* row_begin, int nv,
                 const double2* cores, const double2* x, double2* y, int max_c, cudaStream_t st) {
  if (nctas == 0) return;
  const bool mma = gemv_uses_mma(nv, max_c);
  const size_t smem =
      sizeof(double2) * (mma ? static_cast<size_t>(max_c | 1) * nv : static_cast<size_t>(max_c) * (nv == 1 ? 1 : std::min(nv, 4)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(nctas));
  cfg.blockDim = dim3(kGemvThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  if (mma) {
    TBF_CUDA(cudaFuncSetAttribute(k_gemv_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    TBF_CUDA(cudaLaunchKernelEx(&cfg, k_gemv_mma, cta_pair, d, nv, static_cast<long long>(total_rows), row_begin,
                                cores, x, y));
  } else if (gemv_uses_short(nv, max_c)) {
    TBF_CUDA(cudaFuncSetAttribute(k_gemv_short<kShortRL>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    static const int ahead = std::getenv("OIOBF_GEMV_L2AHEAD") ? std::atoi(std::getenv("OIOBF_GEMV_L2AHEAD")) : 1;
    TBF_CUDA(cudaLaunchKernelEx(&cfg, k_gemv_short<kShortRL>, cta_pair, d, static_cast<long long>(total_rows), row_begin,
                                cores, x, y, ahead));
  } else if (nv == 1) {
    TBF_CUDA(cudaFuncSetAttribute(k_gemv<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    TBF_CUDA(cudaLaunchKernelEx(&cfg, k_gemv<1>, cta_pair, d, nv, static_cast<long long>(total_rows), row_begin, cores,
                                x, y));
  } else {
    TBF_CUDA(cudaFuncSetAttribute(k_gemv<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    TBF_CUDA(cudaLaunchKernelEx(&cfg, k_gemv<0>, cta_pair, d, nv, static_cast<long long>(total_rows), row_begin, cores,
                                x, y));
  }
  TBF_CUDA(cudaGetLastError());
}

void launch_gemv_tma(const int* cta_pair, const GemvDesc* d, i64 nctas, i64 total_rows, const i64* row_begin, int nv,
                     int stages, int stage_elems, int xcap, const double2* cores, const double2* x, double2* y,
                     cudaStream_t st) {
  if (nctas == 0) return;
  const size_t smem = gemv_tma_smem_bytes(stages, stage_elems, xcap);
  TBF_CUDA(cudaFuncSetAttribute(k_gemv_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(nctas));
  cfg.blockDim = dim3(kTmaThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  TBF_CUDA(cudaLaunchKernelEx(&cfg, k_gemv_tma, cta_pair, d, nv, static_cast<long long>(total_rows), row_begin, stages,
                              stage_elems, xcap, cores, x, y));
  TBF_CUDA(cudaGetLastError());
}

size_t gemv_tma_smem_bytes(int stages, int stage_elems, int xcap) {
  return 128 * ((2 * static_cast<size_t>(stages) * 8 + 127) / 128) +
         sizeof(double2) * (static_cast<size_t>(stages) * stage_elems + static_cast<size_t>(kTmaMaxPairs) * xcap);
}

int gemv_tma_max_pairs() { return kTmaMaxPairs; }

int gemv_ctas_per_sm(int nv, int max_c) {
  int n = 0;
  if (gemv_uses_mma(nv, max_c)) {
    const size_t smem = sizeof(double2) * static_cast<size_t>(max_c | 1) * nv;
    TBF_CUDA(cudaFuncSetAttribute(k_gemv_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    TBF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_gemv_mma, kGemvThreads, smem));
    return n < 1 ? 1 : n;
  }
  const size_t smem = sizeof(double2) * static_cast<size_t>(max_c) * (nv == 1 ? 1 : std::min(nv, 4));
  if (gemv_uses_short(nv, max_c)) {
    TBF_CUDA(cudaFuncSetAttribute(k_gemv_short<kShortRL>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    TBF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_gemv_short<kShortRL>, kGemvThreads, smem));
  } else if (nv == 1) {
    TBF_CUDA(cudaFuncSetAttribute(k_gemv<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    TBF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_gemv<1>, kGemvThreads, smem));
  } else {
    TBF_CUDA(cudaFuncSetAttribute(k_gemv<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    TBF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_gemv<0>, kGemvThreads, smem));
  }
  return n < 1 ? 1 : n;
}

void launch_sum_children(i64 n, const SumDesc* d, i64 total, const double2* in, double2* out, cudaStream_t st) {
  if (total == 0) return;
  k_sum_children<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(n, d, total, in, out);
  TBF_CUDA(cudaGetLastError());
}


}  // namespace tbf
