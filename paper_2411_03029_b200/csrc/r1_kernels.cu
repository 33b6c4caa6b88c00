// Rank-one apply engine: butterflies whose every ID has rank 1 (the DFT with
// two-sided bit reversal, SURVEY F4 / App. A3 -- config 4: d = 6, n = 16,
// 2.08e8 IDs, 1.7e7 middle pairs).  With r = 1 the factor arenas are regular
// (slot sl's 1 x W block at sl * W, W = the leaf size at level 0 and 2 above),
// every level's intermediate has exactly nmid^2 elements and every core is
// 1 x 1, so the whole contraction runs with implicit geometry: no per-box or
// per-pair descriptors are read (the tiny-box engine spent more HBM traffic on
// metadata than on factors at this scale).  All extents are powers of two, so
// index arithmetic is shifts and masks.
//
//   k_r1_vw  V/W level l (Alg. 2, F_{tau,s} = F_{p(tau),s} x_k W):
//            a CTA stages the input tensors of `gpb` groups (s, parent tau)
//            -- every child tau of a group reads all of it -- and the factor
//            blocks of their children (copied child block by child block, so
//            the loads are coalesced; odd shared-memory stride) on chip; a
//            thread evaluates one output (child, block tuple): the W^d box
//            contracted mode by mode with the child's d factor rows (a
//            running partial per mode, in registers).  At level Lc the
//            epilogue multiplies by the 1 x 1 core K(t, s) (the middle
//            contraction folded into the last V/W level).
//   k_r1_pu  P/U level l (G_{t,p(nu)} = sum_c G_{t,nu_c} x_k P^T): each output
//            of a (group, block tuple) unit is sum_c in_c prod_k b_ck(x_k) over
//            the 2^d children; split the modes into lo / hi halves and it
//            becomes sum_c A_c(x_lo) B_c(x_hi): phase 1 builds A_c, B_c (one
//            thread per child, factors staged as above), phase 2 one thread per
//            output sums the children in ascending order (the reference's
//            order, Alg. 2).
//
// Intermediates (ping-pong, each nmid^2 x nv, vector slowest):
//   V/W level l:  ((v * nmid + s) * nin + tau) * nj^d + jt
//   P/U level l:  ((v * nmid + t) * pnin + p_nu) * E^d + pos   (E = nj * W)
// jt / pos mixed radix, mode 0 fastest.  The level-Lc V/W output is indexed by
// the pair p = s * nmid + t, like the cores.  P/U groups are ordered t fastest
// (g = p_nu * nmid + t), so the level-Lc gather of G_{t,s} reads runs of t.
//
// Sharded (world > 1, a power-of-two number nown of owned multi-sets per rank):
// the outer index s / t above is the LOCAL index i < nown everywhere (buffers
// hold nown * nmid elements per vector, the factor arenas and cores hold only
// the owned slots, in local order) and a.own[i] names the middle multi-set for
// the F / G slabs.  The level-Lc P/U input is then (v * nmid + s) * nown + t
// with s over ALL middle multi-sets: k_r1_pack / k_r1_unpack move the blocks
// G_{t,s} between these buffers and the exchange's send / receive buffers.
#include "kernels.h"

namespace tbf {

namespace {

constexpr int kR1Threads = 256;   // P/U kernels
constexpr int kR1VThreads = 128;  // V/W and middle-level kernels (several CTAs per SM: loads overlap compute)

template <int B, int E>
struct Pow {
  static constexpr int v = B * Pow<B, E - 1>::v;
};
template <int B>
struct Pow<B, 0> {
  static constexpr int v = 1;
};

// inner index of child c of parent inner index pinner at level l >= 1
// (mixed radix 2^l per mode, mode 0 fastest; child bit p selects the half of mode p)
template <int D>
__device__ __forceinline__ i64 r1_child(i64 pinner, int l, int c) {
  i64 inner = 0;
#pragma unroll
  for (int p = D - 1; p >= 0; --p) {
    const i64 pc = (pinner >> ((l - 1) * p)) & ((i64{1} << (l - 1)) - 1);
    inner = (inner << l) | (2 * pc + ((c >> p) & 1));
  }
  return inner;
}

// e / fblk for e < 2^20 (host-computed magic = ceil(2^32 / fblk), fblk < 2^12)
__device__ __forceinline__ int r1_div(int e, unsigned magic) { return static_cast<int>(__umulhi(e, magic)); }

// parent inner index (level l - 1) of inner index `inner` at level l >= 1
template <int D>
__device__ __forceinline__ i64 r1_parent(i64 inner, int l) {
  i64 p = 0;
#pragma unroll
  for (int q = 0; q < D; ++q) p |= (((inner >> (l * q)) & ((i64{1} << l) - 1)) >> 1) << ((l - 1) * q);
  return p;
}

// contiguous factor blocks [src, src + nblk * fblk) -> shared memory at odd stride FS
__device__ __forceinline__ void r1_stage_contig(const R1LevelArgs& a, const double2* __restrict__ src, int nblk,
                                                double2* __restrict__ fs) {
  const int fblk = a.fblk, FS = a.FS;
  for (int e = threadIdx.x; e < nblk * fblk; e += blockDim.x) {
    const int q = r1_div(e, a.magic);
    fs[q * FS + e - q * fblk] = __ldg(src + e);
  }
}

// A_c(x_lo) = val * prod_{k < H} b_k(x_k),  B_c(x_hi) = prod_{k >= H} b_k(x_k)
template <int D, int W, int NA, int NB>
__device__ __forceinline__ void r1_tables(double2 val, const double2 (&b)[D][W], double2 (&A)[NA], double2 (&B)[NB]) {
  constexpr int H = D / 2;
  A[0] = val;
  B[0] = make_double2(1.0, 0.0);
  int sz = 1;
#pragma unroll
  for (int k = 0; k < H; ++k) {
#pragma unroll
    for (int i = NA - 1; i >= 0; --i)
      if (i < sz)
#pragma unroll
        for (int x = W - 1; x >= 0; --x) A[i + sz * x] = cmul(A[i], b[k][x]);
    sz *= W;
  }
  sz = 1;
#pragma unroll
  for (int k = H; k < D; ++k) {
#pragma unroll
    for (int i = NB - 1; i >= 0; --i)
      if (i < sz)
#pragma unroll
        for (int x = W - 1; x >= 0; --x) B[i + sz * x] = k == H ? b[k][x] : cmul(B[i], b[k][x]);
    sz *= W;
  }
}

// P/U output address of (t, parent p_nu, block tuple jt, box position x)
template <int D, int W>
__device__ __forceinline__ i64 r1_pu_out(const R1LevelArgs& a, i64 v, i64 t, i64 pnu, int jt, int x) {
  const int nj = 1 << a.lg_nj;
  int q = x;
  if (a.out_global) {
    const i64 tg = a.own ? a.own[t] : t;  // the middle multi-set of local t
    i64 addr = v << (a.lg_n * D);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int jk = (jt >> (a.lg_nj * k)) & (nj - 1), xk = q % W;
      q /= W;
      addr += ((((tg >> (a.Lc * k)) & (a.mpm - 1)) << a.lg_mid) + jk * W + xk) << (a.lg_n * k);
    }
    return addr;
  }
  i64 pos = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const int jk = (jt >> (a.lg_nj * k)) & (nj - 1), xk = q % W;
    q /= W;
    pos += static_cast<i64>(jk * W + xk) << (a.lg_E * k);
  }
  return (((((v << a.lg_nown) + t) << a.lg_pnin) + pnu) << a.lg_ED) + pos;
}

// V/W level: CTA = (s, T consecutive tau); their parents form a contiguous
// range (aligned power-of-two tau ranges), staged at odd stride XS; the T
// factor blocks are one contiguous run of the arena.
template <int D, int W>
__global__ void __launch_bounds__(kR1Threads, 2) k_r1_vw(R1LevelArgs a, const double2* __restrict__ fac,
                                                          const double2* __restrict__ cores,
                                                          const double2* __restrict__ in, double2* __restrict__ out) {
  extern __shared__ __align__(16) double2 xs[];
  constexpr int NBOX = Pow<W, D>::v;
  const i64 v = blockIdx.y;
  const int lg_T = a.lg_T, T = 1 << lg_T;
  const int lg_ED = a.lg_ED, lg_E = a.lg_E, E = 1 << lg_E, XS = a.XS;
  const i64 blk = blockIdx.x;
  const i64 s = blk >> (a.lg_nin - lg_T);     // local outer index
  const i64 sg = a.own ? a.own[s] : s;        // its middle multi-set (F slab)
  const i64 tau0 = (blk & ((i64{1} << (a.lg_nin - lg_T)) - 1)) << lg_T;
  const i64 pfirst = a.l > 0 ? r1_parent<D>(tau0, a.l) : 0;
  const int np = a.l > 0 ? static_cast<int>(r1_parent<D>(tau0 + T - 1, a.l) - pfirst + 1) : 1;
  double2* fs = xs + a.Pc * XS;
  // ---- stage the parents' tensors (level 0: the F slab of s) ...
  for (int e = threadIdx.x; e < (np << lg_ED); e += blockDim.x) {
    const int pl = e >> lg_ED, loc = e & ((1 << lg_ED) - 1);
    i64 addr;
    if (a.in_global) {
      addr = v << (a.lg_n * D);
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const int ek = (loc >> (lg_E * k)) & (E - 1);
        addr += ((((sg >> (a.Lc * k)) & (a.mpm - 1)) << a.lg_mid) + ek) << (a.lg_n * k);
      }
    } else {
      addr = (((((v << a.lg_nown) + s) << a.lg_pnin) + pfirst + pl) << lg_ED) + loc;
    }
    xs[pl * XS + loc] = __ldg(in + addr);
  }
  // ---- ... and the T children's factor blocks (one contiguous run)
  r1_stage_contig(a, fac + ((s << a.lg_nin) + tau0) * a.fblk, T, fs);
  __syncthreads();
  const int lg_njd = a.lg_njd, lg_nj = a.lg_nj, nj = 1 << lg_nj;
  for (int e = threadIdx.x; e < (T << lg_njd); e += blockDim.x) {
    const int tl = e & (T - 1);  // tau fastest: consecutive outputs, runs of shared parents
    const int jt = e >> lg_T;
    const i64 tau = tau0 + tl;
    const int pl = a.l > 0 ? static_cast<int>(r1_parent<D>(tau, a.l) - pfirst) : 0;
    const double2* fb = fs + tl * a.FS;
    int stk[D];
    int base = pl * XS;
    double2 b[D][W];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int jk = (jt >> (lg_nj * k)) & (nj - 1);
      stk[k] = 1 << (lg_E * k);
      base += (jk * W) << (lg_E * k);
#pragma unroll
      for (int x = 0; x < W; ++x) b[k][x] = fb[(k * nj + jk) * W + x];
    }
    // mode-by-mode contraction of the W^d box: part[k] accumulates mode k
    double2 part[D];
#pragma unroll
    for (int x = 0; x < NBOX; ++x) {
      int o = 0;
      {
        int q = x;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          o += (q % W) * stk[k];
          q /= W;
        }
      }
      const double2 val = xs[base + o];
      const int x0 = x % W;
      if (x0 == 0) part[0] = cmul(b[0][0], val);
      else cfma(part[0], b[0][x0], val);
      // carries: mode k + 1 receives mode k's partial when digits 0..k are all W - 1
      int q = x, full = 1;
#pragma unroll
      for (int k = 0; k + 1 < D; ++k) {
        full *= W;
        if ((x + 1) % full != 0) break;
        q /= W;
        const int xk = q % W;
        if (xk == 0) part[k + 1] = cmul(b[k + 1][0], part[k]);
        else cfma(part[k + 1], b[k + 1][xk], part[k]);
      }
    }
    double2 res = part[D - 1];
    if (a.core_mul) res = cmul(__ldg(cores + (s << a.lg_nmid) + tau), res);
    out[(((((v << a.lg_nown) + s) << a.lg_nin) + tau) << lg_njd) + jt] = res;
  }
}

// V/W level with one block tuple per child (nj = 1, the middle level Lc, the
// bulk of the factor bytes): one WARP per tile of 32 consecutive tau of one
// s.  The warp copies its parents' tensors and its 32 factor blocks (both
// contiguous runs) with coalesced loads into a warp-private shared-memory
// slice and only __syncwarp()s, so warps never wait on each other and the
// loads of some warps overlap the FP64 work of others.
template <int D, int W>
__global__ void __launch_bounds__(kR1VThreads, 6) k_r1_vw_mid(R1LevelArgs a, const double2* __restrict__ fac,
                                                              const double2* __restrict__ cores,
                                                              const double2* __restrict__ in,
                                                              double2* __restrict__ out) {
  extern __shared__ __align__(16) double2 wsm[];
  constexpr int NBOX = Pow<W, D>::v;
  const i64 v = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const i64 tile = static_cast<i64>(blockIdx.x) * (kR1VThreads / 32) + warp;
  if (tile >= (i64{1} << (a.lg_nown + a.lg_nin - 5))) return;
  const int lg_ED = a.lg_ED, lg_E = a.lg_E, XS = a.XS, FS = a.FS, fblk = a.fblk;
  double2* xs = wsm + warp * (a.Pc * XS + 32 * FS);
  double2* fs = xs + a.Pc * XS;
  const i64 s = tile >> (a.lg_nin - 5);
  const i64 tau0 = (tile & ((i64{1} << (a.lg_nin - 5)) - 1)) << 5;
  const i64 pfirst = r1_parent<D>(tau0, a.l);
  const int np = static_cast<int>(r1_parent<D>(tau0 + 31, a.l) - pfirst + 1);
  const i64 tau = tau0 + lane;
  const double2 core = a.core_mul ? __ldg(cores + (s << a.lg_nmid) + tau) : make_double2(1, 0);
  {
    const double2* src = in + ((((v << a.lg_nown) + s) << a.lg_pnin) + pfirst << lg_ED);
    const int n = np << lg_ED;
#pragma unroll 4
    for (int e = lane; e < n; e += 32) xs[(e >> lg_ED) * XS + (e & ((1 << lg_ED) - 1))] = __ldg(src + e);
  }
  {
    const double2* src = fac + ((s << a.lg_nin) + tau0) * fblk;
    const int n = 32 * fblk;
#pragma unroll 4
    for (int e = lane; e < n; e += 32) {
      const int q = r1_div(e, a.magic);
      fs[q * FS + e - q * fblk] = __ldg(src + e);
    }
  }
  __syncwarp();
  const int pl = static_cast<int>(r1_parent<D>(tau, a.l) - pfirst);
  const double2* fb = fs + lane * FS;
  const int base = pl * XS;
  double2 part[D];
#pragma unroll
  for (int x = 0; x < NBOX; ++x) {
    int o = 0;
    {
      int q = x;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        o += (q % W) << (lg_E * k);
        q /= W;
      }
    }
    const double2 val = xs[base + o];
    const int x0 = x % W;
    if (x0 == 0) part[0] = cmul(fb[0], val);
    else cfma(part[0], fb[x0], val);
    int q = x, full = 1;
#pragma unroll
    for (int k = 0; k + 1 < D; ++k) {
      full *= W;
      if ((x + 1) % full != 0) break;
      q /= W;
      const int xk = q % W;
      if (xk == 0) part[k + 1] = cmul(fb[(k + 1) * W], part[k]);
      else cfma(part[k + 1], fb[(k + 1) * W + xk], part[k]);
    }
  }
  out[(((v << a.lg_nown) + s) << a.lg_nin) + tau] = cmul(core, part[D - 1]);
}

// P/U level, general form: CTA = gpb (group, block tuple) units, groups t
// fastest; one thread per (unit, child) builds A_c / B_c, one thread per
// output sums the children in ascending order.
template <int D, int W>
__global__ void __launch_bounds__(kR1Threads, 3) k_r1_pu(R1LevelArgs a, const double2* __restrict__ fac,
                                                         const double2* __restrict__ in, double2* __restrict__ out) {
  extern __shared__ __align__(16) double2 sm[];  // factor blocks, then (aliased) the A / B tables
  __shared__ i64 cbase[kR1Threads];             // arena offset of each staged child block
  constexpr int H = D / 2;
  constexpr int NA = Pow<W, H>::v, NB = Pow<W, D - H>::v, NX = NA * NB;
  constexpr int TS = (NA + NB) | 1;  // odd stride: conflict-free phase-1 stores
  const i64 v = blockIdx.y;
  const i64 u0 = static_cast<i64>(blockIdx.x) * a.gpb;
  const int nu = static_cast<int>(min(static_cast<i64>(a.gpb), a.nunits - u0));
  const int lg_nch = a.lg_nch, lg_njd = a.lg_njd, lg_nj = a.lg_nj, nch = 1 << lg_nch, nj = 1 << lg_nj;
  const i64 gfirst = u0 >> lg_njd;
  const int ngr = static_cast<int>(((u0 + nu - 1) >> lg_njd) - gfirst + 1);
  // ---- stage the factor blocks of the units' groups' children
  for (int q = threadIdx.x; q < (ngr << lg_nch); q += blockDim.x) {
    const int gl = q >> lg_nch, c = q & (nch - 1);
    const i64 g = gfirst + gl;
    const i64 t = g & ((i64{1} << a.lg_nown) - 1), pnu = g >> a.lg_nown;
    cbase[q] = ((t << a.lg_nin) + (a.l > 0 ? r1_child<D>(pnu, a.l, c) : 0)) * a.fblk;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < (ngr << lg_nch) * a.fblk; e += blockDim.x) {
    const int q = r1_div(e, a.magic), off = e - q * a.fblk;
    sm[q * a.FS + off] = __ldg(fac + cbase[q] + off);
  }
  __syncthreads();
  // ---- phase 1: A_c, B_c per (unit, child)
  const int n1 = nu << lg_nch;
  double2 A[NA], B[NB];
  const int e1 = threadIdx.x;  // the CTA has >= nu * nch threads (host sizes gpb so)
  if (e1 < n1) {
    const int c = e1 & (nch - 1), ul = e1 >> lg_nch;
    const i64 u = u0 + ul;
    const i64 g = u >> lg_njd;
    const int jt = static_cast<int>(u & ((i64{1} << lg_njd) - 1));
    const i64 t = g & ((i64{1} << a.lg_nown) - 1), pnu = g >> a.lg_nown;  // groups t fastest
    const i64 nuc = a.l > 0 ? r1_child<D>(pnu, a.l, c) : 0;
    const double2 val =
        __ldg(in + (a.in_transposed ? (((v << a.lg_nmid) + nuc) << a.lg_nown) + t
                                    : (((((v << a.lg_nown) + t) << a.lg_nin) + nuc) << lg_njd) + jt));
    const double2* fb = sm + ((static_cast<int>(g - gfirst) << lg_nch) + c) * a.FS;
    double2 b[D][W];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int jk = (jt >> (lg_nj * k)) & (nj - 1);
#pragma unroll
      for (int x = 0; x < W; ++x) b[k][x] = fb[(k * nj + jk) * W + x];
    }
    r1_tables<D, W, NA, NB>(val, b, A, B);
  }
  __syncthreads();  // factor blocks consumed: the tables alias them
  if (e1 < n1) {
    double2* dst = sm + e1 * TS;
#pragma unroll
    for (int i = 0; i < NA; ++i) dst[i] = A[i];
#pragma unroll
    for (int i = 0; i < NB; ++i) dst[NA + i] = B[i];
  }
  __syncthreads();
  // ---- phase 2: out(jt, x) = sum_c A_c(x_lo) B_c(x_hi), children ascending
  for (int e = threadIdx.x; e < nu * NX; e += blockDim.x) {
    const int x = e % NX, ul = e / NX;
    const int xlo = x % NA, xhi = x / NA;
    const double2* src = sm + (ul << lg_nch) * TS;
    double2 acc = cmul(src[xlo], src[NA + xhi]);
    for (int c = 1; c < nch; ++c) cfma(acc, src[c * TS + xlo], src[c * TS + NA + xhi]);
    const i64 u = u0 + ul;
    const i64 g = u >> lg_njd;
    const int jt = static_cast<int>(u & ((i64{1} << lg_njd) - 1));
    const i64 t = g & ((i64{1} << a.lg_nown) - 1), pnu = g >> a.lg_nown;
    out[r1_pu_out<D, W>(a, v, t, pnu, jt, x)] = acc;
  }
}

// P/U levels l >= 1 (the middle level Lc holds the bulk of the factor bytes):
// one WARP per unit (group (t, p_nu), block tuple jt).  The children are
// taken 32 at a time: the warp copies their factor blocks with cp.async into
// one of two warp-private shared-memory buffers (each lane computes one
// child's arena offset, the copy loop fetches it by shuffle; the next chunk's
// copies are in flight while this one is computed), lane c builds A_c / B_c
// (aliasing the buffer), and the outputs accumulate over the chunk's children
// with no CTA-wide barrier: for d = 6 (8 x 8 output per unit) as FP64
// tensor-core MMAs over 4-child k-steps, otherwise one lane per output summing
// the children in ascending order.
__device__ __forceinline__ void r1_cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}

// D(8x8) += A(8x4) * B(4x8), FP64 tensor core (per-lane fragments, see k_r1_pu_mid)
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int D, int W>
__global__ void __launch_bounds__(kR1VThreads, 3) k_r1_pu_mid(R1LevelArgs a, const double2* __restrict__ fac,
                                                              const double2* __restrict__ in,
                                                              double2* __restrict__ out) {
  extern __shared__ __align__(16) double2 wsm[];
  constexpr int H = D / 2;
  constexpr int NA = Pow<W, H>::v, NB = Pow<W, D - H>::v, NX = NA * NB;
  constexpr int TS = (NA + NB) | 1;
  constexpr int OPL = (NX + 31) / 32;  // outputs per lane
  const i64 v = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const i64 u = static_cast<i64>(blockIdx.x) * (kR1VThreads / 32) + warp;  // unit (group, block tuple)
  if (u >= a.nunits) return;
  const i64 g = u >> a.lg_njd;
  const int jt = static_cast<int>(u & ((i64{1} << a.lg_njd) - 1));
  constexpr int SL = ((D * W) | 1) > TS ? ((D * W) | 1) : TS;
  double2* ws = wsm + warp * 2 * 32 * SL;  // two chunk buffers (factor rows, then aliased tables)
  const i64 t = g & ((i64{1} << a.lg_nown) - 1), pnu = g >> a.lg_nown;  // groups t fastest
  const int nch = 1 << a.lg_nch, fblk = a.fblk;
  const int nchunk = (nch + 31) / 32;
  // chunk c0 / 32 -> buffer (c0 / 32) & 1: async copies of the chunk's factor
  // rows for this block tuple (d blocks of W per child)
  constexpr int DW = D * W;
  const int nj = 1 << a.lg_nj;
  auto prefetch = [&](int c0, double2& val) {
    const int cn = min(32, nch - c0);
    const i64 nuc = a.l > 0 ? r1_child<D>(pnu, a.l, c0 + lane) : 0;
    const i64 mybase = ((t << a.lg_nin) + nuc) * fblk;
    if (lane < cn)
      val = __ldg(in + (a.in_transposed ? (((v << a.lg_nmid) + nuc) << a.lg_nown) + t
                                        : (((((v << a.lg_nown) + t) << a.lg_nin) + nuc) << a.lg_njd) + jt));
    double2* buf = ws + ((c0 >> 5) & 1) * 32 * SL;
    for (int e0 = 0; e0 < cn * DW; e0 += 32) {
      const int e = min(e0 + lane, cn * DW - 1);
      const int cc = e / DW, r = e - cc * DW, k = r / W, x = r - k * W;
      const i64 base = __shfl_sync(0xffffffffu, mybase, cc);
      const int jk = (jt >> (a.lg_nj * k)) & (nj - 1);
      if (e0 + lane < cn * DW) r1_cp_async16(buf + cc * SL + r, fac + base + (k * nj + jk) * W + x);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // d = 6, W = 2 (config 4): the child sum is an 8 x 2^d x 8 complex GEMM per
  // unit -- run it on the FP64 tensor core (whole 4-child k-steps: 2^d % 4 == 0)
  constexpr bool kMma = NA == 8 && NB == 8;
  double2 acc[OPL];
#pragma unroll
  for (int i = 0; i < OPL; ++i) acc[i] = make_double2(0, 0);
  double cr[2] = {0, 0}, ci[2] = {0, 0};
  double2 val_cur = make_double2(0, 0), val_next = make_double2(0, 0);
  prefetch(0, val_cur);
  for (int ch = 0; ch < nchunk; ++ch) {
    const int c0 = ch * 32, cn = min(32, nch - c0);
    if (ch + 1 < nchunk) {
      prefetch(c0 + 32, val_next);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    double2* buf = ws + (ch & 1) * 32 * SL;
    double2 A[NA], B[NB];
    if (lane < cn) {
      double2 b[D][W];
#pragma unroll
      for (int k = 0; k < D; ++k)
#pragma unroll
        for (int x = 0; x < W; ++x) b[k][x] = buf[lane * SL + k * W + x];
      r1_tables<D, W, NA, NB>(val_cur, b, A, B);
    }
    __syncwarp();
    if (lane < cn) {
#pragma unroll
      for (int i = 0; i < NA; ++i) buf[lane * SL + i] = A[i];
#pragma unroll
      for (int i = 0; i < NB; ++i) buf[lane * SL + NA + i] = B[i];
    }
    __syncwarp();
    if constexpr (kMma) {
      // O(8 x 8) += A(8 x 4) B(4 x 8) per 4 children on the FP64 tensor core
      // (mma.sync m8n8k4: lane l holds A[l/4][l%4], B[l%4][l/4] and
      // C[l/4][2(l%4) + i]); complex = four real MMAs
      for (int k0 = 0; k0 < cn; k0 += 4) {
        const int cc = k0 + (lane & 3);
        const double2 av = buf[cc * SL + (lane >> 2)];
        const double2 bv = buf[cc * SL + NA + (lane >> 2)];
        dmma(cr, av.x, bv.x);
        dmma(cr, -av.y, bv.y);
        dmma(ci, av.x, bv.y);
        dmma(ci, av.y, bv.x);
      }
    } else {
#pragma unroll
      for (int i = 0; i < OPL; ++i) {
        const int o = lane + 32 * i;
        if (o < NX) {
          const int xlo = o % NA, xhi = o / NA;
          for (int cc = 0; cc < cn; ++cc) cfma(acc[i], buf[cc * SL + xlo], buf[cc * SL + NA + xhi]);
        }
      }
    }
    __syncwarp();  // the buffer is refilled two chunks later
    val_cur = val_next;
  }
  if constexpr (kMma) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int x = (lane >> 2) + NA * (2 * (lane & 3) + i);  // x_lo = l / 4, x_hi = 2 (l % 4) + i
      out[r1_pu_out<D, W>(a, v, t, pnu, jt, x)] = make_double2(cr[i], ci[i]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < OPL; ++i) {
      const int o = lane + 32 * i;
      if (o < NX) out[r1_pu_out<D, W>(a, v, t, pnu, jt, o)] = acc[i];
    }
  }
}

// Sharded exchange of the middle level (every block G_{t,s} is one element per
// vector): pack the level-Lc V/W output (v * nown + i) * nmid + t of the owned
// s = own[i] into the send buffer at send_off[t * nmid + s] * nv + v; unpack
// the receive buffer (recv_off[t * nmid + s] * nv + v, t = own[i]) into the
// level-Lc P/U input (v * nmid + s) * nown + i.
__global__ void __launch_bounds__(256) k_r1_pack(R1LevelArgs a, const long long* __restrict__ send_off,
                                                 const double2* __restrict__ in, double2* __restrict__ out) {
  const i64 total = i64{1} << (a.lg_nown + a.lg_nmid);
  for (i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; e < total * a.nv;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 v = e >> (a.lg_nown + a.lg_nmid), r = e & (total - 1);
    const i64 i = r >> a.lg_nmid, t = r & ((i64{1} << a.lg_nmid) - 1);
    const i64 s = a.own[i];
    out[send_off[(t << a.lg_nmid) + s] * a.nv + v] = in[e];
  }
}
__global__ void __launch_bounds__(256) k_r1_unpack(R1LevelArgs a, const long long* __restrict__ recv_off,
                                                   const double2* __restrict__ in, double2* __restrict__ out) {
  const i64 total = i64{1} << (a.lg_nown + a.lg_nmid);
  for (i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; e < total * a.nv;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 v = e >> (a.lg_nown + a.lg_nmid), r = e & (total - 1);
    const i64 s = r >> a.lg_nown, i = r & ((i64{1} << a.lg_nown) - 1);  // output order: t fastest
    const i64 t = a.own[i];
    out[e] = in[recv_off[(t << a.lg_nmid) + s] * a.nv + v];
  }
}

template <int D, int W>
void launch_r1_dw(const R1LevelArgs& a, const double2* fac, const double2* cores, const double2* in, double2* out,
                  cudaStream_t st) {
  const size_t smem = r1_smem_bytes(a);
  if (a.side == 0 && a.warp_tiles) {
    const i64 tiles = i64{1} << (a.lg_nown + a.lg_nin - 5);
    const dim3 grid(static_cast<unsigned>((tiles + kR1VThreads / 32 - 1) / (kR1VThreads / 32)), static_cast<unsigned>(a.nv));
    TBF_CUDA(cudaFuncSetAttribute(k_r1_vw_mid<D, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    k_r1_vw_mid<D, W><<<grid, kR1VThreads, smem, st>>>(a, fac, cores, in, out);
  } else if (a.side == 0) {
    const dim3 grid(static_cast<unsigned>(i64{1} << (a.lg_nown + a.lg_nin - a.lg_T)), static_cast<unsigned>(a.nv));
    TBF_CUDA(cudaFuncSetAttribute(k_r1_vw<D, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    k_r1_vw<D, W><<<grid, kR1Threads, smem, st>>>(a, fac, cores, in, out);
  } else if (a.warp_tiles) {
    const dim3 grid(static_cast<unsigned>((a.nunits + kR1VThreads / 32 - 1) / (kR1VThreads / 32)), static_cast<unsigned>(a.nv));
    TBF_CUDA(cudaFuncSetAttribute(k_r1_pu_mid<D, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    k_r1_pu_mid<D, W><<<grid, kR1VThreads, smem, st>>>(a, fac, in, out);
  } else {
    const dim3 grid(static_cast<unsigned>((a.nunits + a.gpb - 1) / a.gpb), static_cast<unsigned>(a.nv));
    TBF_CUDA(cudaFuncSetAttribute(k_r1_pu<D, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    k_r1_pu<D, W><<<grid, kR1Threads, smem, st>>>(a, fac, in, out);
  }
}

template <int D>
void launch_r1_d(const R1LevelArgs& a, const double2* fac, const double2* cores, const double2* in, double2* out,
                 cudaStream_t st) {
  if (a.W == 1) launch_r1_dw<D, 1>(a, fac, cores, in, out, st);
  else launch_r1_dw<D, 2>(a, fac, cores, in, out, st);
}

}  // namespace

size_t r1_smem_bytes(const R1LevelArgs& a) {
  if (a.side == 0 && a.warp_tiles)
    return sizeof(double2) * (kR1VThreads / 32) * (static_cast<size_t>(a.Pc) * a.XS + 32 * static_cast<size_t>(a.FS));
  if (a.side == 0) return sizeof(double2) * (static_cast<size_t>(a.Pc) * a.XS + (size_t{1} << a.lg_T) * a.FS);
  const int H = a.d / 2;
  int na = 1, nb = 1;
  for (int k = 0; k < H; ++k) na *= a.W;
  for (int k = H; k < a.d; ++k) nb *= a.W;
  const size_t ts = static_cast<size_t>((na + nb) | 1);
  if (a.warp_tiles)
    return sizeof(double2) * (kR1VThreads / 32) * 2 * 32 * std::max<size_t>(ts, static_cast<size_t>((a.d * a.W) | 1));
  const size_t tabs = (static_cast<size_t>(a.gpb) << a.lg_nch) * ts;
  const size_t ngr = std::max<size_t>(1, static_cast<size_t>(a.gpb) >> a.lg_njd);  // groups a CTA's units span
  const size_t facs = (ngr << a.lg_nch) * static_cast<size_t>(a.FS);
  return sizeof(double2) * std::max(tabs, facs);
}

void launch_r1_exchange(const R1LevelArgs& a, int unpack, const long long* off, const double2* in, double2* out,
                        cudaStream_t st) {
  const i64 total = (i64{1} << (a.lg_nown + a.lg_nmid)) * a.nv;
  const unsigned grid = static_cast<unsigned>(std::min<i64>((total + 255) / 256, 148 * 16));
  if (unpack) k_r1_unpack<<<grid, 256, 0, st>>>(a, off, in, out);
  else k_r1_pack<<<grid, 256, 0, st>>>(a, off, in, out);
  TBF_CUDA(cudaGetLastError());
}

int r1_threads() { return kR1Threads; }
int r1_vthreads() { return kR1VThreads; }

void launch_r1_level(const R1LevelArgs& a, const double2* fac, const double2* cores, const double2* in, double2* out,
                     cudaStream_t st) {
  if (a.W != 1 && a.W != 2) throw std::runtime_error("rank-one engine: box width must be 1 or 2");
  if (a.side == 1 && (static_cast<i64>(a.gpb) << a.lg_nch) > kR1Threads)
    throw std::runtime_error("rank-one engine: P/U units exceed the CTA");
  switch (a.d) {
    case 1: launch_r1_d<1>(a, fac, cores, in, out, st); break;
    case 2: launch_r1_d<2>(a, fac, cores, in, out, st); break;
    case 3: launch_r1_d<3>(a, fac, cores, in, out, st); break;
    case 4: launch_r1_d<4>(a, fac, cores, in, out, st); break;
    case 5: launch_r1_d<5>(a, fac, cores, in, out, st); break;
    case 6: launch_r1_d<6>(a, fac, cores, in, out, st); break;
    default: throw std::runtime_error("rank-one engine: d out of range");
  }
  TBF_CUDA(cudaGetLastError());
}

}  // namespace tbf
