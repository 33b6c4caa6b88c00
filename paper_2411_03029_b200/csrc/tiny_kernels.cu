// Apply engine for butterflies made of tiny boxes (config 4: d = 6, every
// block has 1 or 2 rows/columns per mode, 1.7e7 middle pairs, ~1e8 boxes).
// Per-box descriptors would need tens of GB and one CTA per box would be
// launch-bound, so this engine is metadata-light:
//
//   k_tiny_level  one CTA per GROUP of boxes that share data.
//                 V/W level l: the 2^d children tau of a parent (s, p_tau)
//                 all contract the parent's output tensor with their own
//                 factors (l = 0: the single item (s, 0) reading the F slab).
//                 P/U level l: the 2^d children nu of a parent (t, p_nu) all
//                 add into the parent's output (Alg. 2;
//                 ascending nu, as the reference).  The CTA loads the group's
//                 block geometry (rank / width / interp offset per child,
//                 mode and block) and its input into shared memory once, then
//                 sweeps the group's output elements; each output is the
//                 multilinear sum  sum_x in(x) prod_k M_k(a_k, x_k)  over its
//                 box, with the factor product updated incrementally
//                 (about one complex multiply per box element).
//   k_tiny_gemv   one thread per core row: y_r = sum_c K(r, c) x_c.
#include "kernels.h"

namespace tbf {

namespace {

constexpr int kTinyThreads = 256;

// shared-memory layout of one group (host and device agree)
struct TinyLayout {
  int nsl;  // nch * d * nj slot entries
  int nck;  // nch * d (child, mode) pairs
  int ntab; // nch * d * maxo (child, mode, output coordinate) table entries
  __host__ __device__ TinyLayout(const TinyLevelArgs& a)
      : nsl(a.nch * a.d * static_cast<int>(a.nj)), nck(a.nch * a.d), ntab(a.nch * a.d * static_cast<int>(a.maxo)) {}
  // slot entries: moff (i64) + r, w, out-prefix, in-prefix, factor-prefix (int);
  // (child, mode): out ext, in ext, input stride (int); child: output size,
  // input stride of the nv mode (int), global offset (i64); table: factor base
  // (i64) + factor step, box extent, input offset (int); then factor blocks
  // (nch * d * fstride) and the staged input (double2)
  __host__ __device__ size_t bytes_meta(const TinyLevelArgs& a) const {
    const size_t b = 28 * static_cast<size_t>(nsl) + 12 * static_cast<size_t>(nck) + 16 * static_cast<size_t>(a.nch) +
                     20 * static_cast<size_t>(ntab);
    return (b + 15) / 16 * 16;
  }
  __host__ __device__ size_t fac_elems(const TinyLevelArgs& a) const {
    return static_cast<size_t>(a.nch) * a.d * static_cast<size_t>(a.fstride);
  }
};

template <int D>  // d, compile time: per-mode state stays in registers
__global__ void __launch_bounds__(kTinyThreads) k_tiny_level(TinyLevelArgs a, const TinyGroup* __restrict__ groups,
                                                             const i64* __restrict__ off_of,
                                                             const int* __restrict__ rank,
                                                             const int* __restrict__ width,
                                                             const i64* __restrict__ moff,
                                                             const double2* __restrict__ mats,
                                                             const double2* __restrict__ in,
                                                             double2* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const TinyLayout lay(a);
  constexpr int d = D;
  const int nch = a.nch, nj = static_cast<int>(a.nj), nsl = lay.nsl, nck = lay.nck;
  const int maxo = static_cast<int>(a.maxo);
  unsigned char* p = smem;
  i64* s_mo = reinterpret_cast<i64*>(p);
  p += 8 * nsl;
  i64* t_fb = reinterpret_cast<i64*>(p);  // table: factor base index
  p += 8 * lay.ntab;
  i64* s_go = reinterpret_cast<i64*>(p);  // [child] global offset (V/W output, P/U input)
  p += 8 * nch;
  int* s_r = reinterpret_cast<int*>(p);
  int* s_w = s_r + nsl;
  int* s_po = s_w + nsl;  // prefix of output blocks (V/W: r, P/U: w) over j
  int* s_pi = s_po + nsl;  // prefix of input blocks (V/W: w, P/U: r) over j
  int* s_pf = s_pi + nsl;  // factor-block offset in fm
  int* s_oe = s_pf + nsl;  // [child][mode] output extent
  int* s_ie = s_oe + nck;  // [child][mode] input extent
  int* s_is = s_ie + nck;  // [child][mode] input stride
  int* s_cs = s_is + nck;  // [child] output elements
  int* s_isv = s_cs + nch; // [child] input stride of the nv mode
  int* t_fs = s_isv + nch; // table: factor step per x
  int* t_iw = t_fs + lay.ntab;  // table: box extent
  int* t_io = t_iw + lay.ntab;  // table: input offset term
  double2* fm = reinterpret_cast<double2*>(smem + lay.bytes_meta(a));  // factor blocks
  double2* xs = fm + lay.fac_elems(a);                                   // staged input
  const bool fsm = a.fstride > 0;
  const TinyGroup g = groups[blockIdx.x];
  const int tid = threadIdx.x;
  const int nth = static_cast<int>(blockDim.x);
  // inner index of child c (ascending nu / tau)
  auto child_inner = [&](int c) -> i64 {
    if (a.l == 0) return 0;
    i64 inner = 0;
    for (int q = d - 1; q >= 0; --q) {
      const i64 pc = (g.pinner >> ((a.l - 1) * q)) & ((i64{1} << (a.l - 1)) - 1);
      inner = (inner << a.l) | (2 * pc + ((c >> q) & 1));
    }
    return inner;
  };
  // ---- block geometry of every child, mode and block
  for (int e = tid; e < nsl; e += nth) {
    const int j = e % nj, k = (e / nj) % d, c = e / (nj * d);
    const i64 sl = ((g.outer * a.nin + child_inner(c)) * d + k) * a.nj + j;
    s_mo[e] = moff[sl];
    s_r[e] = rank[sl];
    s_w[e] = width[sl];
  }
  for (int c = tid; c < nch; c += nth) s_go[c] = off_of[g.outer * a.nin + child_inner(c)];
  __syncthreads();
  for (int ck = tid; ck < nck; ck += nth) {
    int po = 0, pi = 0, pf = ck * static_cast<int>(a.fstride);
    for (int j = 0; j < nj; ++j) {
      const int e = ck * nj + j;
      s_po[e] = po;
      s_pi[e] = pi;
      s_pf[e] = pf;
      po += a.side == 0 ? s_r[e] : s_w[e];
      pi += a.side == 0 ? s_w[e] : s_r[e];
      pf += s_r[e] * s_w[e];
    }
    s_oe[ck] = po;
    s_ie[ck] = pi;
  }
  __syncthreads();
  for (int c = tid; c < nch; c += nth) {
    int so = a.nv, st = 1;
    for (int k = 0; k < d; ++k) {
      so *= s_oe[c * d + k];
      s_is[c * d + k] = st;
      st *= s_ie[c * d + k];
    }
    s_cs[c] = so;
    s_isv[c] = st;
  }
  __syncthreads();
  // ---- table over (child, mode, output coordinate): block, factor base / step, box extent, input offset
  for (int t = tid; t < lay.ntab; t += nth) {
    const int ck = t / maxo, pos = t - ck * maxo;
    if (pos >= s_oe[ck]) continue;
    const int base = ck * nj;
    int j = 0;
    while (j + 1 < nj && pos >= s_po[base + j + 1]) ++j;
    const int e = base + j;
    const int al = pos - s_po[e], r = s_r[e];
    // V/W: M(a, x) = B[a + r x];  P/U: M(a, x) = B^T = B[x + r a]
    t_fb[t] = (fsm ? static_cast<i64>(s_pf[e]) : s_mo[e]) + (a.side == 0 ? al : static_cast<i64>(r) * al);
    t_fs[t] = a.side == 0 ? r : 1;
    t_iw[t] = a.side == 0 ? s_w[e] : r;
    t_io[t] = s_pi[e] * s_is[ck];
  }
  // ---- stage the factor blocks (r x w column-major each) ...
  if (fsm)
    for (int e = tid; e < nsl; e += nth) {  // blocks are tiny: one thread per block
      const int sz = s_r[e] * s_w[e];
      for (int q = 0; q < sz; ++q) fm[s_pf[e] + q] = __ldg(mats + s_mo[e] + q);
    }
  // ---- ... and the input(s): packed first-mode-fastest (or global strides at V0);
  // one flat loop over (child, element) so tiny children do not serialize
  {
    const int nsrc = a.side == 0 ? 1 : nch;
    const int xst = a.side == 0 ? s_isv[0] * a.nv : static_cast<int>(a.xstride);
    for (int e = tid; e < nsrc * xst; e += nth) {
      const int c = e / xst, loc = e - c * xst;
      if (loc >= s_isv[c] * a.nv) continue;
      const i64 base = a.side == 0 ? g.io_off : s_go[c];
      int rem = loc;
      i64 addr = base;
      int st = 1;
      for (int k = 0; k < d; ++k) {
        const int ext = s_ie[c * d + k];
        const int q = rem / ext;
        const int x = rem - q * ext;
        rem = q;
        addr += a.in_global ? x * a.gstride[k] : static_cast<i64>(x * st);
        st *= ext;
      }
      addr += a.in_global ? rem * a.gstride[d] : static_cast<i64>(rem * st);
      xs[(a.side == 0 ? 0 : c * static_cast<int>(a.xstride)) + loc] = in[addr];
    }
  }
  __syncthreads();
  const double2* F = fsm ? fm : mats;
  // ---- outputs.  V/W: child c's outputs are [c * ostride, c * ostride + size_c)
  const int total = a.side == 0 ? nch * static_cast<int>(a.ostride) : s_cs[0];
  for (int e = tid; e < total; e += nth) {
    int c0 = 0;
    int loc = e;
    if (a.side == 0) {
      c0 = e / static_cast<int>(a.ostride);
      loc = e - c0 * static_cast<int>(a.ostride);
      if (loc >= s_cs[c0]) continue;
    }
    int pos[D];
    i64 oaddr = 0;
    int ost = 1;
#pragma unroll
    for (int k = 0; k < d; ++k) {
      const int ext = s_oe[c0 * d + k];
      const int q = loc / ext;
      pos[k] = loc - q * ext;
      loc = q;
      oaddr += a.out_global ? pos[k] * a.gstride[k] : static_cast<i64>(pos[k] * ost);
      ost *= ext;
    }
    oaddr += a.out_global ? loc * a.gstride[d] : static_cast<i64>(loc * ost);
    const int v = loc;
    double2 acc = make_double2(0, 0);
    const int cb = a.side == 0 ? c0 : 0, ce = a.side == 0 ? c0 + 1 : nch;
    for (int c = cb; c < ce; ++c) {
      int iw[D], fs[D], istr[D];
      i64 fb[D];
      int ioff = (a.side == 0 ? 0 : c * static_cast<int>(a.xstride)) + v * s_isv[c];
      bool empty = false;
#pragma unroll
      for (int k = 0; k < d; ++k) {
        const int t = (c * d + k) * maxo + pos[k];
        fb[k] = t_fb[t];
        fs[k] = t_fs[t];
        iw[k] = t_iw[t];
        ioff += t_io[t];
        istr[k] = s_is[c * d + k];
        empty |= iw[k] == 0;
      }
      if (empty) continue;
      // incremental product over the box: pp[k] = prod_{k' >= k} M_k'(x_k')
      int x[D];
      double2 pp[D + 1];
      pp[d] = make_double2(1, 0);
#pragma unroll
      for (int k = d - 1; k >= 0; --k) {
        x[k] = 0;
        pp[k] = cmul(F[fb[k]], pp[k + 1]);
      }
      int addr = ioff;
      for (;;) {
        cfma(acc, xs[addr], pp[0]);
        // advance the mixed-radix counter (mode 0 fastest); kc = highest mode changed
        int kc = d;
#pragma unroll
        for (int k = 0; k < d; ++k) {
          if (kc == d) {
            addr += istr[k];
            if (++x[k] < iw[k]) {
              kc = k;
            } else {
              addr -= iw[k] * istr[k];
              x[k] = 0;
            }
          }
        }
        if (kc == d) break;
#pragma unroll
        for (int q = d - 1; q >= 0; --q)
          if (q <= kc) pp[q] = cmul(F[fb[q] + static_cast<i64>(fs[q]) * x[q]], pp[q + 1]);
      }
    }
    const i64 ob = a.side == 0 ? s_go[c0] : g.io_off;
    out[ob + oaddr] = acc;
  }
}

__global__ void k_tiny_gemv(const GemvDesc* __restrict__ ds, i64 npairs, i64 total_rows, int nv,
                            const double2* __restrict__ cores, const double2* __restrict__ x,
                            double2* __restrict__ y) {
  const i64 g = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= total_rows * nv) return;
  const i64 v = g / total_rows, row = g - v * total_rows;
  i64 lo = 0, hi = npairs - 1;
  while (lo < hi) {
    const i64 mid = (lo + hi + 1) >> 1;
    if (ds[mid].cta_off <= row) lo = mid;
    else hi = mid - 1;
  }
  const GemvDesc D = ds[lo];
  const i64 r = row - D.cta_off;
  const double2* krow = cores + D.core_off + r * D.C;
  const double2* xv = x + D.x_off + v * D.C;
  double2 acc = make_double2(0, 0);
  for (int c = 0; c < D.C; ++c) cfma(acc, krow[c], xv[c]);
  y[D.y_off + r + v * D.R] = acc;
}

}  // namespace

size_t tiny_smem_bytes(const TinyLevelArgs& a) {
  const TinyLayout lay(a);
  return lay.bytes_meta(a) + sizeof(double2) * (lay.fac_elems(a) + static_cast<size_t>(a.max_in));
}

void launch_tiny_level(const TinyLevelArgs& a, const TinyGroup* groups, const i64* off_of, const int* rank,
                       const int* width, const i64* moff, const double2* mats, const double2* in, double2* out,
                       cudaStream_t st) {
  if (a.ngroups == 0) return;
  const size_t smem = tiny_smem_bytes(a);
  if (smem > static_cast<size_t>(kMaxDynSmem)) throw std::runtime_error("tiny engine: group does not fit on chip");
  auto go = [&](auto kern) {
    TBF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    kern<<<static_cast<unsigned>(a.ngroups), a.threads, smem, st>>>(a, groups, off_of, rank, width, moff, mats, in,
                                                                    out);
  };
  switch (a.d) {
    case 1: go(k_tiny_level<1>); break;
    case 2: go(k_tiny_level<2>); break;
    case 3: go(k_tiny_level<3>); break;
    case 4: go(k_tiny_level<4>); break;
    case 5: go(k_tiny_level<5>); break;
    case 6: go(k_tiny_level<6>); break;
    default: throw std::runtime_error("tiny engine: d out of range");
  }
  TBF_CUDA(cudaGetLastError());
}

void launch_tiny_gemv(const GemvDesc* d, i64 npairs, i64 total_rows, int nv, const double2* cores, const double2* x,
                      double2* y, cudaStream_t st) {
  if (total_rows == 0) return;
  const i64 n = total_rows * nv;
  k_tiny_gemv<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(d, npairs, total_rows, nv, cores, x, y);
  TBF_CUDA(cudaGetLastError());
}

}  // namespace tbf
