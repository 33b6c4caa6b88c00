// Apply engine for butterflies made of tiny boxes (config 4: d = 6, every
// block has 1 or 2 rows/columns per mode, 1.7e7 middle pairs, ~1e8 boxes).
// Per-box descriptors would need tens of GB, and one CTA per box would be
// launch-bound, so this engine is metadata-light and thread-per-output:
//
//   k_tiny_level  one thread per output element of a level.  Items are the
//                 level's output tensors (V/W: (s, tau); P/U: parents
//                 (t, p_nu)); the thread finds its item by binary search over
//                 the items' output prefix, decodes its position, and for each
//                 contributing child box (one on the V/W side, the 2^d
//                 children nu of p_nu in ascending order on the P/U side,
//                 PAPER.md Alg. 2) evaluates the multilinear sum
//                 out(a) = sum_x in(x) prod_k M_k(a_k, x_k)
//                 directly over the box (<= kTinyBox elements).  Block
//                 geometry (ranks, widths, interp offsets) is read from the
//                 level's slot arrays: nothing per box is stored.
//   k_tiny_gemv   one thread per core row: y_r = sum_c K(r, c) x_c.
#include "kernels.h"

namespace tbf {

namespace {

__device__ __forceinline__ i64 find_item(const TinyItem* __restrict__ items, i64 n, i64 e) {
  i64 lo = 0, hi = n - 1;
  while (lo < hi) {
    const i64 mid = (lo + hi + 1) >> 1;
    if (items[mid].out_start <= e) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void k_tiny_level(TinyLevelArgs a, const TinyItem* __restrict__ items,
                             const i64* __restrict__ in_off_of, const int* __restrict__ rank,
                             const int* __restrict__ width, const i64* __restrict__ moff,
                             const double2* __restrict__ mats, const double2* __restrict__ in,
                             double2* __restrict__ out) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= a.total_out) return;
  const i64 it = find_item(items, a.nitems, e);
  const TinyItem I = items[it];
  const int d = a.d;
  const i64 nj = a.nj;
  // output extents of the item: V/W sum_j r(k, j); P/U sum_j w(k, j) (common
  // to all children of a parent, so child 0 describes them)
  const i64 first_inner = a.side == 0 ? I.inner : (a.l == 0 ? 0 : I.first_child);
  auto slot_of = [&](i64 inner, int k, i64 j) { return ((I.outer * a.nin + inner) * d + k) * nj + j; };
  i64 rem = e - I.out_start;
  int pos[kMaxD];
  i64 oext[kMaxD];
  for (int k = 0; k < d; ++k) {
    i64 ext = 0;
    for (i64 j = 0; j < nj; ++j) {
      const i64 sl = slot_of(first_inner, k, j);
      ext += a.side == 0 ? rank[sl] : width[sl];
    }
    oext[k] = ext;
    pos[k] = static_cast<int>(rem % ext);
    rem /= ext;
  }
  const i64 v = rem;
  // output address
  i64 oaddr = I.out_off;
  {
    i64 st = 1;
    for (int k = 0; k < d; ++k) {
      const i64 sk = a.out_global ? a.gstride[k] : st;
      oaddr += pos[k] * sk;
      st *= oext[k];
    }
    oaddr += v * (a.out_global ? a.gstride[d] : st);
  }
  double2 acc = make_double2(0, 0);
  const int nchild = a.side == 0 || a.l == 0 ? 1 : (1 << d);
  for (int c = 0; c < nchild; ++c) {
    // the contributing box-group (outer, inner)
    i64 inner;
    if (a.side == 0) {
      inner = I.inner;
    } else if (a.l == 0) {
      inner = 0;
    } else {  // child c of parent p_nu: mode p coordinate 2 * pc_p + bit_p (ascending nu)
      inner = 0;
      for (int p = d - 1; p >= 0; --p) {
        const i64 pc = (I.inner >> ((a.l - 1) * p)) & ((i64{1} << (a.l - 1)) - 1);
        inner = (inner << a.l) | (2 * pc + ((c >> p) & 1));
      }
    }
    const i64 base_in = in_off_of[I.outer * a.nin + inner];
    // per mode: block j, position inside it, input extents and offsets
    int al[kMaxD], iw[kMaxD];
    i64 ioff = base_in, istr[kMaxD + 1], mo[kMaxD];
    int rr[kMaxD];
    {
      i64 st = 1;
      for (int k = 0; k < d; ++k) {
        i64 opre = 0, ipre = 0, iext = 0;
        int jb = -1, alk = 0, iwk = 0, rk = 0;
        i64 mok = 0;
        for (i64 j = 0; j < nj; ++j) {
          const i64 sl = slot_of(inner, k, j);
          const int r = rank[sl], w = width[sl];
          const int ob = a.side == 0 ? r : w;  // output block extent
          const int ib = a.side == 0 ? w : r;  // input block extent
          if (jb < 0 && pos[k] < opre + ob) {
            jb = static_cast<int>(j);
            alk = static_cast<int>(pos[k] - opre);
            iwk = ib;
            rk = r;
            mok = moff[sl];
            ipre = iext;
          }
          opre += ob;
          iext += ib;
        }
        al[k] = alk;
        iw[k] = iwk;
        rr[k] = rk;
        mo[k] = mok;
        istr[k] = a.in_global ? a.gstride[k] : st;
        ioff += ipre * istr[k];
        st *= iext;
      }
      istr[d] = a.in_global ? a.gstride[d] : st;
    }
    ioff += v * istr[d];
    // sum over the box: mixed-radix counter over x
    int x[kMaxD];
    i64 box = 1;
    for (int k = 0; k < d; ++k) {
      x[k] = 0;
      box *= iw[k];
    }
    for (i64 q = 0; q < box; ++q) {
      i64 addr = ioff;
      double2 wgt = make_double2(1, 0);
      for (int k = 0; k < d; ++k) {
        addr += x[k] * istr[k];
        // V/W: M = B (r x w): M(a, x) = B[a + r x];  P/U: M = B^T: M(a, x) = B[x + r a]
        const i64 mi = a.side == 0 ? al[k] + static_cast<i64>(rr[k]) * x[k] : x[k] + static_cast<i64>(rr[k]) * al[k];
        wgt = cmul(wgt, mats[mo[k] + mi]);
      }
      cfma(acc, in[addr], wgt);
      for (int k = 0; k < d; ++k) {
        if (++x[k] < iw[k]) break;
        x[k] = 0;
      }
    }
  }
  out[oaddr] = acc;
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

void launch_tiny_level(const TinyLevelArgs& a, const TinyItem* items, const i64* in_off_of, const int* rank,
                       const int* width, const i64* moff, const double2* mats, const double2* in, double2* out,
                       cudaStream_t st) {
  if (a.total_out == 0) return;
  k_tiny_level<<<static_cast<unsigned>((a.total_out + 127) / 128), 128, 0, st>>>(a, items, in_off_of, rank, width,
                                                                                 moff, mats, in, out);
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
