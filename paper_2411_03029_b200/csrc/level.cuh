// Level descriptors shared by the construction kernels and the host runtime.
//
// Canonical slot order, for one side and level l:
//   idx = ((outer * nin + inner) * d + k) * nj + j
//   side 0 (V/W):  outer = s   (mid column multi-set, level Lc)
//                  inner = tau (row multi-set at level l), node nu = (L-l, s_k*nj + j)
//                  unfolded mode d+k  (Alg. 1)
//   side 1 (U/P):  outer = t, inner = nu (column multi-set at level l),
//                  node tau = (L-l, t_k*nj + j), unfolded mode k (Alg. 1)
// Multi-set indices are mixed radix, mode 0 fastest.  Node (lev, pos) covers
// 1-based [pos*(n>>lev)+1, (pos+1)*(n>>lev)].
#pragma once

#include "common.cuh"

namespace tbf {

constexpr int kMaxD = 6;
constexpr int kMaxModes = 2 * kMaxD;
constexpr int kMaxW = 96;  // widest ID (candidate columns) supported by the SMEM kernels

struct LevelDesc {
  int d, side, l, L, Lc;
  int proxy_mode;
  i64 n;
  i64 nslots, nin, nj, mpm;
  i64 m;       // proxy rows per ID (uniform over the level)
  i64 psize;   // proxy ints per slot (max over k of the per-slot list total)
  i64 wmax;    // max candidate columns
  i64 per_mode;
  u64 seed;
  u64 side_tag;
  int counts[kMaxD][kMaxModes];  // per unfolded-mode k, per range p (0 at skip)
  int poff[kMaxD][kMaxModes];    // list offsets within the slot's proxy block
  // panel decomposition
  i64 nparts;  // row partitions per ID
  i64 rpp;     // rows per partition
  int pr;      // panel rows
  // children (level l-1) for l >= 1
  i64 c_nin, c_nj;
  // sharded construction: this rank builds only slots whose outer middle
  // multi-set belongs to it (others get width 0 -> rank 0): owner[outer] ==
  // rank when a device ownership map is set, outer % world == rank otherwise
  int rank, world;
  const int* owner;
};

__device__ inline bool owns_outer(const LevelDesc& L, i64 outer) {
  if (L.world <= 1) return true;
  return (L.owner ? L.owner[outer] : static_cast<int>(outer % L.world)) == L.rank;
}

struct SlotPos {
  i64 outer, inner, k, j;
  i64 lo[kMaxModes], sz[kMaxModes];
  int skip;
};

__host__ __device__ inline SlotPos decode_slot(const LevelDesc& L, i64 idx) {
  SlotPos s;
  s.j = idx % L.nj;
  s.k = (idx / L.nj) % L.d;
  s.inner = (idx / (L.nj * L.d)) % L.nin;
  s.outer = idx / (L.nj * L.d * L.nin);
  const int mid_off = L.side == 0 ? L.d : 0;
  const int in_off = L.side == 0 ? 0 : L.d;
  for (int p = 0; p < L.d; ++p) {
    const i64 op = (s.outer >> (L.Lc * p)) & (L.mpm - 1);
    const i64 ip = (s.inner >> (L.l * p)) & ((i64{1} << L.l) - 1);
    const i64 msz = L.n >> L.Lc, isz = L.n >> L.l;
    s.lo[mid_off + p] = op * msz + 1;
    s.sz[mid_off + p] = msz;
    s.lo[in_off + p] = ip * isz + 1;
    s.sz[in_off + p] = isz;
  }
  s.skip = mid_off + static_cast<int>(s.k);
  const i64 op_k = (s.outer >> (L.Lc * s.k)) & (L.mpm - 1);
  const i64 nsz = L.n >> (L.L - L.l);
  s.lo[s.skip] = (op_k * L.nj + s.j) * nsz + 1;
  s.sz[s.skip] = nsz;
  return s;
}

// Level l-1 slot holding child c (0/1) of slot `idx` at level l >= 1.
__host__ __device__ inline i64 child_slot(const LevelDesc& L, const SlotPos& s, int c) {
  i64 pin = 0;
  for (int p = L.d - 1; p >= 0; --p) {
    const i64 ip = (s.inner >> (L.l * p)) & ((i64{1} << L.l) - 1);
    pin = (pin << (L.l - 1)) | (ip >> 1);
  }
  return ((s.outer * L.c_nin + pin) * L.d + s.k) * L.c_nj + 2 * s.j + c;
}

}  // namespace tbf
