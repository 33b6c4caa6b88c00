// oiobf drop-in: the tensor butterfly sharded over several GPUs of one process
// (PAPER.md:502 -- the reference's distributed setting).
//
// Host orchestration in C++ over the C ABI, no Python: one library handle per
// device (rank r of `devices.size()`), each owning the middle multi-sets o with
// owner(o) == r on both sides -- o % world by default, or an ownership map
// (`balanced_owners`: byte-balanced over the measured per-s core bytes;
// `tbf_construct_sharded_balanced` measures and applies it):
//   construction  per side and level, every rank builds its slots (one host
//                 thread per distinct device), then r_est = max over ranks
//                 (identical to the single-GPU r_est); the
//                 U-side middle skeletons are summed across ranks on the host
//                 (every rank needs the row skeletons of all t for its cores)
//   apply         phase 1 (V/W levels + core GEMV of the owned s) on every
//                 device, the exchange of the blocks G_{t,s} as peer copies
//                 (NVLink / NVSwitch) straight from each sender's send buffer
//                 into each receiver's receive buffer, phase 2 (P/U levels of
//                 the owned t) on every device
// The same device may appear several times (ranks then share it and run one
// after the other -- the test configuration on a one-GPU box).  The
// multi-process equivalent (one process per GPU, NCCL) is
// paper_2411_03029_b200/sharded.py; both use the same exchange layout.
#ifndef OIOBF_DROPIN_SHARDED_HPP
#define OIOBF_DROPIN_SHARDED_HPP

#include <algorithm>
#include <functional>
#include <memory>
#include <set>
#include <thread>
#include <vector>

#include "oiobf/butterfly.hpp"

namespace oiobf {

namespace detail {

inline std::int64_t owner_of(std::int64_t outer, std::int64_t world, const std::vector<std::int32_t>& owners) {
  return owners.empty() ? outer % world : owners[static_cast<std::size_t>(outer)];
}
inline bool owns_outer(std::int64_t outer, std::int64_t rank, std::int64_t world,
                       const std::vector<std::int32_t>& owners = {}) {
  return world <= 1 || owner_of(outer, world, owners) == rank;
}

// run f(r) for every rank: concurrently (one host thread per rank) when the
// devices are distinct, in rank order when some device is shared
inline void for_ranks(const std::vector<int>& devices, const std::function<void(std::size_t)>& f) {
  const std::set<int> distinct(devices.begin(), devices.end());
  if (distinct.size() < devices.size()) {
    for (std::size_t r = 0; r < devices.size(); ++r) f(r);
    return;
  }
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> err(devices.size());
  for (std::size_t r = 0; r < devices.size(); ++r)
    th.emplace_back([&, r] {
      try {
        f(r);
      } catch (...) {
        err[r] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

struct DeviceBuffer {
  void* p = nullptr;
  int device = 0;
  DeviceBuffer() = default;
  DeviceBuffer(int dev, std::int64_t bytes) : device(dev) {
    check(oiobf_set_device(dev));
    check(oiobf_device_alloc(std::max<std::int64_t>(bytes, 16), &p));
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() {
    if (p) {
      oiobf_set_device(device);
      oiobf_device_free(p);
    }
  }
};

}  // namespace detail

// Exchange layout of one rank (sharded.py exchange_layout): the send buffer
// holds, per destination q ascending, the blocks (t owned by q, s owned by me)
// in (t, s) order; the receive buffer, per source q ascending, the blocks
// (t owned by me, s owned by q) in the same order -- sender and receiver agree
// without metadata.  Offsets in elements at n_v = 1 (-1: not this rank's).
struct ShardLayout {
  std::vector<std::int64_t> send_off, recv_off, send_counts, recv_counts;
  std::int64_t send_total() const {
    std::int64_t s = 0;
    for (auto c : send_counts) s += c;
    return s;
  }
  std::int64_t recv_total() const {
    std::int64_t s = 0;
    for (auto c : recv_counts) s += c;
    return s;
  }
};

inline ShardLayout shard_layout(const std::vector<std::int64_t>& R, std::int64_t nmid, std::int64_t rank,
                                std::int64_t world, const std::vector<std::int32_t>& owners = {}) {
  ShardLayout lay;
  lay.send_off.assign(static_cast<std::size_t>(nmid * nmid), -1);
  lay.recv_off.assign(static_cast<std::size_t>(nmid * nmid), -1);
  lay.send_counts.assign(static_cast<std::size_t>(world), 0);
  lay.recv_counts.assign(static_cast<std::size_t>(world), 0);
  std::int64_t cur = 0;
  for (std::int64_t q = 0; q < world; ++q) {
    const std::int64_t start = cur;
    for (std::int64_t t = 0; t < nmid; ++t) {
      if (!detail::owns_outer(t, q, world, owners)) continue;
      for (std::int64_t s = 0; s < nmid; ++s)
        if (detail::owns_outer(s, rank, world, owners)) {
          lay.send_off[static_cast<std::size_t>(t * nmid + s)] = cur;
          cur += R[static_cast<std::size_t>(t * nmid + s)];
        }
    }
    lay.send_counts[static_cast<std::size_t>(q)] = cur - start;
  }
  cur = 0;
  for (std::int64_t q = 0; q < world; ++q) {
    const std::int64_t start = cur;
    for (std::int64_t t = 0; t < nmid; ++t) {
      if (!detail::owns_outer(t, rank, world, owners)) continue;
      for (std::int64_t s = 0; s < nmid; ++s)
        if (detail::owns_outer(s, q, world, owners)) {
          lay.recv_off[static_cast<std::size_t>(t * nmid + s)] = cur;
          cur += R[static_cast<std::size_t>(t * nmid + s)];
        }
    }
    lay.recv_counts[static_cast<std::size_t>(q)] = cur - start;
  }
  return lay;
}

// Byte-balanced ownership map (sharded.py balanced_owners): longest-processing-
// time bin packing of per-multi-set weights over `world` ranks with at most
// ceil(n / world) multi-sets each; deterministic (ties to the lower index /
// rank); the round-robin map when that is at least as good.
inline std::vector<std::int32_t> balanced_owners(const std::vector<double>& w, std::int64_t world) {
  const std::size_t n = w.size();
  std::vector<std::int32_t> own(n, 0);
  if (world <= 1) return own;
  const std::size_t cap = (n + static_cast<std::size_t>(world) - 1) / static_cast<std::size_t>(world);
  std::vector<std::size_t> order(n);
  for (std::size_t i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) { return w[a] > w[b]; });
  std::vector<double> load(static_cast<std::size_t>(world), 0.0), rr(static_cast<std::size_t>(world), 0.0);
  std::vector<std::size_t> cnt(static_cast<std::size_t>(world), 0);
  for (std::size_t i : order) {
    std::size_t best = n;  // sentinel
    for (std::size_t r = 0; r < static_cast<std::size_t>(world); ++r)
      if (cnt[r] < cap && (best == n || load[r] < load[best])) best = r;
    own[i] = static_cast<std::int32_t>(best);
    load[best] += w[i];
    ++cnt[best];
  }
  for (std::size_t i = 0; i < n; ++i) rr[i % static_cast<std::size_t>(world)] += w[i];
  if (*std::max_element(rr.begin(), rr.end()) <= *std::max_element(load.begin(), load.end()))
    for (std::size_t i = 0; i < n; ++i) own[i] = static_cast<std::int32_t>(i % static_cast<std::size_t>(world));
  return own;
}

class ShardedTensorButterfly {
 public:
  std::int64_t d() const { return eval_.d; }
  std::int64_t world() const { return static_cast<std::int64_t>(devices_.size()); }
  std::int64_t nmid() const { return nmid_; }
  std::int64_t middle_level() const { return Lc_; }
  const std::vector<int>& devices() const { return devices_; }
  const KernelEvaluator& evaluator() const { return eval_; }
  oiobf_tbf* handle(std::size_t rank) const { return h_[rank].get(); }
  const ShardLayout& layout(std::size_t rank) const { return lay_[rank]; }
  const std::vector<std::int64_t>& block_rows() const { return R_; }
  // ownership map of the middle multi-sets (empty: o % world)
  const std::vector<std::int32_t>& owners() const { return owners_; }
  std::int64_t owner_of(std::int64_t outer) const { return detail::owner_of(outer, world(), owners_); }
  // core bytes read by the owner of each s (the weights of balanced_owners)
  std::vector<double> core_bytes_per_s() const {
    std::vector<double> w(static_cast<std::size_t>(nmid_), 0.0);
    std::vector<std::int64_t> cr(static_cast<std::size_t>(nmid_ * nmid_)), cc(cr.size());
    for (std::size_t r = 0; r < h_.size(); ++r) {
      detail::check(oiobf_set_device(devices_[r]));
      detail::check(oiobf_tbf_export(h_[r].get(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                                     cr.data(), cc.data(), nullptr));
      for (std::int64_t s = 0; s < nmid_; ++s)
        if (owner_of(s) == static_cast<std::int64_t>(r))
          for (std::int64_t t = 0; t < nmid_; ++t) {  // pair p = s * nmid + t
            const std::size_t p = static_cast<std::size_t>(s * nmid_ + t);
            w[static_cast<std::size_t>(s)] += 16.0 * static_cast<double>(cr[p]) * static_cast<double>(cc[p]);
          }
    }
    return w;
  }

 private:
  friend ShardedTensorButterfly tbf_construct_sharded(const KernelEvaluator&, std::int64_t, double, const ProxyStrategy&,
                                                      std::uint64_t, const std::vector<int>&,
                                                      const std::vector<std::int32_t>&);
  std::vector<std::int32_t> owners_;
  std::vector<int> devices_;
  KernelEvaluator eval_;
  std::int64_t L_ = 0, Lc_ = 0, nmid_ = 0;
  std::vector<std::shared_ptr<oiobf_tbf>> h_;
  std::vector<std::int64_t> R_;  // rows of G_{t,s}, index t * nmid + s
  std::vector<ShardLayout> lay_;
};

// Alg. 1 over devices.size() GPUs (ranks in the order given).  owners: the
// ownership map of the middle multi-sets (entries in [0, devices.size())), or
// empty for o % world.
inline ShardedTensorButterfly tbf_construct_sharded(const KernelEvaluator& eval, std::int64_t L, double tol,
                                                    const ProxyStrategy& proxies, std::uint64_t seed,
                                                    const std::vector<int>& devices,
                                                    const std::vector<std::int32_t>& owners = {}) {
  require(!devices.empty(), "tbf_construct_sharded: no devices");
  const oiobf_kernel_spec& spec = eval.device_spec();
  oiobf_proxy_strategy ps{};
  ps.mode = static_cast<int32_t>(proxies.mode);
  ps.q = proxies.q;
  ps.max_retries = proxies.max_retries;
  ps.row_cap = proxies.row_cap;
  ShardedTensorButterfly bf;
  bf.devices_ = devices;
  bf.eval_ = eval;
  bf.L_ = L;
  bf.Lc_ = L / 2;
  const auto world = static_cast<std::int64_t>(devices.size());
  bf.h_.resize(devices.size());
  for (std::size_t r = 0; r < devices.size(); ++r) {
    detail::check(oiobf_set_device(devices[r]));
    oiobf_tbf* h = nullptr;
    detail::check(oiobf_tbf_shard_begin(&spec, static_cast<int32_t>(L), tol, &ps, seed, static_cast<int32_t>(r),
                                        static_cast<int32_t>(world), &h));
    bf.h_[r] = std::shared_ptr<oiobf_tbf>(h, &oiobf_tbf_destroy);
    if (!owners.empty()) {
      std::int64_t hi[10];
      detail::check(oiobf_tbf_info(h, hi));
      require(static_cast<std::int64_t>(owners.size()) == hi[4], "tbf_construct_sharded: owners needs nmid entries");
      detail::check(oiobf_tbf_shard_set_owners(h, owners.data()));
    }
  }
  bf.owners_ = owners;
  // levels, r_est level-synchronous across ranks (the max plays the all-reduce)
  std::vector<std::int64_t> local(devices.size());
  for (int side = 0; side < 2; ++side) {
    std::int64_t r_est = 8;
    for (std::int64_t l = 0; l <= bf.Lc_; ++l) {
      detail::for_ranks(devices, [&](std::size_t r) {
        detail::check(oiobf_set_device(devices[r]));
        detail::check(oiobf_tbf_shard_level(bf.h_[r].get(), side, static_cast<int32_t>(l), r_est, &local[r]));
      });
      for (auto v : local) r_est = std::max(r_est, v);
    }
  }
  // U-side middle ranks / skeletons of every t, summed across ranks
  std::int64_t nslots = 0, wpad = 1;
  for (std::size_t r = 0; r < devices.size(); ++r) {
    std::int64_t info[2];
    detail::check(oiobf_tbf_umid_info(bf.h_[r].get(), info));
    nslots = info[0];
    wpad = std::max(wpad, info[1]);
  }
  std::vector<std::int64_t> ranks_all(static_cast<std::size_t>(nslots), 0);
  std::vector<std::int32_t> skel_all(static_cast<std::size_t>(nslots * wpad), 0);
  for (std::size_t r = 0; r < devices.size(); ++r) {
    std::vector<std::int64_t> rk(static_cast<std::size_t>(nslots));
    std::vector<std::int32_t> sk(static_cast<std::size_t>(nslots * wpad));
    detail::check(oiobf_set_device(devices[r]));
    detail::check(oiobf_tbf_umid_export(bf.h_[r].get(), rk.data(), sk.data(), wpad));
    for (std::size_t i = 0; i < rk.size(); ++i) ranks_all[i] += rk[i];
    for (std::size_t i = 0; i < sk.size(); ++i) skel_all[i] += sk[i];
  }
  detail::for_ranks(devices, [&](std::size_t r) {
    detail::check(oiobf_set_device(devices[r]));
    detail::check(oiobf_tbf_umid_import(bf.h_[r].get(), ranks_all.data(), skel_all.data(), wpad));
  });
  // block rows R[t, s] = prod_k U-side middle rank (Lc, t, nu = s, k)
  const std::int64_t d = eval.d;
  std::int64_t info[10];
  detail::check(oiobf_tbf_info(bf.h_[0].get(), info));
  const std::int64_t nm = info[4];
  require(nslots == nm * nm * d, "tbf_construct_sharded: unexpected middle-level slot count");
  bf.nmid_ = nm;
  bf.R_.assign(static_cast<std::size_t>(nm * nm), 1);
  for (std::int64_t p = 0; p < nm * nm; ++p)
    for (std::int64_t k = 0; k < d; ++k) bf.R_[static_cast<std::size_t>(p)] *= ranks_all[static_cast<std::size_t>(p * d + k)];
  for (std::size_t r = 0; r < devices.size(); ++r) {
    bf.lay_.push_back(shard_layout(bf.R_, nm, static_cast<std::int64_t>(r), world, owners));
    const ShardLayout& lay = bf.lay_.back();
    detail::check(oiobf_tbf_set_exchange(bf.h_[r].get(), lay.send_off.data(), lay.recv_off.data(), lay.send_total(),
                                         lay.recv_total()));
  }
  return bf;
}

// Byte-balanced sharded construction: a first construction with the default
// map measures the core bytes of every s, a second one uses the LPT map of
// those bytes (construction is deterministic and independent of the
// ownership, so both build identical factors; the second costs one more
// construction and pays off over repeated applies -- the core stage is
// HBM-bound, config 3 at world 8: heaviest rank 1.61x -> 1.00x the mean).
inline ShardedTensorButterfly tbf_construct_sharded_balanced(const KernelEvaluator& eval, std::int64_t L, double tol,
                                                             const ProxyStrategy& proxies, std::uint64_t seed,
                                                             const std::vector<int>& devices) {
  std::vector<std::int32_t> owners;
  {
    const ShardedTensorButterfly first = tbf_construct_sharded(eval, L, tol, proxies, seed, devices);
    owners = balanced_owners(first.core_bytes_per_s(), first.world());
  }
  return tbf_construct_sharded(eval, L, tol, proxies, seed, devices, owners);
}

// Alg. 2 over the ranks: G = K x F, F of shape (n_1..n_d[, n_v]).
inline DenseTensor tbf_contract(const ShardedTensorButterfly& bf, const DenseTensor& F) {
  const std::int64_t d = bf.d();
  require(F.mode_count() == d || F.mode_count() == d + 1, "tbf_contract: input must have d or d+1 modes");
  for (std::int64_t k = 0; k < d; ++k)
    require(F.extent(k + 1) == bf.evaluator().col_extents[static_cast<std::size_t>(k)], "tbf_contract: shape mismatch");
  const std::int64_t nv = F.mode_count() == d + 1 ? F.extent(d + 1) : 1;
  const auto& dev = bf.devices();
  const std::int64_t world = bf.world();
  const std::int64_t bytes = F.size() * 16;
  std::vector<std::unique_ptr<detail::DeviceBuffer>> dF(dev.size()), dG(dev.size()), send(dev.size()),
      recv(dev.size());
  for (std::size_t r = 0; r < dev.size(); ++r) {
    dF[r] = std::make_unique<detail::DeviceBuffer>(dev[r], bytes);
    dG[r] = std::make_unique<detail::DeviceBuffer>(dev[r], bytes);
    send[r] = std::make_unique<detail::DeviceBuffer>(dev[r], 16 * bf.layout(r).send_total() * nv);
    recv[r] = std::make_unique<detail::DeviceBuffer>(dev[r], 16 * bf.layout(r).recv_total() * nv);
  }
  // phase 1 on every rank: V/W levels + core GEMV of the owned s
  detail::for_ranks(dev, [&](std::size_t r) {
    detail::check(oiobf_set_device(dev[r]));
    detail::check(oiobf_memcpy(dF[r]->p, F.data().data(), bytes));
    detail::check(oiobf_tbf_contract_phase(bf.handle(r), 1, dF[r]->p, send[r]->p, nv, nullptr));
    detail::check(oiobf_synchronize());
  });
  // exchange: sender r's segment for destination q -> receiver q's segment from source r
  for (std::int64_t q = 0; q < world; ++q) {
    std::int64_t roff = 0;
    for (std::int64_t r = 0; r < world; ++r) {
      const ShardLayout& ls = bf.layout(static_cast<std::size_t>(r));
      std::int64_t soff = 0;
      for (std::int64_t x = 0; x < q; ++x) soff += ls.send_counts[static_cast<std::size_t>(x)];
      const std::int64_t n = ls.send_counts[static_cast<std::size_t>(q)] * nv;
      if (n > 0) {
        detail::check(oiobf_set_device(dev[static_cast<std::size_t>(q)]));
        detail::check(oiobf_memcpy(static_cast<char*>(recv[static_cast<std::size_t>(q)]->p) + 16 * roff,
                                   static_cast<const char*>(send[static_cast<std::size_t>(r)]->p) + 16 * soff * nv,
                                   16 * n));
      }
      roff += n;
    }
  }
  // phase 2 on every rank: P/U levels of the owned t, then its row slabs to the host
  DenseTensor G(F.shape());
  std::vector<std::vector<Complex>> Gr(dev.size());
  detail::for_ranks(dev, [&](std::size_t r) {
    detail::check(oiobf_set_device(dev[r]));
    detail::check(oiobf_tbf_contract_phase(bf.handle(r), 2, recv[r]->p, dG[r]->p, nv, nullptr));
    detail::check(oiobf_synchronize());
    Gr[r].resize(static_cast<std::size_t>(F.size()));
    detail::check(oiobf_memcpy(Gr[r].data(), dG[r]->p, bytes));
  });
  // assemble: output slab t (middle multi-set, mixed radix, mode 0 fastest) from its owner
  const std::int64_t nmid = bf.nmid();
  const std::int64_t mpm = std::int64_t(1) << bf.middle_level();  // middle nodes per mode
  const std::int64_t n = bf.evaluator().row_extents[0];
  const std::int64_t mid = n / mpm;
  const std::int64_t N = F.size() / nv;
  for (std::int64_t t = 0; t < nmid; ++t) {
    const auto& src = Gr[static_cast<std::size_t>(bf.owner_of(t))];
    std::int64_t base = 0, st = 1, rem = t;
    for (std::int64_t k = 0; k < d; ++k) {
      base += (rem % mpm) * mid * st;
      rem /= mpm;
      st *= n;
    }
    // every element of the slab: indices (i_0..i_{d-1}) in [0, mid)^d, and v
    const std::int64_t cnt = [&] {
      std::int64_t c = 1;
      for (std::int64_t k = 0; k < d; ++k) c *= mid;
      return c;
    }();
    for (std::int64_t v = 0; v < nv; ++v)
      for (std::int64_t e = 0; e < cnt; ++e) {
        std::int64_t off = base + v * N, r2 = e, s2 = 1;
        for (std::int64_t k = 0; k < d; ++k) {
          off += (r2 % mid) * s2;
          r2 /= mid;
          s2 *= n;
        }
        G.data()[static_cast<std::size_t>(off)] = src[static_cast<std::size_t>(off)];
      }
  }
  return G;
}

}  // namespace oiobf

#endif
