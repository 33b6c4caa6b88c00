// Host runtime + C ABI of the B200 tensor-butterfly library.
//
// Construction (Alg. 1 / SPEC.md:268-276): for each side (V/W then
// U/P) and level l = 0..Lc, one batch of IDs on the device (proxy lists,
// candidate columns, fused entry generation + TSQR, reference pivoting), then
// the ranks come back to the host to size the next level (the only host sync
// per level).  r_est is level-synchronous: r_est(l) =
// max(8, max rank over levels < l of the same side).  Cores are generated on
// the device at the end.
//
// Apply (Alg. 2 / SPEC.md:277-285): a static plan of batched kernel
// launches (one per level and mode, plus the core GEMV and the ordered child
// sums), captured once into a CUDA graph and replayed.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "kernels.h"

namespace tbf {
int gemv_rows_per_cta();
void launch_subtensor(const KSpec& ks, const i64* counts_h, const int* lists, i64 total, double2* out,
                      cudaStream_t st);
void launch_matrix_ids(i64 njobs, const i64* a_off, const i64* m, const int* n, const double2* A, i64 nparts, i64 rpp,
                       int pr, i64 wmax, double2* rpart, cudaStream_t st);
void launch_finish_var(const LevelDesc& L, const i64* mrows, double tol, double tie_eps, const i64* max_rank,
                       const double2* rpart, const int* targets, const int* width, int* rank, int* sat, int* perm,
                       int* skel_tmp, double2* interp_tmp, double* gaps, cudaStream_t st);
}  // namespace tbf

namespace {

using namespace tbf;

thread_local std::string g_err;
thread_local int g_device = 0;

struct InvalidArg : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void require(bool c, const std::string& msg) {
  if (!c) throw InvalidArg(msg);
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      reset();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { reset(); }
  void alloc(size_t count) {
    reset();
    n = count;
    if (count) TBF_CUDA(cudaMalloc(&p, sizeof(T) * count));
  }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void upload(const T* h, size_t count, cudaStream_t st) {
    if (count) TBF_CUDA(cudaMemcpyAsync(p, h, sizeof(T) * count, cudaMemcpyHostToDevice, st));
  }
  void download(T* h, size_t count, cudaStream_t st) const {
    if (count) TBF_CUDA(cudaMemcpyAsync(h, p, sizeof(T) * count, cudaMemcpyDeviceToHost, st));
  }
};

template <class T>
DevBuf<T> to_device(const std::vector<T>& v, cudaStream_t st) {
  DevBuf<T> b(v.size());
  b.upload(v.data(), v.size(), st);
  return b;
}

i64 ipow(i64 b, i64 e) {
  i64 r = 1;
  while (e-- > 0) r *= b;
  return r;
}

void ensure_device() {
  int cnt = 0;
  cudaError_t e = cudaGetDeviceCount(&cnt);
  if (e != cudaSuccess || cnt == 0)
    throw std::runtime_error("no CUDA device available (the B200 path has no CPU fallback)");
  TBF_CUDA(cudaSetDevice(g_device));
  cudaDeviceProp pr;
  TBF_CUDA(cudaGetDeviceProperties(&pr, g_device));
  if (pr.major < 10) throw std::runtime_error("device is not sm_100-class (Blackwell) — this build targets sm_100a");
}

struct EventTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t st;
  explicit EventTimer(cudaStream_t s) : st(s) {
    TBF_CUDA(cudaEventCreate(&a));
    TBF_CUDA(cudaEventCreate(&b));
    TBF_CUDA(cudaEventRecord(a, st));
  }
  double stop() {
    TBF_CUDA(cudaEventRecord(b, st));
    TBF_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    TBF_CUDA(cudaEventElapsedTime(&ms, a, b));
    return ms;
  }
  ~EventTimer() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
};

struct LevelData {
  LevelDesc L{};
  i64 nslots = 0;
  DevBuf<int> rank, width, perm, skel;
  DevBuf<double2> interp;
  DevBuf<i64> skel_off, interp_off;
  DevBuf<double> gaps;
  std::vector<int> h_rank, h_width, h_sat;
  std::vector<i64> h_skel_off, h_interp_off;
  i64 total_skel = 0, total_interp = 0;
  int max_rank = 0;
};

struct TRef {
  i64 off = 0;
  int nd = 0;
  int ext[kMaxTM] = {0};
  i64 stride[kMaxTM] = {0};
  i64 size() const {
    i64 s = 1;
    for (int p = 0; p < nd; ++p) s *= ext[p];
    return s;
  }
};

TRef packed(i64 off, int nd, const int* ext) {
  TRef t;
  t.off = off;
  t.nd = nd;
  i64 st = 1;
  for (int p = 0; p < nd; ++p) {
    t.ext[p] = ext[p];
    t.stride[p] = st;
    st *= ext[p];
  }
  return t;
}

enum BufId { BUF_F = 0, BUF_G = 1, BUF_SCRATCH = 2, BUF_SEND = 3, BUF_RECV = 4 };

struct MPLaunch {
  int side, level;  // factor arena
  int in_buf, out_buf;
  i64 step_begin, nsteps, total_out;
};
struct SumLaunch {
  i64 begin, n, total;  // total: CTAs for k_sum_parent launches
  i64 work_begin = 0;   // first (parent, chunk) pair in the CTA map
};
struct BoxLaunch {
  int side, level, in_buf, out_buf;
  i64 item_begin, nitems;
  BoxLaunchInfo info;
};
struct Op {
  int kind;  // 0 mode product, 1 gemv, 2 sum, 3 fused boxes
  i64 idx;
  int group;  // 0 V/W, 1 core, 2 P/U
};

struct Plan {
  i64 nv = 0;
  i64 scratch_elems = 0;
  std::vector<MPStep> steps;
  std::vector<Blk> blks;
  std::vector<MPLaunch> mps;
  std::vector<GemvDesc> gemv;
  i64 gemv_ctas = 0;
  i64 gemv_total_rows = 0, gemv_rows_per_cta = 1;
  bool gemv_tma = false;
  i64 tma_ctas = 0, tma_rows_per_cta = 1;
  int tma_stages = 0, tma_stage_elems = 0, tma_xcap = 0;
  std::vector<int> tma_map;
  DevBuf<int> d_tma_map;
  int gemv_max_c = 0;
  std::vector<SumDesc> sums;
  std::vector<SumLaunch> sum_launches;
  std::vector<Op> ops;
  std::vector<BoxItem> bitems;
  std::vector<BoxTerm> bterms;
  std::vector<BoxLaunch> boxes;
  DevBuf<BoxItem> d_bitems;
  DevBuf<BoxTerm> d_bterms;
  DevBuf<MPStep> d_steps;
  DevBuf<Blk> d_blks;
  DevBuf<GemvDesc> d_gemv;
  DevBuf<int> d_gemv_map;  // CTA -> pair
  std::vector<int> sum_map;
  DevBuf<int> d_sum_map;   // k_sum_parent CTA -> (parent, chunk)
  DevBuf<SumDesc> d_sums;
  DevBuf<double2> scratch;
  DevBuf<double2> stage_F, stage_G;  // host-buffer contract staging
  i64 gemv_y_base = 0;
  // sharded plans (world > 1): phase 1 = V/W + GEMV (writes the send buffer),
  // phase 2 = P/U (reads the receive buffer)
  bool sharded = false;
  // graph cache
  cudaGraphExec_t gexec = nullptr;
  const void* g_F = nullptr;
  void* g_G = nullptr;
  cudaStream_t g_st = nullptr;
  ~Plan() {
    if (gexec) cudaGraphExecDestroy(gexec);
  }
};

}  // namespace

struct oiobf_tbf {
  oiobf_kernel_spec spec{};
  KSpec ks{};
  int d = 0, L = 0, Lc = 0;
  i64 n = 0, nmid = 0;
  double tol = 0;
  oiobf_proxy_strategy strat{};
  u64 seed = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  // sharding: this rank owns middle multi-sets with
  // index % world == rank on both sides
  int rank = 0, world = 1;
  bool owns(i64 outer) const { return world <= 1 || outer % world == rank; }
  // U-side middle-level (l = Lc) ranks / skeletons of ALL t (gathered from the
  // other ranks) -- the row skeletons of the cores of the owned pairs (t, s)
  std::vector<int> umid_rank;
  std::vector<i64> umid_skel_off;
  DevBuf<int> umid_skel;
  // exchange tables (element offsets per pair t*nmid+s, nv = 1 units), -1 = none
  std::vector<i64> send_off, recv_off;
  i64 send_elems = 0, recv_elems = 0;
  std::vector<LevelData> side[2];
  std::vector<i64> r_est[2];
  DevBuf<double2> cores;
  std::vector<PairDesc> h_pairs;
  i64 total_core = 0;
  std::map<i64, std::unique_ptr<Plan>> plans;
  double t_ms[6] = {0, 0, 0, 0, 0, 0};
  std::mutex mu;
  ~oiobf_tbf() {
    plans.clear();
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

constexpr double kTieEps = 1e-12;

LevelDesc make_level(const oiobf_tbf& b, int sd, int l, i64 r_est, i64 wmax) {
  LevelDesc L{};
  L.d = b.d;
  L.side = sd;
  L.l = l;
  L.L = b.L;
  L.Lc = b.Lc;
  L.proxy_mode = b.strat.mode;
  L.n = b.n;
  L.nin = ipow(2, static_cast<i64>(b.d) * l);
  L.nj = ipow(2, b.Lc - l);
  L.mpm = ipow(2, b.Lc);
  L.nslots = b.nmid * L.nin * b.d * L.nj;
  L.per_mode = b.strat.q * r_est;  // attempt 0 (id.cpp:257)
  L.seed = b.seed;
  L.side_tag = sd == 0 ? 0x56ULL : 0x55ULL;
  L.wmax = wmax;
  L.c_nin = l > 0 ? ipow(2, static_cast<i64>(b.d) * (l - 1)) : 0;
  L.c_nj = l > 0 ? ipow(2, b.Lc - l + 1) : 0;
  const int D = 2 * b.d;
  const int mid_off = sd == 0 ? b.d : 0, in_off = sd == 0 ? 0 : b.d;
  L.psize = 0;
  i64 m = -1;
  for (int k = 0; k < b.d; ++k) {
    i64 sizes[kMaxModes], counts[kMaxModes];
    for (int p = 0; p < b.d; ++p) {
      sizes[mid_off + p] = b.n >> b.Lc;
      sizes[in_off + p] = b.n >> l;
    }
    const int skip = mid_off + k;
    sizes[skip] = b.n >> (b.L - l);
    proxy_counts(D, sizes, skip, L.per_mode, b.strat.mode, b.strat.row_cap, counts);
    i64 tot = 0, rows = 1;
    for (int p = 0; p < D; ++p) {
      require(counts[p] <= kMaxProxy || b.strat.mode != OIOBF_PROXY_UNIFORM_RANDOM,
              "proxy count per mode exceeds the device limit (64)");
      L.counts[k][p] = static_cast<int>(counts[p]);
      L.poff[k][p] = static_cast<int>(tot);
      tot += counts[p];
      if (p != skip) rows *= counts[p];
    }
    L.psize = std::max(L.psize, tot);
    if (m >= 0 && m != rows) throw std::runtime_error("internal: non-uniform proxy row count");
    m = rows;
  }
  L.m = m;
  L.pr = wmax <= 16 ? 256 : wmax <= 32 ? 128 : wmax <= 64 ? 64 : 32;
  L.rank = b.rank;
  L.world = b.world;
  const i64 target_ctas = 148 * 8;
  const i64 owned = (L.nslots + b.world - 1) / b.world;
  i64 parts = (target_ctas + owned - 1) / owned;
  const i64 max_parts = std::max<i64>(1, (L.m + 4 * L.pr - 1) / (4 * L.pr));  // >= 4 panels per part
  parts = std::max<i64>(1, std::min(parts, max_parts));
  L.nparts = parts;
  L.rpp = (L.m + parts - 1) / parts;
  return L;
}

void build_side_level(oiobf_tbf& b, int sd, int l, i64 r_est) {
  cudaStream_t st = b.stream;
  const int d = b.d;
  // widest candidate set: leaf size (l=0) or max r(child0)+r(child1)
  i64 wmax;
  if (l == 0) {
    wmax = b.n >> b.L;
  } else {
    const LevelData& c = b.side[sd][static_cast<size_t>(l - 1)];
    LevelDesc tmp = make_level(b, sd, l, r_est, 1);
    wmax = 0;
    for (i64 idx = 0; idx < tmp.nslots; ++idx) {
      const SlotPos s = decode_slot(tmp, idx);
      const i64 w = c.h_rank[static_cast<size_t>(child_slot(tmp, s, 0))] +
                    c.h_rank[static_cast<size_t>(child_slot(tmp, s, 1))];
      wmax = std::max(wmax, w);
    }
  }
  wmax = std::max<i64>(wmax, 1);
  require(wmax <= kMaxW, "ID width " + std::to_string(wmax) + " exceeds the supported maximum " +
                             std::to_string(kMaxW));
  LevelData& ld = b.side[sd][static_cast<size_t>(l)];
  ld.L = make_level(b, sd, l, r_est, wmax);
  LevelDesc& L = ld.L;
  ld.nslots = L.nslots;
  const i64 ns = L.nslots;
  (void)d;
  DevBuf<int> proxies(static_cast<size_t>(ns * L.psize));
  DevBuf<int> targets(static_cast<size_t>(ns * wmax));
  ld.width.alloc(static_cast<size_t>(ns));
  EventTimer t0(st);
  launch_gen_proxies(L, proxies.p, st);
  if (l == 0) {
    launch_targets(L, nullptr, nullptr, nullptr, targets.p, ld.width.p, st);
  } else {
    const LevelData& c = b.side[sd][static_cast<size_t>(l - 1)];
    launch_targets(L, c.rank.p, c.skel_off.p, c.skel.p, targets.p, ld.width.p, st);
  }
  b.t_ms[0] += t0.stop();
  DevBuf<double2> rpart(static_cast<size_t>(ns * L.nparts * wmax * wmax));
  EventTimer t1(st);
  launch_panel(L, b.ks, proxies.p, targets.p, ld.width.p, rpart.p, st);
  b.t_ms[1] += t1.stop();
  ld.rank.alloc(static_cast<size_t>(ns));
  DevBuf<int> sat(static_cast<size_t>(ns));
  ld.perm.alloc(static_cast<size_t>(ns * wmax));
  ld.gaps.alloc(static_cast<size_t>(ns));
  DevBuf<int> skel_tmp(static_cast<size_t>(ns * wmax));
  DevBuf<double2> interp_tmp(static_cast<size_t>(ns * wmax * wmax));
  EventTimer t2(st);
  launch_finish(L, b.tol, kTieEps, -1, rpart.p, targets.p, ld.width.p, ld.rank.p, sat.p, ld.perm.p, skel_tmp.p,
                interp_tmp.p, ld.gaps.p, st);
  b.t_ms[2] += t2.stop();
  ld.h_rank.resize(static_cast<size_t>(ns));
  ld.h_width.resize(static_cast<size_t>(ns));
  ld.h_sat.resize(static_cast<size_t>(ns));
  ld.rank.download(ld.h_rank.data(), static_cast<size_t>(ns), st);
  ld.width.download(ld.h_width.data(), static_cast<size_t>(ns), st);
  sat.download(ld.h_sat.data(), static_cast<size_t>(ns), st);
  TBF_CUDA(cudaStreamSynchronize(st));
  ld.h_skel_off.resize(static_cast<size_t>(ns));
  ld.h_interp_off.resize(static_cast<size_t>(ns));
  i64 so = 0, io = 0;
  ld.max_rank = 0;
  for (i64 i = 0; i < ns; ++i) {
    ld.h_skel_off[static_cast<size_t>(i)] = so;
    ld.h_interp_off[static_cast<size_t>(i)] = io;
    so += ld.h_rank[static_cast<size_t>(i)];
    io += static_cast<i64>(ld.h_rank[static_cast<size_t>(i)]) * ld.h_width[static_cast<size_t>(i)];
    ld.max_rank = std::max(ld.max_rank, ld.h_rank[static_cast<size_t>(i)]);
  }
  ld.total_skel = so;
  ld.total_interp = io;
  EventTimer t3(st);
  ld.skel_off = to_device(ld.h_skel_off, st);
  ld.interp_off = to_device(ld.h_interp_off, st);
  ld.skel.alloc(static_cast<size_t>(std::max<i64>(so, 1)));
  ld.interp.alloc(static_cast<size_t>(std::max<i64>(io, 1)));
  launch_compact(ns, wmax, ld.rank.p, ld.width.p, ld.skel_off.p, ld.interp_off.p, skel_tmp.p, interp_tmp.p, ld.skel.p,
                 ld.interp.p, st);
  b.t_ms[3] += t3.stop();
  // saturation would trigger the doubling retry (id.cpp:256-269); with the
  // default rank limit it is unreachable, so it is only reported.
}

// Cores K(tbar, sbar) of the pairs (t, s) whose s this rank owns (all pairs
// when world == 1).  Row skeletons come from the U side at level Lc -- local
// when world == 1, gathered from every rank (umid_*) otherwise.
void build_cores(oiobf_tbf& b) {
  cudaStream_t st = b.stream;
  const int d = b.d;
  const LevelData& U = b.side[1][static_cast<size_t>(b.Lc)];
  const LevelData& V = b.side[0][static_cast<size_t>(b.Lc)];
  const bool gathered = b.world > 1;
  const int* urank = gathered ? b.umid_rank.data() : U.h_rank.data();
  const i64* uskel_off = gathered ? b.umid_skel_off.data() : U.h_skel_off.data();
  const int* uskel = gathered ? b.umid_skel.p : U.skel.p;
  const i64 P = b.nmid * b.nmid;
  b.h_pairs.assign(static_cast<size_t>(P), PairDesc{});
  i64 off = 0;
  for (i64 p = 0; p < P; ++p) {
    const i64 s = p / b.nmid, t = p % b.nmid;
    PairDesc& pd = b.h_pairs[static_cast<size_t>(p)];
    pd.R = 1;
    pd.C = 1;
    for (int k = 0; k < d; ++k) {
      const i64 us = (t * b.nmid + s) * d + k;  // U slot (Lc, t, nu=s, k, j=0)
      const i64 vs = (s * b.nmid + t) * d + k;  // V slot (Lc, s, tau=t, k, j=0)
      pd.rr[k] = urank[us];
      pd.rc[k] = V.h_rank[static_cast<size_t>(vs)];
      pd.rs_off[k] = uskel_off[us];
      pd.cs_off[k] = V.h_skel_off[static_cast<size_t>(vs)];
      pd.R *= pd.rr[k];
      pd.C *= pd.rc[k];
    }
    if (!b.owns(s)) pd.C = 0;  // another rank generates and applies this core
    pd.core_off = off;
    pd.work_off = off;
    off += static_cast<i64>(pd.R) * pd.C;
  }
  b.total_core = off;
  b.cores.alloc(static_cast<size_t>(std::max<i64>(off, 1)));
  DevBuf<PairDesc> dp = to_device(b.h_pairs, st);
  EventTimer t(st);
  launch_cores(b.ks, P, dp.p, off, uskel, V.skel.p, b.cores.p, st);
  b.t_ms[4] += t.stop();
}

void validate_spec(const oiobf_kernel_spec& s) {
  require(s.d >= 1 && s.d <= kMaxD, "kernel spec: d must be in [1,6]");
  require(s.n >= 1, "kernel spec: n must be positive");
  require(s.kind >= 0 && s.kind <= 2, "make_kernel: unknown kernel kind");
  require(s.kind != OIOBF_KERNEL_RADON2D || s.d == 2, "kernel spec: radon2d needs d=2");
  require(s.kind != OIOBF_KERNEL_GREEN || s.d <= 3, "kernel spec: green needs d<=3");
  if (s.bitrev) require((s.n & (s.n - 1)) == 0, "reorder_bit_reversal: extent must be a power of two");
}

std::unique_ptr<oiobf_tbf> construct_begin(const oiobf_kernel_spec& spec, int L, double tol,
                                           const oiobf_proxy_strategy& ps, u64 seed, int rank, int world) {
  validate_spec(spec);
  require(L >= 0 && L % 2 == 0, "tbf_construct: L must be even and >= 0");
  require((spec.n >> L) >= 1 && spec.n % (i64{1} << L) == 0, "tbf_construct: extent must equal C_b * 2^L");
  require(tol > 0 && tol < 1, "column_id: tolerance must be in (0,1)");
  require(ps.q >= 1 && ps.row_cap >= 1, "ProxyStrategy: q and row_cap must be positive");
  require(ps.mode >= 0 && ps.mode <= 2, "ProxyStrategy: unknown mode");
  require(world >= 1 && rank >= 0 && rank < world, "tbf_construct: bad rank / world");
  ensure_device();
  auto b = std::make_unique<oiobf_tbf>();
  b->spec = spec;
  b->ks = kspec_from(spec);
  b->d = spec.d;
  b->L = L;
  b->Lc = L / 2;
  b->n = spec.n;
  b->nmid = ipow(2, static_cast<i64>(spec.d) * b->Lc);
  b->tol = tol;
  b->strat = ps;
  b->seed = seed;
  b->device = g_device;
  b->rank = rank;
  b->world = world;
  for (int sd = 0; sd < 2; ++sd) b->side[sd].resize(static_cast<size_t>(b->Lc + 1));
  TBF_CUDA(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking));
  return b;
}

oiobf_tbf* construct(const oiobf_kernel_spec& spec, int L, double tol, const oiobf_proxy_strategy& ps, u64 seed) {
  auto b = construct_begin(spec, L, tol, ps, seed, 0, 1);
  auto t_start = std::chrono::steady_clock::now();
  for (int sd = 0; sd < 2; ++sd) {
    i64 r_est = 8;
    for (int l = 0; l <= b->Lc; ++l) {
      b->r_est[sd].push_back(r_est);
      build_side_level(*b, sd, l, r_est);
      r_est = std::max<i64>(r_est, b->side[sd][static_cast<size_t>(l)].max_rank);
    }
  }
  build_cores(*b);
  TBF_CUDA(cudaStreamSynchronize(b->stream));
  b->t_ms[5] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  return b.release();
}

// ------------------------------------------------------------------ apply plan
void add_mp(Plan& pl, int side, int level, int in_buf, int out_buf, const std::vector<MPStep>& items,
            const std::vector<std::vector<Blk>>& blocks, int group) {
  MPLaunch m;
  m.side = side;
  m.level = level;
  m.in_buf = in_buf;
  m.out_buf = out_buf;
  m.step_begin = static_cast<i64>(pl.steps.size());
  m.nsteps = static_cast<i64>(items.size());
  i64 work = 0;
  for (size_t i = 0; i < items.size(); ++i) {
    MPStep s = items[i];
    s.work_off = work;
    work += s.total;
    s.blk_off = static_cast<i64>(pl.blks.size());
    s.nblk = static_cast<int>(blocks[i].size());
    pl.blks.insert(pl.blks.end(), blocks[i].begin(), blocks[i].end());
    pl.steps.push_back(s);
  }
  m.total_out = work;
  pl.ops.push_back(Op{0, static_cast<i64>(pl.mps.size()), group});
  pl.mps.push_back(m);
}

MPStep make_step(const TRef& in, const TRef& out, int mode, int transpose) {
  MPStep s{};
  s.in_off = in.off;
  s.out_off = out.off;
  s.nd = out.nd;
  s.mode = mode;
  s.transpose = transpose;
  s.total = out.size();
  for (int p = 0; p < out.nd; ++p) {
    s.ext[p] = out.ext[p];
    s.in_stride[p] = in.stride[p];
    s.out_stride[p] = out.stride[p];
  }
  return s;
}

std::unique_ptr<Plan> build_plan(oiobf_tbf& b, i64 nv) {
  auto pl = std::make_unique<Plan>();
  pl->nv = nv;
  const int d = b.d;
  const int nd = d + 1;
  const i64 n = b.n;
  const i64 N = ipow(n, d);
  const i64 mid = n >> b.Lc;
  const i64 mpm = ipow(2, b.Lc);
  i64 scratch = 0;
  auto alloc = [&](int ndims, const int* ext) {
    TRef t = packed(scratch, ndims, ext);
    scratch += t.size();
    return t;
  };
  auto global_slab = [&](i64 outer) {  // F(s) or G(t) view in the global tensor
    TRef t;
    t.nd = nd;
    i64 off = 0, st = 1;
    for (int p = 0; p < d; ++p) {
      const i64 pos = (outer / ipow(mpm, p)) % mpm;
      off += pos * mid * st;
      t.ext[p] = static_cast<int>(mid);
      t.stride[p] = st;
      st *= n;
    }
    t.ext[d] = static_cast<int>(nv);
    t.stride[d] = N;
    t.off = off;
    return t;
  };
  // Per-level slot accessors
  auto slot_info = [&](int sd, int l, i64 outer, i64 inner, int k, i64 j, int& r, int& w, i64& moff) {
    const LevelData& ld = b.side[sd][static_cast<size_t>(l)];
    const i64 slot = ((outer * ld.L.nin + inner) * d + k) * ld.L.nj + j;
    r = ld.h_rank[static_cast<size_t>(slot)];
    w = ld.h_width[static_cast<size_t>(slot)];
    moff = ld.h_interp_off[static_cast<size_t>(slot)];
  };
  auto parent_of = [&](i64 inner, int l) {
    i64 pi = 0;
    for (int p = d - 1; p >= 0; --p) pi = (pi << (l - 1)) | (((inner >> (l * p)) & ((i64{1} << l) - 1)) >> 1);
    return pi;
  };
  // Finish a batch of single-term box items: size shared memory (input box +
  // factors + two intermediates) and record a box launch, or report "too big".
  auto commit_boxes = [&](std::vector<BoxItem>& items, std::vector<std::vector<BoxTerm>>& terms, int sd, int l,
                          int in_buf, int out_buf, int transpose, int group) -> bool {
    // cluster size: split each box's last input mode over cs CTAs (DSMEM
    // reduction) so small levels still occupy every SM
    static const int cs_env = std::getenv("OIOBF_BOX_CLUSTER") ? std::atoi(std::getenv("OIOBF_BOX_CLUSTER")) : 0;
    int cs = cs_env > 0 ? cs_env
                        : static_cast<int>(std::min<i64>(8, std::max<i64>(1, (2 * 148 + static_cast<i64>(items.size()) - 1) /
                                                                                  std::max<i64>(1, items.size()))));
    cs = std::max(1, std::min(cs, 8));
    i64 max_in = 1, max_ab = 1, max_mat = 1, max_out = 1;
    for (size_t i = 0; i < items.size(); ++i) {
      if (terms[i].size() != 1) throw std::runtime_error("internal: box items carry exactly one term");
      const BoxTerm& t = terms[i][0];
      i64 e[kMaxTM];
      i64 isz = nv, msz = 0, osz = nv;  // input slab with padded leading dimension
      for (int p = 0; p < d; ++p) {
        e[p] = p == d - 1 ? (t.in_ext[p] + cs - 1) / cs : t.in_ext[p];
        isz *= (p == 0 ? e[p] + 1 : e[p]);
        osz *= transpose ? t.mcols[p] : t.mrows[p];
      }
      max_out = std::max(max_out, osz);
      max_in = std::max(max_in, isz);
      for (int k = 0; k < d; ++k) msz += static_cast<i64>(t.mrows[k]) * t.mcols[k];
      max_mat = std::max(max_mat, msz);
      for (int k = 0; k < d - 1; ++k) {
        e[k] = transpose ? t.mcols[k] : t.mrows[k];
        i64 cur = nv;
        for (int p = 0; p < d; ++p) cur *= e[p];
        max_ab = std::max(max_ab, cur);
      }
    }
    if (cs == 1) max_out = 0;
    if (max_in + max_mat + 2 * max_ab + max_out > 14000) return false;  // > ~219 KB of shared memory
    // single wave: shrink the cluster until every cluster is co-resident
    while (cs_env <= 0 && cs > 1) {
      BoxLaunchInfo probe{};
      probe.smem_elems_in = static_cast<int>(max_in);
      probe.smem_elems_mat = static_cast<int>(max_mat);
      probe.smem_elems_a = probe.smem_elems_b = static_cast<int>(max_ab);
      probe.smem_elems_acc = static_cast<int>(max_out);
      if (box_max_active_clusters(cs, box_smem_bytes(probe)) >= static_cast<int>(items.size())) break;
      --cs;
      // recompute the slab-dependent sizes for the smaller cluster
      max_in = max_ab = 1;
      for (size_t i = 0; i < items.size(); ++i) {
        const BoxTerm& t = terms[i][0];
        i64 e[kMaxTM];
        i64 isz = nv;
        for (int p = 0; p < d; ++p) {
          e[p] = p == d - 1 ? (t.in_ext[p] + cs - 1) / cs : t.in_ext[p];
          isz *= (p == 0 ? e[p] + 1 : e[p]);
        }
        max_in = std::max(max_in, isz);
        for (int k = 0; k < d - 1; ++k) {
          e[k] = transpose ? t.mcols[k] : t.mrows[k];
          i64 cur = nv;
          for (int p = 0; p < d; ++p) cur *= e[p];
          max_ab = std::max(max_ab, cur);
        }
      }
      if (cs == 1) max_out = 0;
    }
    BoxLaunch bl;
    bl.side = sd;
    bl.level = l;
    bl.in_buf = in_buf;
    bl.out_buf = out_buf;
    bl.item_begin = static_cast<i64>(pl->bitems.size());
    bl.nitems = static_cast<i64>(items.size());
    bl.info.d = d;
    bl.info.nv = static_cast<int>(nv);
    bl.info.transpose = transpose;
    bl.info.smem_elems_in = static_cast<int>(max_in);
    bl.info.smem_elems_mat = static_cast<int>(max_mat);
    bl.info.smem_elems_a = static_cast<int>(max_ab);
    bl.info.smem_elems_b = static_cast<int>(max_ab);
    bl.info.cs = cs;
    bl.info.smem_elems_acc = static_cast<int>(max_out);
    for (size_t i = 0; i < items.size(); ++i) {
      BoxItem x = items[i];
      x.term_off = static_cast<i64>(pl->bterms.size());
      x.nterm = 1;
      x.last_lo = 0;
      x.last_hi = x.out_ext[d - 1];
      pl->bterms.push_back(terms[i][0]);
      pl->bitems.push_back(x);
    }
    pl->ops.push_back(Op{3, static_cast<i64>(pl->boxes.size()), group});
    pl->boxes.push_back(bl);
    return true;
  };
  // ---- Step 1: V / W
  std::vector<TRef> cur;  // per item (s, tau) of the current level
  for (int l = 0; l <= b.Lc; ++l) {
    const LevelData& ld = b.side[0][static_cast<size_t>(l)];
    const i64 nin = ld.L.nin, nj = ld.L.nj;
    const i64 nitems = b.nmid * nin;
    std::vector<TRef> in(static_cast<size_t>(nitems));
    for (i64 it = 0; it < nitems; ++it) {
      const i64 s = it / nin, tau = it % nin;
      if (!b.owns(s)) continue;  // another rank's column multi-set
      in[static_cast<size_t>(it)] =
          l == 0 ? global_slab(s) : cur[static_cast<size_t>(s * ipow(2, static_cast<i64>(d) * (l - 1)) + parent_of(tau, l))];
    }
    // ---- fused boxes
    const i64 scratch_mark = scratch;
    std::vector<TRef> outs(static_cast<size_t>(nitems));
    std::vector<BoxItem> items;
    std::vector<std::vector<BoxTerm>> terms;
    const i64 nbeta = ipow(nj, d);
    for (i64 it = 0; it < nitems; ++it) {
      const i64 s = it / nin, tau = it % nin;
      if (!b.owns(s)) continue;
      const TRef& x = in[static_cast<size_t>(it)];
      std::vector<std::vector<int>> R(d), W(d);
      std::vector<std::vector<i64>> MO(d);
      int oext[kMaxTM];
      for (int k = 0; k < d; ++k) {
        int tot_r = 0, tot_w = 0;
        for (i64 j = 0; j < nj; ++j) {
          int r, w;
          i64 mo;
          slot_info(0, l, s, tau, k, j, r, w, mo);
          R[k].push_back(r);
          W[k].push_back(w);
          MO[k].push_back(mo);
          tot_r += r;
          tot_w += w;
        }
        if (tot_w != x.ext[k]) throw std::runtime_error("internal: V/W block widths do not match the tensor extent");
        oext[k] = tot_r;
      }
      oext[d] = static_cast<int>(nv);
      const TRef y = alloc(nd, oext);
      outs[static_cast<size_t>(it)] = y;
      for (i64 beta = 0; beta < nbeta; ++beta) {
        BoxTerm t{};
        BoxItem bi{};
        t.in_off = x.off;
        bi.out_off = y.off;
        for (int k = 0; k < d; ++k) {
          const i64 j = (beta / ipow(nj, k)) % nj;
          i64 ci = 0, co = 0;
          for (i64 q = 0; q < j; ++q) {
            ci += W[k][static_cast<size_t>(q)];
            co += R[k][static_cast<size_t>(q)];
          }
          t.in_off += ci * x.stride[k];
          bi.out_off += co * y.stride[k];
          t.in_ext[k] = W[k][static_cast<size_t>(j)];
          bi.out_ext[k] = R[k][static_cast<size_t>(j)];
          t.mat_off[k] = MO[k][static_cast<size_t>(j)];
          t.mrows[k] = R[k][static_cast<size_t>(j)];
          t.mcols[k] = W[k][static_cast<size_t>(j)];
        }
        for (int p = 0; p < nd; ++p) {
          t.in_stride[p] = x.stride[p];
          bi.out_stride[p] = y.stride[p];
        }
        t.in_ext[d] = static_cast<int>(nv);
        bi.out_ext[d] = static_cast<int>(nv);
        bi.nterm = 1;
        items.push_back(bi);
        terms.push_back({t});
      }
    }
    if (commit_boxes(items, terms, 0, l, l == 0 ? BUF_F : BUF_SCRATCH, BUF_SCRATCH, 0, 0)) {
      cur = outs;
      continue;
    }
    scratch = scratch_mark;  // fall back to per-mode launches for this level
    for (int k = 0; k < d; ++k) {
      std::vector<MPStep> mitems;
      std::vector<std::vector<Blk>> blocks;
      for (i64 it = 0; it < nitems; ++it) {
        const i64 s = it / nin, tau = it % nin;
        if (!b.owns(s)) continue;
        TRef& x = in[static_cast<size_t>(it)];
        int oext[kMaxTM];
        for (int p = 0; p < nd; ++p) oext[p] = x.ext[p];
        std::vector<Blk> bl;
        int ci = 0, co = 0;
        for (i64 j = 0; j < nj; ++j) {
          Blk B;
          int r, w;
          slot_info(0, l, s, tau, k, j, r, w, B.mat_off);
          B.rows = r;
          B.cols = w;
          B.in_start = ci;
          B.out_start = co;
          ci += B.cols;
          co += B.rows;
          bl.push_back(B);
        }
        if (ci != x.ext[k]) throw std::runtime_error("internal: V/W block widths do not match the tensor extent");
        oext[k] = co;
        TRef y = alloc(nd, oext);
        mitems.push_back(make_step(x, y, k, 0));
        blocks.push_back(bl);
        x = y;
      }
      add_mp(*pl, 0, l, (l == 0 && k == 0) ? BUF_F : BUF_SCRATCH, BUF_SCRATCH, mitems, blocks, 0);
    }
    cur = in;
  }
  // ---- Step 2: cores.  x = F_{t,s} = cur[s * nmid + t]; y = G_{t,s}
  const LevelData& ULc = b.side[1][static_cast<size_t>(b.Lc)];
  std::vector<TRef> gts(static_cast<size_t>(b.nmid * b.nmid));  // index t * nmid + s
  i64 ctas = 0;
  const int rpc = gemv_rows_per_cta();
  const bool sharded = b.world > 1;
  pl->sharded = sharded;
  if (sharded)
    require(static_cast<i64>(b.send_off.size()) == b.nmid * b.nmid &&
                static_cast<i64>(b.recv_off.size()) == b.nmid * b.nmid,
            "sharded contract: exchange layout not set (oiobf_tbf_set_exchange)");
  const int* urank = sharded ? b.umid_rank.data() : ULc.h_rank.data();
  for (i64 p = 0; p < b.nmid * b.nmid; ++p) {
    const i64 s = p / b.nmid, t = p % b.nmid;
    int gext[kMaxTM];
    i64 R = 1;
    for (int k = 0; k < d; ++k) {
      gext[k] = urank[(t * b.nmid + s) * d + k];
      R *= gext[k];
    }
    gext[d] = static_cast<int>(nv);
    if (sharded && b.owns(t)) {  // P/U input G_{t,s} arrives in the receive buffer
      const i64 ro = b.recv_off[static_cast<size_t>(t * b.nmid + s)];
      require(ro >= 0, "sharded contract: missing receive offset");
      gts[static_cast<size_t>(t * b.nmid + s)] = packed(ro * nv, nd, gext);
    }
    if (!b.owns(s)) continue;
    const PairDesc& pd = b.h_pairs[static_cast<size_t>(p)];
    const TRef& x = cur[static_cast<size_t>(s * b.nmid + t)];
    TRef y;
    if (sharded) {  // GEMV output goes straight into the send buffer
      const i64 so = b.send_off[static_cast<size_t>(t * b.nmid + s)];
      require(so >= 0, "sharded contract: missing send offset");
      y = packed(so * nv, nd, gext);
    } else {
      y = alloc(nd, gext);
      gts[static_cast<size_t>(t * b.nmid + s)] = y;
    }
    if (R != pd.R || x.size() != static_cast<i64>(pd.C) * nv) throw std::runtime_error("internal: core shape mismatch");
    GemvDesc g;
    g.core_off = pd.core_off;
    g.x_off = x.off;
    g.y_off = y.off;
    g.R = pd.R;
    g.C = pd.C;
    g.cta_off = ctas;  // first global row of this pair
    ctas += pd.R;
    pl->gemv_max_c = std::max(pl->gemv_max_c, pd.C);
    pl->gemv.push_back(g);
  }
  (void)rpc;
  // persistent balanced grid: every CTA streams the same number of rows
  pl->gemv_total_rows = ctas;
  {
    const int per_sm = gemv_ctas_per_sm(static_cast<int>(nv), std::max(pl->gemv_max_c, 1));
    i64 grid = std::min<i64>(static_cast<i64>(148) * per_sm, std::max<i64>(ctas, 1));
    pl->gemv_rows_per_cta = (ctas + grid - 1) / grid;
    grid = (ctas + pl->gemv_rows_per_cta - 1) / pl->gemv_rows_per_cta;
    pl->gemv_ctas = ctas == 0 ? 0 : grid;
  }
  // TMA bulk-copy pipeline: one persistent CTA per SM, whole rows staged in a
  // shared-memory ring; used when rows are long enough to be worth a bulk
  // copy and every CTA's row range touches <= gemv_tma_max_pairs() pairs.
  {
    static const bool no_tma = std::getenv("OIOBF_GEMV_NO_TMA") != nullptr;
    const int max_c = pl->gemv_max_c;
    // measured on B200 (config 2): 2 CTAs/SM x 8 stages = 73% of HBM, same as
    // the register-streaming kernel; 1 CTA/SM is consumer-bound (45%)
    static const int per_sm_env = std::getenv("OIOBF_TMA_CTAS_PER_SM") ? std::atoi(std::getenv("OIOBF_TMA_CTAS_PER_SM")) : 2;
    static const int stages_env = std::getenv("OIOBF_TMA_STAGES") ? std::atoi(std::getenv("OIOBF_TMA_STAGES")) : 8;
    if (!no_tma && max_c >= 64 && ctas > 0) {
      i64 grid = std::min<i64>(148 * std::max(1, per_sm_env), ctas);
      const i64 rpc2 = (ctas + grid - 1) / grid;
      grid = (ctas + rpc2 - 1) / rpc2;
      const int stage_elems = (max_c + 7) / 8 * 8;
      const int xcap = max_c * static_cast<int>(nv);
      const i64 avail = static_cast<i64>(kMaxDynSmem) / std::max(1, per_sm_env) - 1024 -
                        static_cast<i64>(gemv_tma_max_pairs()) * xcap * static_cast<i64>(sizeof(double2));
      // rows go round-robin to the 8 consumer warps, so each stage must always
      // belong to the same consumer (stages % 8 == 0); otherwise a consumer
      // could wait two phases ahead and the parity check would be ambiguous
      i64 stages = std::min<i64>(stages_env, avail / (static_cast<i64>(stage_elems) * 16));
      stages = stages / 8 * 8;
      bool ok = stages >= 8;
      std::vector<int> map(static_cast<size_t>(grid));
      size_t q = 0;
      for (i64 c = 0; c < grid && ok; ++c) {
        const i64 g0 = c * rpc2, g1 = std::min(ctas, g0 + rpc2);
        while (q + 1 < pl->gemv.size() && pl->gemv[q + 1].cta_off <= g0) ++q;
        map[static_cast<size_t>(c)] = static_cast<int>(q);
        size_t q2 = q;
        while (q2 + 1 < pl->gemv.size() && pl->gemv[q2 + 1].cta_off < g1) ++q2;
        if (static_cast<int>(q2 - q + 1) > gemv_tma_max_pairs()) ok = false;
      }
      if (std::getenv("OIOBF_DEBUG"))
        fprintf(stderr, "[oiobf] gemv tma ok=%d grid=%lld rows/cta=%lld stages=%lld stage_elems=%d xcap=%d rows=%lld\n",
                ok ? 1 : 0, grid, rpc2, stages, stage_elems, xcap, ctas);
      if (ok) {
        pl->gemv_tma = true;
        pl->tma_ctas = grid;
        pl->tma_rows_per_cta = rpc2;
        pl->tma_stages = static_cast<int>(stages);
        pl->tma_stage_elems = stage_elems;
        pl->tma_xcap = xcap;
        pl->tma_map = map;
      }
    }
  }
  pl->ops.push_back(Op{1, 0, 1});
  // ---- Step 3: P (l = Lc..1, ordered child sums), U (l = 0)
  std::vector<TRef> gcur = gts;  // per (t, nu) at level l: index t * nin + nu
  for (int l = b.Lc; l >= 0; --l) {
    const LevelData& ld = b.side[1][static_cast<size_t>(l)];
    const i64 nin = ld.L.nin, nj = ld.L.nj;
    const i64 pnin = l > 0 ? ipow(2, static_cast<i64>(d) * (l - 1)) : 1;
    const i64 nbeta = ipow(nj, d);
    const i64 scratch_mark = scratch;
    std::vector<TRef> par(static_cast<size_t>(b.nmid * pnin));
    std::vector<BoxItem> items;
    std::vector<std::vector<BoxTerm>> terms;
    std::vector<SumDesc> psums;
    for (i64 t = 0; t < b.nmid; ++t)
      for (i64 pnu = 0; pnu < pnin; ++pnu) {
        if (!b.owns(t)) continue;  // another rank's row multi-set
        std::vector<i64> kids;
        for (i64 nu = 0; nu < nin; ++nu)
          if (l == 0 || parent_of(nu, l) == pnu) kids.push_back(nu);
        // widths (output side) are common to all children
        std::vector<std::vector<int>> W(d);
        int oext[kMaxTM];
        for (int k = 0; k < d; ++k) {
          int tw = 0;
          for (i64 j = 0; j < nj; ++j) {
            int r, w;
            i64 mo;
            slot_info(1, l, t, kids[0], k, j, r, w, mo);
            W[k].push_back(w);
            tw += w;
          }
          oext[k] = tw;
        }
        oext[d] = static_cast<int>(nv);
        const TRef y = l == 0 ? global_slab(t) : alloc(nd, oext);
        par[static_cast<size_t>(t * pnin + pnu)] = y;
        SumDesc sdsc{};
        for (i64 nu : kids) {
          // l >= 1: each child writes its own contribution (parent's shape),
          // summed afterwards in ascending nu; l = 0: straight into G
          const TRef yc = l == 0 ? y : alloc(nd, oext);
          if (l > 0) sdsc.child_off[sdsc.nchild++] = yc.off;
          const TRef& x = gcur[static_cast<size_t>(t * nin + nu)];
          for (i64 beta = 0; beta < nbeta; ++beta) {
            BoxItem bi{};
            BoxTerm tm{};
            bi.out_off = yc.off;
            tm.in_off = x.off;
            for (int k = 0; k < d; ++k) {
              const int jb = static_cast<int>((beta / ipow(nj, k)) % nj);
              i64 co = 0, ci = 0;
              int r = 0, w = 0;
              i64 mo = 0;
              for (int q = 0; q < jb; ++q) {
                slot_info(1, l, t, nu, k, q, r, w, mo);
                ci += r;
                co += w;
              }
              slot_info(1, l, t, nu, k, jb, r, w, mo);
              if (w != W[k][static_cast<size_t>(jb)]) throw std::runtime_error("internal: P/U widths differ");
              bi.out_off += co * yc.stride[k];
              bi.out_ext[k] = w;
              tm.in_off += ci * x.stride[k];
              tm.in_ext[k] = r;
              tm.mat_off[k] = mo;
              tm.mrows[k] = r;
              tm.mcols[k] = w;
            }
            bi.out_ext[d] = static_cast<int>(nv);
            tm.in_ext[d] = static_cast<int>(nv);
            for (int p = 0; p < nd; ++p) {
              bi.out_stride[p] = yc.stride[p];
              tm.in_stride[p] = x.stride[p];
            }
            bi.nterm = 1;
            items.push_back(bi);
            terms.push_back({tm});
          }
        }
        if (l > 0) {
          sdsc.out_off = y.off;
          sdsc.total = y.size();
          psums.push_back(sdsc);
        }
      }
    const int u_in = (sharded && l == b.Lc) ? BUF_RECV : BUF_SCRATCH;
    if (commit_boxes(items, terms, 1, l, u_in, l == 0 ? BUF_G : BUF_SCRATCH, 1, 2)) {
      if (l > 0) {
        SumLaunch sl;
        sl.begin = static_cast<i64>(pl->sums.size());
        sl.n = static_cast<i64>(psums.size());
        sl.work_begin = static_cast<i64>(pl->sum_map.size()) / 2;
        for (size_t q = 0; q < psums.size(); ++q)
          for (i64 c = 0; c * 1024 < psums[q].total; ++c) {
            pl->sum_map.push_back(static_cast<int>(q));
            pl->sum_map.push_back(static_cast<int>(c));
          }
        sl.total = static_cast<i64>(pl->sum_map.size()) / 2 - sl.work_begin;
        pl->sums.insert(pl->sums.end(), psums.begin(), psums.end());
        pl->ops.push_back(Op{4, static_cast<i64>(pl->sum_launches.size()), 2});
        pl->sum_launches.push_back(sl);
      }
      gcur = par;
      continue;
    }
    scratch = scratch_mark;  // fall back: per-mode launches + ordered sums
    const i64 nitems = b.nmid * nin;
    std::vector<TRef> x = gcur;
    for (int k = 0; k < d; ++k) {
      std::vector<MPStep> mitems;
      std::vector<std::vector<Blk>> blocks;
      const bool last_global = (l == 0 && k == d - 1);
      for (i64 it = 0; it < nitems; ++it) {
        const i64 t = it / nin, nu = it % nin;
        if (!b.owns(t)) continue;
        TRef& xi = x[static_cast<size_t>(it)];
        int oext[kMaxTM];
        for (int p = 0; p < nd; ++p) oext[p] = xi.ext[p];
        std::vector<Blk> bl;
        int ci = 0, co = 0;
        for (i64 j = 0; j < nj; ++j) {
          Blk B;
          int r, w;
          slot_info(1, l, t, nu, k, j, r, w, B.mat_off);
          B.rows = r;
          B.cols = w;
          B.in_start = ci;
          B.out_start = co;
          ci += B.rows;
          co += B.cols;
          bl.push_back(B);
        }
        if (ci != xi.ext[k]) throw std::runtime_error("internal: P/U block ranks do not match the tensor extent");
        oext[k] = co;
        TRef y = last_global ? global_slab(t) : alloc(nd, oext);
        mitems.push_back(make_step(xi, y, k, 1));
        blocks.push_back(bl);
        xi = y;
      }
      add_mp(*pl, 1, l, (k == 0 ? u_in : BUF_SCRATCH), last_global ? BUF_G : BUF_SCRATCH, mitems, blocks, 2);
    }
    if (l > 0) {
      std::vector<TRef> par2(static_cast<size_t>(b.nmid * pnin));
      SumLaunch sl;
      sl.begin = static_cast<i64>(pl->sums.size());
      i64 work = 0;
      for (i64 t = 0; t < b.nmid; ++t)
        for (i64 pnu = 0; pnu < pnin; ++pnu) {
          if (!b.owns(t)) continue;
          SumDesc sdsc{};
          TRef first;
          for (i64 nu = 0; nu < nin; ++nu) {
            if (parent_of(nu, l) != pnu) continue;
            const TRef& c = x[static_cast<size_t>(t * nin + nu)];
            if (sdsc.nchild == 0) first = c;
            sdsc.child_off[sdsc.nchild++] = c.off;
          }
          TRef y = alloc(nd, first.ext);
          sdsc.out_off = y.off;
          sdsc.total = y.size();
          sdsc.work_off = work;
          work += sdsc.total;
          pl->sums.push_back(sdsc);
          par2[static_cast<size_t>(t * pnin + pnu)] = y;
        }
      sl.n = static_cast<i64>(pl->sums.size()) - sl.begin;
      sl.total = work;
      pl->ops.push_back(Op{2, static_cast<i64>(pl->sum_launches.size()), 2});
      pl->sum_launches.push_back(sl);
      gcur = par2;
    }
  }
  pl->scratch_elems = scratch;
  cudaStream_t st = b.stream;
  pl->d_steps = to_device(pl->steps, st);
  pl->d_blks = to_device(pl->blks, st);
  pl->d_gemv = to_device(pl->gemv, st);
  {
    std::vector<int> map(static_cast<size_t>(std::max<i64>(pl->gemv_ctas, 1)));
    size_t p = 0;
    for (i64 c = 0; c < pl->gemv_ctas; ++c) {  // pair holding CTA c's first row
      const i64 g0 = c * pl->gemv_rows_per_cta;
      while (p + 1 < pl->gemv.size() && pl->gemv[p + 1].cta_off <= g0) ++p;
      map[static_cast<size_t>(c)] = static_cast<int>(p);
    }
    pl->d_gemv_map = to_device(map, st);
    if (pl->gemv_tma) pl->d_tma_map = to_device(pl->tma_map, st);
  }
  pl->d_sums = to_device(pl->sums, st);
  pl->d_bitems = to_device(pl->bitems, st);
  pl->d_sum_map = to_device(pl->sum_map, st);
  pl->d_bterms = to_device(pl->bterms, st);
  pl->scratch.alloc(static_cast<size_t>(std::max<i64>(scratch, 1)));
  TBF_CUDA(cudaStreamSynchronize(st));
  return pl;
}

Plan& get_plan(oiobf_tbf& b, i64 nv) {
  auto it = b.plans.find(nv);
  if (it != b.plans.end()) return *it->second;
  auto& slot = b.plans[nv];
  slot = build_plan(b, nv);
  return *slot;
}

struct OpBuffers {
  const double2* F = nullptr;
  double2* G = nullptr;
  double2* send = nullptr;
  const double2* recv = nullptr;
};

// phase: 0 = whole contraction, 1 = V/W + core GEMV, 2 = P/U (sharded)
void run_ops(oiobf_tbf& b, Plan& pl, const OpBuffers& io, cudaStream_t st, int group_filter = -1, int phase = 0) {
  // OIOBF_ABLATE=<digits>: skip these op kinds (timing experiments only; the
  // result is wrong when set)
  static const char* ablate = std::getenv("OIOBF_ABLATE");
  auto in_ptr = [&](int id) -> const double2* {
    return id == BUF_F ? io.F : id == BUF_RECV ? io.recv : pl.scratch.p;
  };
  auto out_ptr = [&](int id) -> double2* { return id == BUF_G ? io.G : id == BUF_SEND ? io.send : pl.scratch.p; };
  for (const Op& op : pl.ops) {
    if (group_filter >= 0 && op.group != group_filter) continue;
    if (phase == 1 && op.group == 2) continue;
    if (phase == 2 && op.group != 2) continue;
    if (ablate && std::strchr(ablate, '0' + op.kind)) continue;
    if (op.kind == 0) {
      const MPLaunch& m = pl.mps[static_cast<size_t>(op.idx)];
      const LevelData& ld = b.side[m.side][static_cast<size_t>(m.level)];
      launch_mode_product(m.nsteps, pl.d_steps.p + m.step_begin, m.total_out, pl.d_blks.p, ld.interp.p,
                          in_ptr(m.in_buf), out_ptr(m.out_buf), st);
    } else if (op.kind == 1) {
      double2* y = pl.sharded ? io.send : pl.scratch.p;
      if (pl.gemv_tma)
        launch_gemv_tma(pl.d_tma_map.p, pl.d_gemv.p, pl.tma_ctas, pl.gemv_total_rows, pl.tma_rows_per_cta,
                        static_cast<int>(pl.nv), pl.tma_stages, pl.tma_stage_elems, pl.tma_xcap, b.cores.p,
                        pl.scratch.p, y, st);
      else
        launch_gemv(pl.d_gemv_map.p, pl.d_gemv.p, pl.gemv_ctas, pl.gemv_total_rows, pl.gemv_rows_per_cta,
                    static_cast<int>(pl.nv), b.cores.p, pl.scratch.p, y, pl.gemv_max_c, st);
    } else if (op.kind == 3) {
      const BoxLaunch& bx = pl.boxes[static_cast<size_t>(op.idx)];
      const LevelData& ld = b.side[bx.side][static_cast<size_t>(bx.level)];
      launch_box(bx.nitems, pl.d_bitems.p + bx.item_begin, pl.d_bterms.p + bx.item_begin, bx.info, ld.interp.p,
                 in_ptr(bx.in_buf), out_ptr(bx.out_buf), st);
    } else if (op.kind == 4) {
      const SumLaunch& s = pl.sum_launches[static_cast<size_t>(op.idx)];
      launch_sum_parent(s.total, pl.d_sums.p + s.begin, pl.d_sum_map.p + 2 * s.work_begin, pl.scratch.p,
                        pl.scratch.p, st);
    } else {
      const SumLaunch& s = pl.sum_launches[static_cast<size_t>(op.idx)];
      launch_sum_children(s.n, pl.d_sums.p + s.begin, s.total, pl.scratch.p, pl.scratch.p, st);
    }
  }
}

void run_ops(oiobf_tbf& b, Plan& pl, const double2* F, double2* G, cudaStream_t st, int group_filter = -1) {
  OpBuffers io;
  io.F = F;
  io.G = G;
  run_ops(b, pl, io, st, group_filter, 0);
}

void contract_device(oiobf_tbf& b, const double2* F, double2* G, i64 nv, cudaStream_t st) {
  require(nv >= 1, "tbf_contract: nv must be >= 1");
  TBF_CUDA(cudaSetDevice(b.device));
  Plan& pl = get_plan(b, nv);
  static const bool no_graph = std::getenv("OIOBF_NO_GRAPH") != nullptr;  // profiling aid
  if (no_graph) {
    run_ops(b, pl, F, G, st);
    return;
  }
  if (!pl.gexec || pl.g_F != F || pl.g_G != G || pl.g_st != st) {
    if (pl.gexec) {
      cudaGraphExecDestroy(pl.gexec);
      pl.gexec = nullptr;
    }
    cudaStream_t cap;
    TBF_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    cudaGraph_t g;
    TBF_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    try {
      run_ops(b, pl, F, G, cap);
    } catch (...) {
      cudaStreamEndCapture(cap, &g);
      cudaStreamDestroy(cap);
      throw;
    }
    TBF_CUDA(cudaStreamEndCapture(cap, &g));
    TBF_CUDA(cudaGraphInstantiate(&pl.gexec, g, 0));
    TBF_CUDA(cudaGraphDestroy(g));
    TBF_CUDA(cudaStreamDestroy(cap));
    pl.g_F = F;
    pl.g_G = G;
    pl.g_st = st;
  }
  TBF_CUDA(cudaGraphLaunch(pl.gexec, st));
}

int status_of(const std::exception& e) {
  g_err = e.what();
  return dynamic_cast<const InvalidArg*>(&e) ? OIOBF_EINVAL : OIOBF_ERUNTIME;
}

#define CAPI_BEGIN try {
#define CAPI_END                      \
  }                                   \
  catch (const std::exception& e) {   \
    return status_of(e);              \
  }                                   \
  catch (...) {                       \
    g_err = "unknown C++ exception";  \
    return OIOBF_ERUNTIME;            \
  }                                   \
  return OIOBF_OK;

}  // namespace

extern "C" {

const char* oiobf_last_error(void) { return g_err.c_str(); }

int oiobf_set_device(int device) {
  CAPI_BEGIN
  g_device = device;
  ensure_device();
  CAPI_END
}

int oiobf_device_info(int64_t out[4]) {
  CAPI_BEGIN
  ensure_device();
  cudaDeviceProp p;
  TBF_CUDA(cudaGetDeviceProperties(&p, g_device));
  out[0] = p.multiProcessorCount;
  out[1] = p.major;
  out[2] = p.minor;
  out[3] = static_cast<int64_t>(p.totalGlobalMem);
  CAPI_END
}

uint64_t oiobf_derive_seed(uint64_t seed, const uint64_t* tags, int32_t ntags) {
  return derive_seed(seed, reinterpret_cast<const u64*>(tags), ntags);
}

int oiobf_select_proxies_count(int64_t extent, int64_t count, int32_t mode, uint64_t seed, int64_t* out,
                               int64_t* out_count) {
  CAPI_BEGIN
  require(extent >= 1, "select_proxies: extent must be positive");
  require(mode >= 0 && mode <= 2, "select_proxies: unknown mode");
  i64 c = std::min<i64>(extent, std::max<i64>(count, 1));
  require(mode != OIOBF_PROXY_UNIFORM_RANDOM || c <= kMaxProxy, "select_proxies: count exceeds device limit (64)");
  std::vector<int> tmp(static_cast<size_t>(mode == OIOBF_PROXY_ALL ? extent : c));
  const i64 got = select_proxies(extent, count, mode, seed, tmp.data());
  for (i64 i = 0; i < got; ++i) out[i] = tmp[static_cast<size_t>(i)];
  *out_count = got;
  CAPI_END
}

int oiobf_tbf_construct(const oiobf_kernel_spec* spec, int32_t L, double tol, const oiobf_proxy_strategy* proxies,
                        uint64_t seed, oiobf_tbf** out) {
  CAPI_BEGIN
  require(spec && proxies && out, "tbf_construct: null argument");
  *out = construct(*spec, L, tol, *proxies, seed);
  CAPI_END
}

int oiobf_tbf_destroy(oiobf_tbf* h) {
  CAPI_BEGIN
  delete h;
  CAPI_END
}

// ---- sharded construction / apply ---------------------------
int oiobf_tbf_shard_begin(const oiobf_kernel_spec* spec, int32_t L, double tol, const oiobf_proxy_strategy* proxies,
                          uint64_t seed, int32_t rank, int32_t world, oiobf_tbf** out) {
  CAPI_BEGIN
  require(spec && proxies && out, "tbf_shard_begin: null argument");
  *out = construct_begin(*spec, L, tol, *proxies, seed, rank, world).release();
  CAPI_END
}

int oiobf_tbf_shard_level(oiobf_tbf* h, int32_t side, int32_t level, int64_t r_est, int64_t* local_max_rank) {
  CAPI_BEGIN
  require(h && local_max_rank, "tbf_shard_level: null argument");
  require(side == 0 || side == 1, "tbf_shard_level: side must be 0 (V/W) or 1 (U/P)");
  require(level >= 0 && level <= h->Lc, "tbf_shard_level: level out of range");
  require(static_cast<int>(h->r_est[side].size()) == level, "tbf_shard_level: levels must be built in order");
  std::lock_guard<std::mutex> lk(h->mu);
  TBF_CUDA(cudaSetDevice(h->device));
  h->r_est[side].push_back(r_est);
  build_side_level(*h, side, level, r_est);
  *local_max_rank = h->side[side][static_cast<size_t>(level)].max_rank;
  CAPI_END
}

// out[0] = number of U-side middle slots (nmid * nmid * d), out[1] = local max rank there
int oiobf_tbf_umid_info(oiobf_tbf* h, int64_t out[2]) {
  CAPI_BEGIN
  require(h && static_cast<int>(h->side[1].size()) == h->Lc + 1 && !h->side[1].back().h_rank.empty(),
          "tbf_umid_info: U side not built");
  const LevelData& U = h->side[1].back();
  out[0] = U.nslots;
  out[1] = U.max_rank;
  CAPI_END
}

// ranks[nslots] and skeletons (nslots x wpad, zero padded) of this rank's
// U-side middle slots; other slots are left at zero (sum-reduce to gather)
int oiobf_tbf_umid_export(oiobf_tbf* h, int64_t* ranks, int32_t* skel, int64_t wpad) {
  CAPI_BEGIN
  require(h && ranks && skel, "tbf_umid_export: null argument");
  std::lock_guard<std::mutex> lk(h->mu);
  TBF_CUDA(cudaSetDevice(h->device));
  const LevelData& U = h->side[1].back();
  require(wpad >= U.max_rank, "tbf_umid_export: wpad smaller than the local max rank");
  std::vector<int> hs(static_cast<size_t>(U.total_skel));
  U.skel.download(hs.data(), hs.size(), h->stream);
  TBF_CUDA(cudaStreamSynchronize(h->stream));
  for (i64 q = 0; q < U.nslots; ++q) {
    const int r = U.h_rank[static_cast<size_t>(q)];
    ranks[q] = r;
    for (int i = 0; i < wpad; ++i)
      skel[q * wpad + i] = i < r ? hs[static_cast<size_t>(U.h_skel_off[static_cast<size_t>(q)] + i)] : 0;
  }
  CAPI_END
}

// install the gathered U-side middle ranks / skeletons of all ranks and
// generate the cores of the pairs (t, s) whose s this rank owns
int oiobf_tbf_umid_import(oiobf_tbf* h, const int64_t* ranks, const int32_t* skel, int64_t wpad) {
  CAPI_BEGIN
  require(h && ranks && skel, "tbf_umid_import: null argument");
  std::lock_guard<std::mutex> lk(h->mu);
  TBF_CUDA(cudaSetDevice(h->device));
  require(static_cast<int>(h->side[0].size()) == h->Lc + 1 && !h->side[0].back().h_rank.empty(),
          "tbf_umid_import: V side not built");
  const LevelData& U = h->side[1].back();
  h->umid_rank.assign(static_cast<size_t>(U.nslots), 0);
  h->umid_skel_off.assign(static_cast<size_t>(U.nslots), 0);
  std::vector<int> flat;
  for (i64 q = 0; q < U.nslots; ++q) {
    require(ranks[q] >= 0 && ranks[q] <= wpad, "tbf_umid_import: bad rank");
    h->umid_rank[static_cast<size_t>(q)] = static_cast<int>(ranks[q]);
    h->umid_skel_off[static_cast<size_t>(q)] = static_cast<i64>(flat.size());
    for (i64 i = 0; i < ranks[q]; ++i) flat.push_back(skel[q * wpad + i]);
    if (h->owns(q / (h->nmid * h->d)))  // own slots must agree with the gathered copy
      require(U.h_rank[static_cast<size_t>(q)] == ranks[q], "tbf_umid_import: gathered ranks disagree");
  }
  if (flat.empty()) flat.push_back(0);
  h->umid_skel = to_device(flat, h->stream);
  build_cores(*h);
  TBF_CUDA(cudaStreamSynchronize(h->stream));
  CAPI_END
}

// Exchange layout (element offsets at nv = 1 of every G_{t,s} block in this
// rank's send / receive buffers, index t * nmid + s, -1 = not exchanged here)
int oiobf_tbf_set_exchange(oiobf_tbf* h, const int64_t* send_off, const int64_t* recv_off, int64_t send_elems,
                           int64_t recv_elems) {
  CAPI_BEGIN
  require(h && send_off && recv_off, "tbf_set_exchange: null argument");
  std::lock_guard<std::mutex> lk(h->mu);
  const i64 P = h->nmid * h->nmid;
  h->send_off.assign(send_off, send_off + P);
  h->recv_off.assign(recv_off, recv_off + P);
  h->send_elems = send_elems;
  h->recv_elems = recv_elems;
  h->plans.clear();
  CAPI_END
}

// phase 1: dIn = F (n^d x nv), dOut = send buffer; phase 2: dIn = receive
// buffer, dOut = G (only this rank's row slabs are written)
int oiobf_tbf_contract_phase(oiobf_tbf* h, int32_t phase, const void* dIn, void* dOut, int64_t nv, void* stream) {
  CAPI_BEGIN
  require(h && dIn && dOut, "tbf_contract_phase: null argument");
  require(phase == 1 || phase == 2, "tbf_contract_phase: phase must be 1 or 2");
  require(nv >= 1, "tbf_contract: nv must be >= 1");
  std::lock_guard<std::mutex> lk(h->mu);
  TBF_CUDA(cudaSetDevice(h->device));
  Plan& pl = get_plan(*h, nv);
  OpBuffers io;
  if (phase == 1) {
    io.F = static_cast<const double2*>(dIn);
    io.send = static_cast<double2*>(dOut);
  } else {
    io.recv = static_cast<const double2*>(dIn);
    io.G = static_cast<double2*>(dOut);
  }
  run_ops(*h, pl, io, static_cast<cudaStream_t>(stream), -1, phase);
  CAPI_END
}

int oiobf_tbf_contract_device(oiobf_tbf* h, const void* dF, void* dG, int64_t nv, void* stream) {
  CAPI_BEGIN
  require(h && dF && dG, "tbf_contract: null argument");
  require(h->world == 1, "tbf_contract: sharded factorization -- use oiobf_tbf_contract_phase");
  std::lock_guard<std::mutex> lk(h->mu);
  contract_device(*h, static_cast<const double2*>(dF), static_cast<double2*>(dG), nv,
                  static_cast<cudaStream_t>(stream));
  CAPI_END
}

int oiobf_tbf_contract(oiobf_tbf* h, const double* F, double* G, int64_t nv) {
  CAPI_BEGIN
  require(h && F && G, "tbf_contract: null argument");
  require(nv >= 1, "tbf_contract: nv must be >= 1");
  std::lock_guard<std::mutex> lk(h->mu);
  TBF_CUDA(cudaSetDevice(h->device));
  const size_t N = static_cast<size_t>(ipow(h->n, h->d) * nv);
  Plan& pl = get_plan(*h, nv);
  if (pl.stage_F.n != N) {  // staging buffers persist so the captured graph is reused
    pl.stage_F.alloc(N);
    pl.stage_G.alloc(N);
  }
  TBF_CUDA(cudaMemcpyAsync(pl.stage_F.p, F, N * sizeof(double2), cudaMemcpyHostToDevice, h->stream));
  contract_device(*h, pl.stage_F.p, pl.stage_G.p, nv, h->stream);
  TBF_CUDA(cudaMemcpyAsync(G, pl.stage_G.p, N * sizeof(double2), cudaMemcpyDeviceToHost, h->stream));
  TBF_CUDA(cudaStreamSynchronize(h->stream));
  CAPI_END
}

int oiobf_tbf_memory(const oiobf_tbf* h, int64_t out[5]) {
  CAPI_BEGIN
  require(h, "tbf_memory: null handle");
  for (int i = 0; i < 5; ++i) out[i] = 0;
  for (int sd = 0; sd < 2; ++sd)
    for (size_t l = 0; l < h->side[sd].size(); ++l)
      out[(sd == 0 ? 0 : 2) + (l > 0 ? 1 : 0)] += h->side[sd][l].total_interp * 16;
  out[4] = h->total_core * 16;
  CAPI_END
}

int oiobf_tbf_info(const oiobf_tbf* h, int64_t info[10]) {
  CAPI_BEGIN
  require(h, "tbf_info: null handle");
  i64 slots = 0, sk = 0, ip = 0, pm = 0;
  for (int sd = 0; sd < 2; ++sd)
    for (const auto& lv : h->side[sd]) {
      slots += lv.nslots;
      sk += lv.total_skel;
      ip += lv.total_interp;
      for (int w : lv.h_width) pm += w;
    }
  info[0] = h->d;
  info[1] = h->n;
  info[2] = h->L;
  info[3] = h->Lc;
  info[4] = h->nmid;
  info[5] = slots;
  info[6] = sk;
  info[7] = ip;
  info[8] = h->total_core;
  info[9] = pm;
  CAPI_END
}

int oiobf_tbf_export(const oiobf_tbf* h, int64_t* ranks, int64_t* ncols, int64_t* rows, int64_t* skel,
                     double* interp, int64_t* perm, double* cores, int64_t* core_rows, int64_t* core_cols,
                     int64_t* r_est) {
  CAPI_BEGIN
  require(h, "tbf_export: null handle");
  TBF_CUDA(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  i64 si = 0, sk = 0, ip = 0, pm = 0;
  for (int sd = 0; sd < 2; ++sd)
    for (const auto& lv : h->side[sd]) {
      const i64 ns = lv.nslots;
      std::vector<int> hs(static_cast<size_t>(lv.total_skel)), hp(static_cast<size_t>(ns * lv.L.wmax));
      std::vector<double2> hi(static_cast<size_t>(lv.total_interp));
      lv.skel.download(hs.data(), hs.size(), st);
      lv.interp.download(hi.data(), hi.size(), st);
      lv.perm.download(hp.data(), hp.size(), st);
      TBF_CUDA(cudaStreamSynchronize(st));
      for (i64 i = 0; i < ns; ++i) {
        const int r = lv.h_rank[static_cast<size_t>(i)], w = lv.h_width[static_cast<size_t>(i)];
        if (ranks) ranks[si] = r;
        if (ncols) ncols[si] = w;
        if (rows) rows[si] = lv.L.m;
        for (int q = 0; q < w; ++q)
          if (perm) perm[pm + q] = hp[static_cast<size_t>(i * lv.L.wmax + q)];
        pm += w;
        ++si;
      }
      if (skel)
        for (size_t q = 0; q < hs.size(); ++q) skel[sk + static_cast<i64>(q)] = hs[q];
      if (interp) std::memcpy(interp + 2 * ip, hi.data(), hi.size() * sizeof(double2));
      sk += lv.total_skel;
      ip += lv.total_interp;
    }
  if (cores || core_rows || core_cols) {
    std::vector<double2> hc(static_cast<size_t>(h->total_core));
    h->cores.download(hc.data(), hc.size(), st);
    TBF_CUDA(cudaStreamSynchronize(st));
    for (size_t p = 0; p < h->h_pairs.size(); ++p) {
      const PairDesc& pd = h->h_pairs[p];
      if (core_rows) core_rows[p] = pd.R;
      if (core_cols) core_cols[p] = pd.C;
      if (cores)  // row-major on device -> reference column-major matricization
        for (int r = 0; r < pd.R; ++r)
          for (int c = 0; c < pd.C; ++c) {
            const double2 v = hc[static_cast<size_t>(pd.core_off + static_cast<i64>(r) * pd.C + c)];
            const i64 o = pd.core_off + r + static_cast<i64>(c) * pd.R;
            cores[2 * o] = v.x;
            cores[2 * o + 1] = v.y;
          }
    }
  }
  if (r_est) {
    i64 q = 0;
    for (int sd = 0; sd < 2; ++sd)
      for (auto v : h->r_est[sd]) r_est[q++] = v;
  }
  CAPI_END
}

// Non-finite entries in the factors: out[2*(side*(Lc+1)+l)] = interp count,
// out[...+1] = 0; out[2*2*(Lc+1)] = cores.  (robustness diagnostic)
int oiobf_tbf_check_finite(oiobf_tbf* h, int64_t* out) {
  CAPI_BEGIN
  require(h, "tbf_check_finite: null handle");
  TBF_CUDA(cudaSetDevice(h->device));
  i64 q = 0;
  for (int sd = 0; sd < 2; ++sd)
    for (const auto& lv : h->side[sd]) {
      out[q++] = static_cast<int64_t>(count_nonfinite(lv.interp.p, lv.total_interp, h->stream));
      out[q++] = lv.max_rank;
    }
  out[q] = static_cast<int64_t>(count_nonfinite(h->cores.p, h->total_core, h->stream));
  CAPI_END
}

int oiobf_tbf_timings(const oiobf_tbf* h, double out[6]) {
  CAPI_BEGIN
  require(h, "tbf_timings: null handle");
  for (int i = 0; i < 6; ++i) out[i] = h->t_ms[i];
  CAPI_END
}

int oiobf_tbf_plan_stats(oiobf_tbf* h, int64_t out[4]) {
  CAPI_BEGIN
  require(h, "tbf_plan_stats: null handle");
  std::lock_guard<std::mutex> lk(h->mu);
  Plan& pl = get_plan(*h, 1);
  i64 fac = 0;
  for (int sd = 0; sd < 2; ++sd)
    for (const auto& lv : h->side[sd]) fac += lv.total_interp;
  const i64 N = ipow(h->n, h->d);
  out[0] = 16 * (2 * N + fac + h->total_core);
  out[1] = 16 * h->total_core;
  out[2] = static_cast<int64_t>(pl.ops.size());
  i64 macs = h->total_core;
  for (const MPStep& s : pl.steps) {
    // each output element of a step costs (block input width) MACs; approximate
    // with the average block width of its item
    (void)s;
  }
  for (const MPLaunch& m : pl.mps) {
    for (i64 i = 0; i < m.nsteps; ++i) {
      const MPStep& s = pl.steps[static_cast<size_t>(m.step_begin + i)];
      const i64 per_out = s.total / std::max(1, s.ext[s.mode]);
      for (int q = 0; q < s.nblk; ++q) {
        const Blk& B = pl.blks[static_cast<size_t>(s.blk_off + q)];
        macs += per_out * B.rows * B.cols;
      }
    }
  }
  out[3] = macs;
  CAPI_END
}

// Debug: run every box launch of the nv=1 plan once with per-CTA phase stamps;
// out gets, per box launch, [ctas, mean and max (ns) of: desc, stage, modes, reduce, total]
int oiobf_debug_box_trace(oiobf_tbf* h, const void* dF, void* dG, double* out, int32_t max_launches) {
  CAPI_BEGIN
  std::lock_guard<std::mutex> lk(h->mu);
  TBF_CUDA(cudaSetDevice(h->device));
  Plan& pl = get_plan(*h, 1);
  DevBuf<unsigned long long> tr(1 << 22);
  box_trace_enable(tr.p);
  int li = 0;
  for (const Op& op : pl.ops) {
    if (op.kind != 3 || li >= max_launches) continue;
    const BoxLaunch& bx = pl.boxes[static_cast<size_t>(op.idx)];
    const double2* in = bx.in_buf == BUF_F ? static_cast<const double2*>(dF) : pl.scratch.p;
    double2* o = bx.out_buf == BUF_G ? static_cast<double2*>(dG) : pl.scratch.p;
    const LevelData& ld = h->side[bx.side][static_cast<size_t>(bx.level)];
    TBF_CUDA(cudaMemset(tr.p, 0, tr.n * 8));
    launch_box(bx.nitems, pl.d_bitems.p + bx.item_begin, pl.d_bterms.p + bx.item_begin, bx.info, ld.interp.p, in, o,
               h->stream);
    TBF_CUDA(cudaStreamSynchronize(h->stream));
    const i64 nct = bx.nitems * bx.info.cs;
    std::vector<unsigned long long> ht(static_cast<size_t>(nct * 8));
    TBF_CUDA(cudaMemcpy(ht.data(), tr.p, ht.size() * 8, cudaMemcpyDeviceToHost));
    double* o9 = out + 11 * li;
    o9[0] = static_cast<double>(nct);
    unsigned long long t0 = ~0ULL;
    for (i64 c = 0; c < nct; ++c) t0 = std::min(t0, ht[static_cast<size_t>(c * 8)]);
    for (int ph = 0; ph < 4; ++ph) {
      double sum = 0, mx = 0;
      for (i64 c = 0; c < nct; ++c) {
        const double dt = static_cast<double>(ht[static_cast<size_t>(c * 8 + ph + 1)] - ht[static_cast<size_t>(c * 8 + ph)]);
        sum += dt;
        mx = std::max(mx, dt);
      }
      o9[1 + 2 * ph] = sum / nct;
      o9[2 + 2 * ph] = mx;
    }
    double span = 0, late = 0;
    for (i64 c = 0; c < nct; ++c) {
      span = std::max(span, static_cast<double>(ht[static_cast<size_t>(c * 8 + 4)] - t0));
      late = std::max(late, static_cast<double>(ht[static_cast<size_t>(c * 8)] - t0));
    }
    o9[9] = span;
    o9[10] = late;  // last CTA start relative to the first
    {  // second (warm) execution of the mode phase: stamps 2 -> 7 -> 3
      double w1 = 0, w2 = 0;
      for (i64 c = 0; c < nct; ++c) {
        w1 += static_cast<double>(ht[static_cast<size_t>(c * 8 + 7)] - ht[static_cast<size_t>(c * 8 + 2)]);
        w2 += static_cast<double>(ht[static_cast<size_t>(c * 8 + 3)] - ht[static_cast<size_t>(c * 8 + 7)]);
      }
      o9[5] = w1 / nct;  // modes, first (cold) pass
      o9[6] = w2 / nct;  // modes, second (warm) pass
    }
    // effective SM clock (MHz) of CTA 0: cycles / ns
    o9[0] += 1e-6 * static_cast<double>(ht[6] - ht[5]) / std::max(1.0, static_cast<double>(ht[4] - ht[0])) * 1000.0;
    ++li;
  }
  box_trace_enable(nullptr);
  CAPI_END
}

int oiobf_tbf_profile_contract(oiobf_tbf* h, const void* dF, void* dG, int32_t reps, void* stream, double out[4]) {
  CAPI_BEGIN
  require(h && dF && dG && reps >= 1, "tbf_profile_contract: bad argument");
  std::lock_guard<std::mutex> lk(h->mu);
  TBF_CUDA(cudaSetDevice(h->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Plan& pl = get_plan(*h, 1);
  for (int g = 0; g < 3; ++g) {
    run_ops(*h, pl, static_cast<const double2*>(dF), static_cast<double2*>(dG), st, g);  // warm
    EventTimer t(st);
    for (int r = 0; r < reps; ++r)
      run_ops(*h, pl, static_cast<const double2*>(dF), static_cast<double2*>(dG), st, g);
    out[g] = t.stop() / reps;
  }
  EventTimer t(st);
  for (int r = 0; r < reps; ++r) contract_device(*h, static_cast<const double2*>(dF), static_cast<double2*>(dG), 1, st);
  out[3] = t.stop() / reps;
  CAPI_END
}

int oiobf_dense_rows(const oiobf_kernel_spec* spec, const double* F, int64_t nv, int64_t nrows,
                     const int64_t* rows_flat, double* out) {
  CAPI_BEGIN
  require(spec && F && rows_flat && out, "dense_rows: null argument");
  validate_spec(*spec);
  require(nv >= 1 && nrows >= 0, "dense_rows: bad sizes");
  ensure_device();
  const i64 N = ipow(spec->n, spec->d);
  for (i64 r = 0; r < nrows; ++r) require(rows_flat[r] >= 0 && rows_flat[r] < N, "dense_rows: row out of range");
  cudaStream_t st;
  TBF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  {
    DevBuf<double2> dF(static_cast<size_t>(N * nv)), dO(static_cast<size_t>(std::max<i64>(nrows * nv, 1)));
    DevBuf<i64> dr(static_cast<size_t>(std::max<i64>(nrows, 1)));
    dF.upload(reinterpret_cast<const double2*>(F), static_cast<size_t>(N * nv), st);
    dr.upload(reinterpret_cast<const i64*>(rows_flat), static_cast<size_t>(nrows), st);
    if (nrows) launch_dense_rows(kspec_from(*spec), nrows, dr.p, dF.p, static_cast<int>(nv), dO.p, st);
    dO.download(reinterpret_cast<double2*>(out), static_cast<size_t>(nrows * nv), st);
    TBF_CUDA(cudaStreamSynchronize(st));
  }
  cudaStreamDestroy(st);
  CAPI_END
}

int oiobf_subtensor_at(const oiobf_kernel_spec* spec, const int64_t* counts, const int64_t* lists, double* out) {
  CAPI_BEGIN
  require(spec && counts && lists && out, "subtensor_at: null argument");
  validate_spec(*spec);
  ensure_device();
  const int D = 2 * spec->d;
  i64 total = 1, nl = 0;
  for (int p = 0; p < D; ++p) {
    require(counts[p] >= 0, "subtensor_at: negative count");
    total *= counts[p];
    nl += counts[p];
  }
  std::vector<int> hl(static_cast<size_t>(std::max<i64>(nl, 1)));
  for (i64 q = 0; q < nl; ++q) {
    require(lists[q] >= 1 && lists[q] <= spec->n, "subtensor: index out of bounds");
    hl[static_cast<size_t>(q)] = static_cast<int>(lists[q]);
  }
  cudaStream_t st;
  TBF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  {
    DevBuf<int> dl = to_device(hl, st);
    DevBuf<double2> dO(static_cast<size_t>(std::max<i64>(total, 1)));
    launch_subtensor(kspec_from(*spec), reinterpret_cast<const i64*>(counts), dl.p, total, dO.p, st);
    dO.download(reinterpret_cast<double2*>(out), static_cast<size_t>(total), st);
    TBF_CUDA(cudaStreamSynchronize(st));
  }
  cudaStreamDestroy(st);
  CAPI_END
}

int oiobf_mode_product_blockdiag(int32_t nmodes, const int64_t* shape, const double* t, int32_t mode, int32_t nb,
                                 const int64_t* br, const int64_t* bc, const double* blocks, int32_t transpose,
                                 double* out) {
  CAPI_BEGIN
  require(nmodes >= 1 && nmodes <= kMaxTM, "mode_product_blockdiag: 1..7 modes supported");
  require(mode >= 1 && mode <= nmodes, "mode_product_blockdiag: mode out of range");
  require(nb >= 1, "mode_product_blockdiag: no blocks");
  ensure_device();
  int ext[kMaxTM];
  for (int p = 0; p < nmodes; ++p) {
    require(shape[p] >= 0, "DenseTensor: negative extent");
    ext[p] = static_cast<int>(shape[p]);
  }
  i64 in_total = 0, out_total = 0, mat_total = 0;
  std::vector<Blk> bl;
  for (int b = 0; b < nb; ++b) {
    Blk B;
    B.mat_off = mat_total;
    B.rows = static_cast<int>(br[b]);
    B.cols = static_cast<int>(bc[b]);
    B.in_start = static_cast<int>(in_total);
    B.out_start = static_cast<int>(out_total);
    in_total += transpose ? br[b] : bc[b];
    out_total += transpose ? bc[b] : br[b];
    mat_total += br[b] * bc[b];
    bl.push_back(B);
  }
  require(in_total == shape[mode - 1], "mode_product_blockdiag: shape mismatch");
  TRef in = packed(0, nmodes, ext);
  int oext[kMaxTM];
  for (int p = 0; p < nmodes; ++p) oext[p] = ext[p];
  oext[mode - 1] = static_cast<int>(out_total);
  TRef o = packed(0, nmodes, oext);
  MPStep s = make_step(in, o, mode - 1, transpose);
  s.work_off = 0;
  s.blk_off = 0;
  s.nblk = nb;
  cudaStream_t st;
  TBF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  {
    std::vector<MPStep> sv{s};
    DevBuf<MPStep> ds = to_device(sv, st);
    DevBuf<Blk> db = to_device(bl, st);
    DevBuf<double2> dm(static_cast<size_t>(std::max<i64>(mat_total, 1))), di(static_cast<size_t>(std::max<i64>(in.size(), 1))),
        dO(static_cast<size_t>(std::max<i64>(o.size(), 1)));
    dm.upload(reinterpret_cast<const double2*>(blocks), static_cast<size_t>(mat_total), st);
    di.upload(reinterpret_cast<const double2*>(t), static_cast<size_t>(in.size()), st);
    launch_mode_product(1, ds.p, o.size(), db.p, dm.p, di.p, dO.p, st);
    dO.download(reinterpret_cast<double2*>(out), static_cast<size_t>(o.size()), st);
    TBF_CUDA(cudaStreamSynchronize(st));
  }
  cudaStreamDestroy(st);
  CAPI_END
}

int oiobf_column_id_batch(int64_t batch, const int64_t* m, const int64_t* n, const int64_t* a_off, const double* A,
                          double tol, const int64_t* max_rank, int64_t* rank, const int64_t* s_off, int64_t* skel,
                          const int64_t* i_off, double* interp, int64_t* perm, int32_t* saturated,
                          double* interp_max_abs) {
  CAPI_BEGIN
  require(batch >= 0, "column_id: negative batch");
  require(tol > 0 && tol < 1, "column_id: tolerance must be in (0,1)");
  if (batch == 0) return OIOBF_OK;
  ensure_device();
  i64 wmax = 1, mmax = 1, atot = 0;
  for (i64 b = 0; b < batch; ++b) {
    require(m[b] > 0 && n[b] > 0, "column_id: empty matrix");
    require(n[b] <= kMaxW, "column_id: more than 96 columns not supported by the device kernel");
    wmax = std::max<i64>(wmax, n[b]);
    mmax = std::max<i64>(mmax, m[b]);
    atot = std::max<i64>(atot, a_off[b] + m[b] * n[b]);
  }
  cudaStream_t st;
  TBF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  {
    LevelDesc L{};
    L.d = 1;
    L.nslots = batch;
    L.wmax = wmax;
    L.m = mmax;
    L.pr = wmax <= 16 ? 256 : wmax <= 32 ? 128 : wmax <= 64 ? 64 : 32;
    if (const char* e = std::getenv("OIOBF_ID_PR")) L.pr = std::atoi(e);  // debug override
    i64 parts = std::max<i64>(1, (148 * 8 + batch - 1) / batch);
    parts = std::min(parts, std::max<i64>(1, (mmax + 4 * L.pr - 1) / (4 * L.pr)));
    if (const char* e = std::getenv("OIOBF_ID_NPARTS")) parts = std::atoi(e);  // debug override
    L.nparts = parts;
    L.rpp = (mmax + parts - 1) / parts;
    std::vector<int> hw(static_cast<size_t>(batch)), ht(static_cast<size_t>(batch * wmax));
    std::vector<i64> hm(m, m + batch), hoff(a_off, a_off + batch), hmr(static_cast<size_t>(batch));
    std::vector<int> hn(static_cast<size_t>(batch));
    for (i64 b = 0; b < batch; ++b) {
      hw[static_cast<size_t>(b)] = static_cast<int>(n[b]);
      hn[static_cast<size_t>(b)] = static_cast<int>(n[b]);
      hmr[static_cast<size_t>(b)] = max_rank ? max_rank[b] : -1;
      for (i64 c = 0; c < n[b]; ++c) ht[static_cast<size_t>(b * wmax + c)] = static_cast<int>(c + 1);
    }
    DevBuf<int> dw = to_device(hw, st), dt = to_device(ht, st), dn = to_device(hn, st);
    DevBuf<i64> dm = to_device(hm, st), doff = to_device(hoff, st), dmr = to_device(hmr, st);
    DevBuf<double2> dA(static_cast<size_t>(atot));
    dA.upload(reinterpret_cast<const double2*>(A), static_cast<size_t>(atot), st);
    DevBuf<double2> rpart(static_cast<size_t>(batch * L.nparts * wmax * wmax));
    launch_matrix_ids(batch, doff.p, dm.p, dn.p, dA.p, L.nparts, L.rpp, L.pr, wmax, rpart.p, st);
    DevBuf<int> drank(static_cast<size_t>(batch)), dsat(static_cast<size_t>(batch)),
        dperm(static_cast<size_t>(batch * wmax)), dsk(static_cast<size_t>(batch * wmax));
    DevBuf<double2> dint(static_cast<size_t>(batch * wmax * wmax));
    DevBuf<double> dgap(static_cast<size_t>(batch));
    launch_finish_var(L, dm.p, tol, kTieEps, dmr.p, rpart.p, dt.p, dw.p, drank.p, dsat.p, dperm.p, dsk.p, dint.p,
                      dgap.p, st);
    std::vector<int> hr(static_cast<size_t>(batch)), hs(static_cast<size_t>(batch)),
        hp(static_cast<size_t>(batch * wmax)), hk(static_cast<size_t>(batch * wmax));
    std::vector<double2> hi(static_cast<size_t>(batch * wmax * wmax));
    drank.download(hr.data(), hr.size(), st);
    dsat.download(hs.data(), hs.size(), st);
    dperm.download(hp.data(), hp.size(), st);
    dsk.download(hk.data(), hk.size(), st);
    dint.download(hi.data(), hi.size(), st);
    TBF_CUDA(cudaStreamSynchronize(st));
    for (i64 b = 0; b < batch; ++b) {
      const int r = hr[static_cast<size_t>(b)];
      const i64 w = n[b];
      rank[b] = r;
      if (saturated) saturated[b] = hs[static_cast<size_t>(b)];
      double mx = 0;
      for (i64 q = 0; q < r * w; ++q) {
        const double2 v = hi[static_cast<size_t>(b * wmax * wmax + q)];
        interp[2 * (i_off[b] + q)] = v.x;
        interp[2 * (i_off[b] + q) + 1] = v.y;
        mx = std::max(mx, std::sqrt(v.x * v.x + v.y * v.y));
      }
      if (interp_max_abs) interp_max_abs[b] = (r > 0) ? mx : 0.0;
      for (int q = 0; q < r; ++q) skel[s_off[b] + q] = hk[static_cast<size_t>(b * wmax + q)];
      if (perm)
        for (i64 q = 0; q < w; ++q) perm[s_off[b] + q] = hp[static_cast<size_t>(b * wmax + q)];
    }
  }
  cudaStreamDestroy(st);
  CAPI_END
}

}  // extern "C"
