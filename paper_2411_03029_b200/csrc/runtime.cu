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
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <queue>
#include <tuple>
#include <string>
#include <vector>

#include "kernels.h"

namespace tbf {
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

// Device buffer.  alloc(): cudaMalloc / cudaFree (long-lived arrays).
// alloc_on(stream): stream-ordered cudaMallocAsync / cudaFreeAsync from the
// device pool (per-level construction temporaries: no device-wide sync on
// free, and the pool keeps the memory for the next level).
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t ast = nullptr;  // set: stream-ordered allocation
  bool async = false;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(size_t count, cudaStream_t st) { alloc_on(count, st); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), ast(o.ast), async(o.async) {
    o.p = nullptr;
    o.n = 0;
    o.async = false;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      reset();
      p = o.p;
      n = o.n;
      ast = o.ast;
      async = o.async;
      o.p = nullptr;
      o.n = 0;
      o.async = false;
    }
    return *this;
  }
  ~DevBuf() { reset(); }
  void alloc(size_t count) {
    reset();
    n = count;
    if (count) TBF_CUDA(cudaMalloc(&p, sizeof(T) * count));
  }
  void alloc_on(size_t count, cudaStream_t st) {
    reset();
    n = count;
    ast = st;
    async = true;
    if (count) TBF_CUDA(cudaMallocAsync(&p, sizeof(T) * count, st));
  }
  void reset() {
    if (p) {
      if (async) cudaFreeAsync(p, ast);
      else cudaFree(p);
    }
    p = nullptr;
    n = 0;
    async = false;
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

// Host bookkeeping at config-4 scale (2e8 slots, 1.7e7 pairs) is dominated by
// serial first-touch of multi-GB arrays: loops over them run on a few host
// threads, chunked.
template <class F>
void parallel_chunks(size_t n, F&& fn) {  // fn(chunk index, begin, end), chunks in order
  static const size_t nt = std::max<size_t>(1, std::min<size_t>(16, std::thread::hardware_concurrency()));
  const size_t nc = n < (size_t{1} << 16) ? 1 : nt;
  if (nc == 1) {
    fn(size_t{0}, size_t{0}, n);
    return;
  }
  std::vector<std::thread> th;
  for (size_t c = 0; c < nc; ++c) th.emplace_back([&, c] { fn(c, n * c / nc, n * (c + 1) / nc); });
  for (auto& t : th) t.join();
}
size_t parallel_nchunks(size_t n) {
  static const size_t nt = std::max<size_t>(1, std::min<size_t>(16, std::thread::hardware_concurrency()));
  return n < (size_t{1} << 16) ? 1 : nt;
}

// std::vector-like host array whose resize does NOT value-initialise (the
// contents are overwritten right after); pages are first touched in parallel.
template <class T>
class HostArray {
  std::unique_ptr<T[]> p_;
  size_t n_ = 0;

 public:
  void resize(size_t n) {
    if (n == n_) return;
    p_.reset(n ? new T[n] : nullptr);  // default-initialised (trivial T: untouched)
    n_ = n;
    char* b = reinterpret_cast<char*>(p_.get());
    parallel_chunks(n * sizeof(T), [&](size_t, size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; i += 4096) b[i] = 0;  // fault the pages in from several threads
    });
  }
  void assign(size_t n, const T& v) {
    resize(n);
    parallel_chunks(n, [&](size_t, size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; ++i) p_[i] = v;
    });
  }
  T* data() { return p_.get(); }
  const T* data() const { return p_.get(); }
  size_t size() const { return n_; }
  bool empty() const { return n_ == 0; }
  T& operator[](size_t i) { return p_[i]; }
  const T& operator[](size_t i) const { return p_[i]; }
  T* begin() { return p_.get(); }
  T* end() { return p_.get() + n_; }
  const T* begin() const { return p_.get(); }
  const T* end() const { return p_.get() + n_; }
};

template <class T>
DevBuf<T> to_device(const HostArray<T>& v, cudaStream_t st) {
  DevBuf<T> b(v.size());
  b.upload(v.data(), v.size(), st);
  return b;
}

i64 ipow(i64 b, i64 e) {
  i64 r = 1;
  while (e-- > 0) r *= b;
  return r;
}

void keep_pool_memory(int dev) {  // freed stream-ordered memory stays cached in the pool
  static bool done[64] = {};
  if (dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ULL;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

void ensure_device() {
  int cnt = 0;
  cudaError_t e = cudaGetDeviceCount(&cnt);
  if (e != cudaSuccess || cnt == 0)
    throw std::runtime_error("no CUDA device available (the B200 path has no CPU fallback)");
  TBF_CUDA(cudaSetDevice(g_device));
  static int checked[64] = {};  // 1: sm_100-class (cudaGetDeviceProperties is slow; query once)
  if (g_device < 0 || g_device >= 64 || !checked[g_device]) {
    int major = 0;
    TBF_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, g_device));
    if (major < 10) throw std::runtime_error("device is not sm_100-class (Blackwell) — this build targets sm_100a");
    if (g_device >= 0 && g_device < 64) checked[g_device] = 1;
  }
  keep_pool_memory(g_device);
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
  HostArray<int> h_rank, h_width, h_sat;
  HostArray<i64> h_skel_off, h_interp_off;
  i64 total_skel = 0, total_interp = 0;
  int max_rank = 0;
};

struct TRef {
  i64 off = 0;
  int nd = 0;
  int nsum = 1;         // > 1: ordered sum of nsum tensors at off + c * sum_stride
  i64 sum_stride = 0;
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
  i64 begin, n, total;  // descriptors [begin, begin + n), total output elements
};
struct BoxLaunch {
  int side, level, in_buf, out_buf;
  i64 item_begin, nitems;
  BoxLaunchInfo info;
  int box2 = 0;       // d = 2 GEMM kernel (k_box2), one CTA per box
  size_t smem2 = 0;
};
struct Op {
  int kind;  // 0 mode product, 1 gemv, 2 ordered child sums, 3 fused boxes, 6 tiny level, 7 tiny gemv, 8 rank-one level
  i64 idx;
  int group;  // 0 V/W, 1 core, 2 P/U
  int chunk = 0;  // pipelined plans: slab group (outer index of mode d-1)
};
// one core-GEMV launch (all pairs, or the pairs of one column-slab group)
struct GemvLaunch {
  i64 desc_begin = 0, ndesc = 0;
  i64 total_rows = 0, ctas = 0;
  i64 map_begin = 0;  // into Plan::gemv_map (CTA -> pair, relative to desc_begin)
  i64 rb_begin = 0;   // into Plan::gemv_rb (CTA row ranges, ctas + 1 entries)
  int max_c = 0;
  bool tma = false;
  i64 tma_ctas = 0, tma_map_begin = 0, tma_rb_begin = 0;
  int tma_stages = 0, tma_stage_elems = 0, tma_xcap = 0;
};

// one in-flight slot of the stream-ordered host-buffer contraction
// (contract_host_async): device staging, its captured compute graph, and the
// events that order reuse of the slot against the previous call that used it
struct AsyncSet {
  DevBuf<double2> F, G, scratch;  // own scratch: the two slots' contractions may overlap
  cudaEvent_t in = nullptr, done = nullptr, out = nullptr;  // H2D landed / compute done / D2H done
  cudaEvent_t user = nullptr;  // the caller's stream at the call: G's previous readers are done
  cudaGraphExec_t gexec = nullptr;
  bool used = false;
  ~AsyncSet() {
    if (gexec) cudaGraphExecDestroy(gexec);
    for (cudaEvent_t e : {in, done, out, user})
      if (e) cudaEventDestroy(e);
  }
};

struct Plan {
  i64 nv = 0;
  i64 scratch_elems = 0;
  bool bfp = false;  // core GEMV on the block-floating-point cores (n_v = 1)
  std::vector<MPStep> steps;
  std::vector<Blk> blks;
  std::vector<MPLaunch> mps;
  int nchunk = 1;  // > 1: host-pipelined plan (ops tagged by slab group)
  // tiny-box engine (tiny_kernels.cu): one launch per level + a row GEMV
  struct TinyLevel {
    int side, l, in_buf, out_buf;
    i64 group_begin, off_begin;
    TinyLevelArgs args;
  };
  std::vector<TinyLevel> tiny_levels;
  std::vector<TinyGroup> tiny_groups;
  std::vector<i64> tiny_off;  // per level: child output (V/W) / input (P/U) offsets by (outer, inner)
  DevBuf<TinyGroup> d_tiny_groups;
  DevBuf<i64> d_tiny_off;
  // rank-one engine (r1_kernels.cu): one launch per level, ping-pong scratch
  struct R1Level {
    R1LevelArgs args;
    i64 in_off, out_off;  // scratch element offsets; -1: F (input) / G (output)
  };
  std::vector<R1Level> r1_levels;
  DevBuf<int> d_r1_own;                      // sharded: local -> middle multi-set
  DevBuf<i64> d_r1_send_off, d_r1_recv_off;  // sharded: exchange offsets per pair t * nmid + s
  std::vector<GemvDesc> gemv;
  std::vector<GemvLaunch> gemvs;
  std::vector<int> gemv_map, tma_map;
  std::vector<i64> gemv_rb;  // CTA row ranges of every GEMV launch (both variants)
  DevBuf<int> d_tma_map;
  DevBuf<i64> d_gemv_rb;
  std::vector<SumDesc> sums;
  std::vector<SumLaunch> sum_launches;
  std::vector<Op> ops;
  std::vector<BoxDesc> bdescs;
  std::vector<BoxLaunch> boxes;
  DevBuf<BoxDesc> d_bdescs;
  DevBuf<MPStep> d_steps;
  DevBuf<Blk> d_blks;
  DevBuf<GemvDesc> d_gemv;
  DevBuf<int> d_gemv_map;  // CTA -> pair (per launch, relative to its first pair)
  DevBuf<SumDesc> d_sums;
  DevBuf<double2> scratch;
  DevBuf<double2> stage_F, stage_G;  // host-buffer contract staging
  i64 gemv_y_base = 0;
  // sharded plans (world > 1): phase 1 = V/W + GEMV (writes the send buffer),
  // phase 2 = P/U (reads the receive buffer)
  bool sharded = false;
  // stream-ordered host-buffer contraction: two slots, used alternately
  AsyncSet aset[2];
  int anext = 0;
  // captured graphs keyed by their buffers (device path: F, G, stream;
  // host pipeline: F, G), a few of each so alternating buffers (vector groups
  // of a wide n_v, ping-pong callers) replay instead of re-capturing
  struct GraphCache {
    struct Entry {
      const void* F;
      const void* G;
      cudaStream_t st;
      cudaGraphExec_t ex;
    };
    std::vector<Entry> e;
    size_t cap = 16;  // raised to the vector-chunk count for wide n_v (no re-capture per call)
    cudaGraphExec_t find(const void* F, const void* G, cudaStream_t st) const {
      for (const Entry& x : e)
        if (x.F == F && x.G == G && x.st == st) return x.ex;
      return nullptr;
    }
    void put(const void* F, const void* G, cudaStream_t st, cudaGraphExec_t ex) {
      if (e.size() >= cap) {
        cudaGraphExecDestroy(e.front().ex);
        e.erase(e.begin());
      }
      e.push_back(Entry{F, G, st, ex});
    }
    ~GraphCache() {
      for (const Entry& x : e) cudaGraphExecDestroy(x.ex);
    }
  };
  GraphCache dev_graphs, host_graphs;
  GraphCache phase_graphs[2];  // sharded phases 1 / 2, keyed by (input, output, stream)
  // device-buffer calls share pl.scratch: a call on a different stream than
  // the previous one waits for it (same-stream calls are ordered already)
  cudaEvent_t dev_done = nullptr;
  cudaStream_t dev_last = nullptr;
  bool dev_used = false;
  ~Plan() {
    if (dev_done) cudaEventDestroy(dev_done);
  }
};

// Fill a GemvLaunch for descs [begin, end) of pl.gemv: persistent balanced
// grid for the register-streaming kernel, and the TMA-ring parameters when
// they apply.  cta_off of the descriptors is relative to the launch.
// Byte-balanced row split of descs [begin, end) over nct CTAs: CTA c gets
// rows [rb[c], rb[c+1]) holding ~1/nct of the core elements (row lengths C
// differ per pair, so equal row counts would leave the long-row CTAs last).
// map[c] = pair (relative to begin) holding CTA c's first row.  Returns the
// largest number of pairs any CTA touches.
int split_rows(const Plan& pl, i64 begin, i64 end, i64 nct, std::vector<i64>& rb, std::vector<int>& map) {
  // cost of a row = its C elements + a fixed per-row overhead (warp reduction,
  // row setup, the dependent load batches of one warp), in element units.
  // Measured on B200: config 2 (C ~ 64..1000) graph 89.5 us at K = 0, ~85 us
  // for K in [128, 1024]; config 5 (C ~ 256..2400) GEMV 14.2 ms at K = 0,
  // 14.4 ms at K = 256, 15.7 ms at K = 1024, 19.1 ms row-balanced.
  // OIOBF_GEMV_ROW_COST overrides.
  static const i64 K = std::getenv("OIOBF_GEMV_ROW_COST") ? std::atoll(std::getenv("OIOBF_GEMV_ROW_COST")) : 256;
  auto cost = [&](i64 q) { return static_cast<i64>(pl.gemv[static_cast<size_t>(q)].C) + K; };
  i64 E = 0;
  for (i64 q = begin; q < end; ++q) E += pl.gemv[static_cast<size_t>(q)].R * cost(q);
  const GemvDesc& last = pl.gemv[static_cast<size_t>(end - 1)];
  const i64 rows = last.cta_off + last.R;
  rb.assign(static_cast<size_t>(nct + 1), rows);
  rb[0] = 0;
  i64 q = begin, before = 0;  // cost before pair q
  for (i64 c = 1; c < nct; ++c) {
    const i64 target = E / nct * c + std::min<i64>(c, E % nct);
    while (q + 1 < end && before + pl.gemv[static_cast<size_t>(q)].R * cost(q) <= target) {
      before += pl.gemv[static_cast<size_t>(q)].R * cost(q);
      ++q;
    }
    const GemvDesc& g = pl.gemv[static_cast<size_t>(q)];
    const i64 r = std::min<i64>(g.R, (target - before + cost(q) - 1) / cost(q));
    rb[static_cast<size_t>(c)] = std::max(rb[static_cast<size_t>(c - 1)], g.cta_off + r);
  }
  map.assign(static_cast<size_t>(nct), 0);
  int maxp = 0;
  size_t p = static_cast<size_t>(begin);
  for (i64 c = 0; c < nct; ++c) {
    const i64 g0 = rb[static_cast<size_t>(c)], g1 = rb[static_cast<size_t>(c + 1)];
    while (p + 1 < static_cast<size_t>(end) && pl.gemv[p + 1].cta_off <= g0) ++p;
    map[static_cast<size_t>(c)] = static_cast<int>(p - static_cast<size_t>(begin));
    size_t p2 = p;
    while (p2 + 1 < static_cast<size_t>(end) && pl.gemv[p2 + 1].cta_off < g1) ++p2;
    if (g1 > g0) maxp = std::max(maxp, static_cast<int>(p2 - p + 1));
  }
  return maxp;
}

// Fill a GemvLaunch for descs [begin, end) of pl.gemv: persistent
// byte-balanced grid for the register-streaming kernel, and the TMA-ring
// parameters when they apply.  cta_off of the descriptors is relative to the
// launch.
void finish_gemv(Plan& pl, i64 begin, i64 end, i64 nv) {
  GemvLaunch gl;
  gl.desc_begin = begin;
  gl.ndesc = end - begin;
  i64 rows = 0;
  for (i64 q = begin; q < end; ++q) {
    GemvDesc& g = pl.gemv[static_cast<size_t>(q)];
    g.cta_off = rows;
    rows += g.R;
    gl.max_c = std::max(gl.max_c, g.C);
  }
  gl.total_rows = rows;
  if (rows == 0) {
    pl.gemvs.push_back(gl);
    return;
  }
  std::vector<i64> rb;
  std::vector<int> map;
  {
    const int per_sm = pl.bfp ? gemv_bfp_ctas_per_sm(std::max(gl.max_c, 1))
                              : gemv_ctas_per_sm(static_cast<int>(nv), std::max(gl.max_c, 1));
    gl.ctas = std::min<i64>(static_cast<i64>(148) * per_sm, rows);
    split_rows(pl, begin, end, gl.ctas, rb, map);
    gl.map_begin = static_cast<i64>(pl.gemv_map.size());
    gl.rb_begin = static_cast<i64>(pl.gemv_rb.size());
    pl.gemv_map.insert(pl.gemv_map.end(), map.begin(), map.end());
    pl.gemv_rb.insert(pl.gemv_rb.end(), rb.begin(), rb.end());
  }
  // TMA bulk-copy pipeline: one persistent CTA per SM, whole rows staged in a
  // shared-memory ring; used when rows are long enough to be worth a bulk
  // copy and every CTA's row range touches <= gemv_tma_max_pairs() pairs.
  static const bool no_tma = std::getenv("OIOBF_GEMV_NO_TMA") != nullptr;
  static const int per_sm_env =
      std::getenv("OIOBF_TMA_CTAS_PER_SM") ? std::atoi(std::getenv("OIOBF_TMA_CTAS_PER_SM")) : 2;
  static const int stages_env = std::getenv("OIOBF_TMA_STAGES") ? std::atoi(std::getenv("OIOBF_TMA_STAGES")) : 8;
  if (!no_tma && !pl.bfp && gl.max_c >= 64) {
    const i64 grid = std::min<i64>(148 * std::max(1, per_sm_env), rows);
    const int stage_elems = (gl.max_c + 7) / 8 * 8;
    const int xcap = gl.max_c * static_cast<int>(nv);
    const i64 avail = static_cast<i64>(kMaxDynSmem) / std::max(1, per_sm_env) - 1024 -
                      static_cast<i64>(gemv_tma_max_pairs()) * xcap * static_cast<i64>(sizeof(double2));
    // rows go round-robin to the 8 consumer warps, so each stage must always
    // belong to the same consumer (stages % 8 == 0); otherwise a consumer
    // could wait two phases ahead and the parity check would be ambiguous
    i64 stages = std::min<i64>(stages_env, avail / (static_cast<i64>(stage_elems) * 16));
    stages = stages / 8 * 8;
    bool ok = stages >= 8;
    std::vector<i64> rb2;
    std::vector<int> map2;
    if (ok) ok = split_rows(pl, begin, end, grid, rb2, map2) <= gemv_tma_max_pairs();
    if (std::getenv("OIOBF_DEBUG"))
      fprintf(stderr, "[oiobf] gemv tma ok=%d grid=%lld stages=%lld stage_elems=%d xcap=%d rows=%lld\n", ok ? 1 : 0,
              grid, stages, stage_elems, xcap, rows);
    if (ok) {
      gl.tma = true;
      gl.tma_ctas = grid;
      gl.tma_stages = static_cast<int>(stages);
      gl.tma_stage_elems = stage_elems;
      gl.tma_xcap = xcap;
      gl.tma_map_begin = static_cast<i64>(pl.tma_map.size());
      gl.tma_rb_begin = static_cast<i64>(pl.gemv_rb.size());
      pl.tma_map.insert(pl.tma_map.end(), map2.begin(), map2.end());
      pl.gemv_rb.insert(pl.gemv_rb.end(), rb2.begin(), rb2.end());
    }
  }
  pl.gemvs.push_back(gl);
}

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
  // sharding: this rank owns the middle multi-sets o with
  // owner_of(o) == rank on both sides -- o % world by default, or the map set
  // by oiobf_tbf_shard_set_owners (byte-balanced ownership)
  int rank = 0, world = 1;
  std::vector<int> owner;  // empty: round-robin
  DevBuf<int> d_owner;
  int owner_of(i64 outer) const {
    return owner.empty() ? static_cast<int>(outer % world) : owner[static_cast<size_t>(outer)];
  }
  bool owns(i64 outer) const { return world <= 1 || owner_of(outer) == rank; }
  // U-side middle-level (l = Lc) ranks / skeletons of ALL t (gathered from the
  // other ranks) -- the row skeletons of the cores of the owned pairs (t, s)
  std::vector<int> umid_rank;
  std::vector<i64> umid_skel_off;
  DevBuf<int> umid_skel;
  // exchange tables (element offsets per pair t*nmid+s, nv = 1 units), -1 = none
  std::vector<i64> send_off, recv_off;
  i64 send_elems = 0, recv_elems = 0;
  // fused exchange: phase-1 GEMV stores into the owners' receive buffers
  std::vector<i64> peer_off;        // per pair (t * nmid + s): offset in the owner's buffer (nv = 1)
  std::vector<u64> peer_base;       // [parity * world + q]: receive buffer addresses
  i64 peer_nv_max = 0;
  bool peer_mode() const { return !peer_base.empty(); }
  std::vector<LevelData> side[2];
  std::vector<i64> r_est[2];
  DevBuf<double2> cores;
  HostArray<PairDesc> h_pairs;
  // block-floating-point copy of the cores (oiobf_tbf_set_core_format 1):
  // pair p's blocks at bfp_off[p] (entries), exponents at bfp_off[p] / 32
  int core_format = 0;
  DevBuf<int2> bfp_q;
  DevBuf<short> bfp_e;
  std::vector<i64> bfp_off;
  i64 bfp_entries = 0;
  i64 total_core = 0;
  std::map<i64, std::unique_ptr<Plan>> plans;
  int apply_engine = 0;  // 0 auto, 1 box engine, 2 tiny-box engine, 4 rank-one engine
  int tiny_auto = -1;    // cached auto decision (-1: not evaluated yet)
  int r1_ok = -1;        // cached rank-one eligibility (-1: not evaluated yet)
  double t_ms[6] = {0, 0, 0, 0, 0, 0};
  std::mutex mu;
  // construction: the V/W and U/P sides are independent until the cores, so
  // they build concurrently (one host thread and one stream each); their
  // phase timers accumulate under t_mu
  cudaStream_t sstream[2] = {nullptr, nullptr};
  std::mutex t_mu;
  cudaStream_t side_stream(int sd) const { return sstream[sd] ? sstream[sd] : stream; }
  void add_ms(int i, double v) {
    std::lock_guard<std::mutex> lk(t_mu);
    t_ms[i] += v;
  }
  // host-buffer contraction pipeline: copy-in / copy-out streams and the
  // events that order them against the compute stream (created on first use)
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaStream_t s_cmp[2] = {nullptr, nullptr};  // compute streams of the two async slots
  std::vector<cudaEvent_t> ev;
  // every stream of the handle idle (before plans and their buffers go away)
  void sync_all() {
    for (cudaStream_t x : {stream, s_in, s_out, s_cmp[0], s_cmp[1]})
      if (x) cudaStreamSynchronize(x);
  }
  ~oiobf_tbf() {
    sync_all();
    plans.clear();
    for (cudaStream_t x : {s_cmp[0], s_cmp[1]})
      if (x) cudaStreamDestroy(x);
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
    for (cudaStream_t x : sstream)
      if (x) cudaStreamDestroy(x);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

constexpr double kTieEps = 1e-12;

int device_sms() {
  static int sms[64] = {0};
  const int dv = g_device >= 0 && g_device < 64 ? g_device : 0;
  if (!sms[dv]) TBF_CUDA(cudaDeviceGetAttribute(&sms[dv], cudaDevAttrMultiProcessorCount, g_device));
  return sms[dv];
}

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
      require(b.n <= (kMaxDynSmem - 16) / 5 || counts[p] <= kMaxProxy || b.strat.mode != OIOBF_PROXY_UNIFORM_RANDOM,
              "proxy count per mode above 64 needs an extent that fits the shared-memory pool");
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
  // R packed: (w(w+1)/2 + pr w) x 16 B fits the 220 KB budget; taller panels
  // amortise the per-column steps (w <= 24 at 256 rows: 2 CTAs/SM, config 2
  // panel time 32.1 -> 28.2 ms against 128 rows at 3 CTAs/SM)
  int cps = 1;
  panel_shape(wmax, L.psize, &L.pr, &cps);
  L.rank = b.rank;
  L.world = b.world;
  L.owner = b.owner.empty() ? nullptr : b.d_owner.p;
  // >= 4 waves of resident CTAs, each CTA >= 4 panels
  const i64 target_ctas = static_cast<i64>(device_sms()) * cps * 4;
  const i64 owned = (L.nslots + b.world - 1) / b.world;
  i64 parts = (target_ctas + owned - 1) / owned;
  const i64 max_parts = std::max<i64>(1, (L.m + 4 * L.pr - 1) / (4 * L.pr));  // >= 4 panels per part
  parts = std::max<i64>(1, std::min(parts, max_parts));
  L.nparts = parts;
  L.rpp = (L.m + parts - 1) / parts;
  return L;
}

void finish_level(oiobf_tbf& b, LevelData& ld, DevBuf<int>& sat, DevBuf<int>& skel_tmp, DevBuf<double2>& interp_tmp);

void build_side_level(oiobf_tbf& b, int sd, int l, i64 r_est) {
  cudaStream_t st = b.side_stream(sd);
  const int d = b.d;
  // widest candidate set: leaf size (l=0) or max r(child0)+r(child1)
  i64 wmax;
  if (l == 0) {
    wmax = b.n >> b.L;
  } else {
    const LevelData& c = b.side[sd][static_cast<size_t>(l - 1)];
    LevelDesc tmp = make_level(b, sd, l, r_est, 1);
    if (tmp.nslots > (i64{1} << 22)) {
      wmax = 2 * static_cast<i64>(c.max_rank);  // bound (exact scan too slow at ~1e8 slots)
    } else {
      wmax = 0;
      for (i64 idx = 0; idx < tmp.nslots; ++idx) {
        const SlotPos s = decode_slot(tmp, idx);
        const i64 w = c.h_rank[static_cast<size_t>(child_slot(tmp, s, 0))] +
                      c.h_rank[static_cast<size_t>(child_slot(tmp, s, 1))];
        wmax = std::max(wmax, w);
      }
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
  static const bool no_narrow = std::getenv("OIOBF_NO_NARROW") != nullptr;
  if (b.ks.kind == OIOBF_KERNEL_DFT && wmax <= 2 && !no_narrow) {
    // closed-form narrow IDs (k_narrow_dft): no proxy / panel / R buffers
    ld.width.alloc(static_cast<size_t>(ns));
    ld.rank.alloc(static_cast<size_t>(ns));
    DevBuf<int> sat(static_cast<size_t>(ns), st);
    ld.perm.alloc(static_cast<size_t>(ns * wmax));
    ld.gaps.alloc(static_cast<size_t>(ns));
    DevBuf<int> skel_tmp(static_cast<size_t>(ns * wmax), st);
    DevBuf<double2> interp_tmp(static_cast<size_t>(ns * wmax * wmax), st);
    EventTimer t2(st);
    const LevelData* c = l > 0 ? &b.side[sd][static_cast<size_t>(l - 1)] : nullptr;
    launch_narrow_dft(L, b.ks, b.tol, c ? c->rank.p : nullptr, c ? c->skel_off.p : nullptr, c ? c->skel.p : nullptr,
                      ld.width.p, ld.rank.p, sat.p, ld.perm.p, skel_tmp.p, interp_tmp.p, ld.gaps.p, st);
    b.add_ms(2, t2.stop());
    finish_level(b, ld, sat, skel_tmp, interp_tmp);
    return;
  }
  DevBuf<int> proxies(static_cast<size_t>(ns * L.psize), st);
  DevBuf<int> targets(static_cast<size_t>(ns * wmax), st);
  ld.width.alloc(static_cast<size_t>(ns));
  EventTimer t0(st);
  launch_gen_proxies(L, proxies.p, st);
  if (l == 0) {
    launch_targets(L, nullptr, nullptr, nullptr, targets.p, ld.width.p, st);
  } else {
    const LevelData& c = b.side[sd][static_cast<size_t>(l - 1)];
    launch_targets(L, c.rank.p, c.skel_off.p, c.skel.p, targets.p, ld.width.p, st);
  }
  b.add_ms(0, t0.stop());
  DevBuf<double2> rpart(static_cast<size_t>(ns * L.nparts * wmax * wmax), st);
  EventTimer t1(st);
  launch_panel(L, b.ks, proxies.p, targets.p, ld.width.p, rpart.p, st);
  b.add_ms(1, t1.stop());
  ld.rank.alloc(static_cast<size_t>(ns));
  DevBuf<int> sat(static_cast<size_t>(ns), st);
  ld.perm.alloc(static_cast<size_t>(ns * wmax));
  ld.gaps.alloc(static_cast<size_t>(ns));
  DevBuf<int> skel_tmp(static_cast<size_t>(ns * wmax), st);
  DevBuf<double2> interp_tmp(static_cast<size_t>(ns * wmax * wmax), st);
  EventTimer t2(st);
  launch_finish(L, b.tol, kTieEps, -1, rpart.p, targets.p, ld.width.p, ld.rank.p, sat.p, ld.perm.p, skel_tmp.p,
                interp_tmp.p, ld.gaps.p, st);
  b.add_ms(2, t2.stop());
  finish_level(b, ld, sat, skel_tmp, interp_tmp);
}

// Host-side bookkeeping after a level's IDs: ranks / widths to the host, skeleton
// and interp offsets, compaction of the per-slot scratch into the level arrays.
void finish_level(oiobf_tbf& b, LevelData& ld, DevBuf<int>& sat, DevBuf<int>& skel_tmp, DevBuf<double2>& interp_tmp) {
  cudaStream_t st = b.side_stream(ld.L.side);
  const i64 ns = ld.nslots;
  const i64 wmax = ld.L.wmax;
  static const bool dbg = std::getenv("OIOBF_DEBUG") != nullptr;
  auto tnow = [] { return std::chrono::steady_clock::now(); };
  auto tms = [](auto a, auto c) { return std::chrono::duration<double, std::milli>(c - a).count(); };
  TBF_CUDA(cudaStreamSynchronize(st));
  const auto f0 = tnow();
  ld.h_rank.resize(static_cast<size_t>(ns));
  ld.h_width.resize(static_cast<size_t>(ns));
  ld.h_sat.resize(static_cast<size_t>(ns));
  ld.rank.download(ld.h_rank.data(), static_cast<size_t>(ns), st);
  ld.width.download(ld.h_width.data(), static_cast<size_t>(ns), st);
  sat.download(ld.h_sat.data(), static_cast<size_t>(ns), st);
  TBF_CUDA(cudaStreamSynchronize(st));
  const auto f1 = tnow();
  ld.h_skel_off.resize(static_cast<size_t>(ns));
  ld.h_interp_off.resize(static_cast<size_t>(ns));
  // exclusive prefix sums of rank and rank * width: chunk totals, then chunk scans
  const size_t nck = parallel_nchunks(static_cast<size_t>(ns));
  std::vector<i64> cso(nck + 1, 0), cio(nck + 1, 0);
  std::vector<int> cmr(nck, 0);
  parallel_chunks(static_cast<size_t>(ns), [&](size_t c, size_t lo, size_t hi) {
    i64 a = 0, bb = 0;
    int mr = 0;
    for (size_t i = lo; i < hi; ++i) {
      a += ld.h_rank[i];
      bb += static_cast<i64>(ld.h_rank[i]) * ld.h_width[i];
      mr = std::max(mr, ld.h_rank[i]);
    }
    cso[c + 1] = a;
    cio[c + 1] = bb;
    cmr[c] = mr;
  });
  ld.max_rank = 0;
  for (size_t c = 0; c < nck; ++c) {
    cso[c + 1] += cso[c];
    cio[c + 1] += cio[c];
    ld.max_rank = std::max(ld.max_rank, cmr[c]);
  }
  parallel_chunks(static_cast<size_t>(ns), [&](size_t c, size_t lo, size_t hi) {
    i64 a = cso[c], bb = cio[c];
    for (size_t i = lo; i < hi; ++i) {
      ld.h_skel_off[i] = a;
      ld.h_interp_off[i] = bb;
      a += ld.h_rank[i];
      bb += static_cast<i64>(ld.h_rank[i]) * ld.h_width[i];
    }
  });
  const i64 so = cso[nck], io = cio[nck];
  ld.total_skel = so;
  ld.total_interp = io;
  const auto f2 = tnow();
  EventTimer t3(st);
  // the device offsets are scanned on the device (same integers as the host mirror)
  ld.skel_off.alloc(static_cast<size_t>(ns));
  ld.interp_off.alloc(static_cast<size_t>(ns));
  scan_slot_offsets(ns, ld.rank.p, ld.width.p, ld.skel_off.p, ld.interp_off.p, st);
  if (dbg) {
    TBF_CUDA(cudaStreamSynchronize(st));
    fprintf(stderr, "[oiobf] finish_level %lld slots: download %.1f ms, prefix %.1f ms, upload %.1f ms\n", ns,
            tms(f0, f1), tms(f1, f2), tms(f2, tnow()));
  }
  ld.skel.alloc(static_cast<size_t>(std::max<i64>(so, 1)));
  ld.interp.alloc(static_cast<size_t>(std::max<i64>(io, 1)));
  launch_compact(ns, wmax, ld.rank.p, ld.width.p, ld.skel_off.p, ld.interp_off.p, skel_tmp.p, interp_tmp.p, ld.skel.p,
                 ld.interp.p, st);
  b.add_ms(3, t3.stop());
  // saturation would trigger the doubling retry (id.cpp:256-269); with the
  // default rank limit it is unreachable, so it is only reported.
}

// Cores K(tbar, sbar) of the pairs (t, s) whose s this rank owns (all pairs
// when world == 1).  Row skeletons come from the U side at level Lc -- local
// when world == 1, gathered from every rank (umid_*) otherwise.
// Pair layout (R, C, ranks, skeleton offsets, arena offsets) of every middle
// pair; returns the core arena size.  Shared by construction and TBF1 load.
i64 layout_pairs(oiobf_tbf& b) {
  const int d = b.d;
  const LevelData& U = b.side[1][static_cast<size_t>(b.Lc)];
  const LevelData& V = b.side[0][static_cast<size_t>(b.Lc)];
  const bool gathered = b.world > 1;
  const int* urank = gathered ? b.umid_rank.data() : U.h_rank.data();
  const i64* uskel_off = gathered ? b.umid_skel_off.data() : U.h_skel_off.data();
  const i64 P = b.nmid * b.nmid;
  b.h_pairs.assign(static_cast<size_t>(P), PairDesc{});
  // per-pair geometry in parallel chunks, then the arena offsets (exclusive
  // prefix of R * C) from chunk totals
  const size_t nck = parallel_nchunks(static_cast<size_t>(P));
  std::vector<i64> ctot(nck + 1, 0);
  parallel_chunks(static_cast<size_t>(P), [&](size_t c, size_t lo, size_t hi) {
    i64 sum = 0;
    for (size_t pp = lo; pp < hi; ++pp) {
      const i64 p = static_cast<i64>(pp);
      const i64 s = p / b.nmid, t = p % b.nmid;
      PairDesc& pd = b.h_pairs[pp];
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
      sum += static_cast<i64>(pd.R) * pd.C;
    }
    ctot[c + 1] = sum;
  });
  for (size_t c = 0; c < nck; ++c) ctot[c + 1] += ctot[c];
  parallel_chunks(static_cast<size_t>(P), [&](size_t c, size_t lo, size_t hi) {
    i64 o = ctot[c];
    for (size_t pp = lo; pp < hi; ++pp) {
      PairDesc& pd = b.h_pairs[pp];
      pd.core_off = o;
      pd.work_off = o;
      o += static_cast<i64>(pd.R) * pd.C;
    }
  });
  const i64 off = ctot[nck];
  b.total_core = off;
  return off;
}

void build_cores(oiobf_tbf& b) {
  cudaStream_t st = b.stream;
  const LevelData& U = b.side[1][static_cast<size_t>(b.Lc)];
  const LevelData& V = b.side[0][static_cast<size_t>(b.Lc)];
  const bool gathered = b.world > 1;
  const int* uskel = gathered ? b.umid_skel.p : U.skel.p;
  const i64 P = b.nmid * b.nmid;
  static const bool dbg = std::getenv("OIOBF_DEBUG") != nullptr;
  auto tnow = [] { return std::chrono::steady_clock::now(); };
  auto tms = [](auto a, auto c) { return std::chrono::duration<double, std::milli>(c - a).count(); };
  const auto c0 = tnow();
  const i64 off = layout_pairs(b);
  const auto c1 = tnow();
  b.cores.alloc(static_cast<size_t>(std::max<i64>(off, 1)));
  DevBuf<PairDesc> dp;
  if (gathered) {
    dp = to_device(b.h_pairs, st);
  } else {  // same layout computed on the device: no multi-GB upload at config-4 scale
    dp.alloc(static_cast<size_t>(P));
    layout_pairs_device(b.d, b.nmid, U.rank.p, U.skel_off.p, V.rank.p, V.skel_off.p, dp.p, st);
  }
  if (dbg) {
    TBF_CUDA(cudaStreamSynchronize(st));
    fprintf(stderr, "[oiobf] cores: layout %.1f ms, upload %.1f ms (%lld pairs)\n", tms(c0, c1), tms(c1, tnow()), P);
  }
  EventTimer t(st);
  launch_cores(b.ks, P, dp.p, off, uskel, V.skel.p, b.cores.p, st);
  b.t_ms[4] += t.stop();
}

void validate_spec(const oiobf_kernel_spec& s) {
  require(s.d >= 1 && s.d <= kMaxD, "kernel spec: d must be in [1,6]");
  require(s.n >= 1, "kernel spec: n must be positive");
  require(s.kind >= 0 && s.kind <= 4, "make_kernel: unknown kernel kind");
  require(s.kind != OIOBF_KERNEL_RADON2D || s.d == 2, "kernel spec: radon2d needs d=2");
  require(s.kind != OIOBF_KERNEL_RADON3D || s.d == 3, "kernel spec: radon3d needs d=3");
  require(s.kind != OIOBF_KERNEL_NUDFT || !s.bitrev, "kernel spec: nudft has no bit-reversed ordering");
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
  static const bool dbg = std::getenv("OIOBF_DEBUG") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  auto t_begin = now();
  auto b = construct_begin(spec, L, tol, ps, seed, 0, 1);
  auto t_start = now();
  for (int sd = 0; sd < 2; ++sd) TBF_CUDA(cudaStreamCreateWithFlags(&b->sstream[sd], cudaStreamNonBlocking));
  auto build_side = [&](int sd) {
    i64 r_est = 8;
    for (int l = 0; l <= b->Lc; ++l) {
      b->r_est[sd].push_back(r_est);
      auto t0 = now();
      build_side_level(*b, sd, l, r_est);
      if (dbg) fprintf(stderr, "[oiobf] construct side %d level %d: %.2f ms\n", sd, l, ms(t0, now()));
      r_est = std::max<i64>(r_est, b->side[sd][static_cast<size_t>(l)].max_rank);
    }
  };
  static const bool serial = std::getenv("OIOBF_SERIAL_SIDES") != nullptr;  // A/B switch
  if (serial) {
    build_side(0);
    build_side(1);
  } else {  // U/P side on a second host thread (same device, own stream)
    std::exception_ptr err;
    const int dev = g_device;
    std::thread th([&] {
      try {
        g_device = dev;
        TBF_CUDA(cudaSetDevice(dev));
        build_side(1);
      } catch (...) {
        err = std::current_exception();
      }
    });
    try {
      build_side(0);
    } catch (...) {
      th.join();
      throw;
    }
    th.join();
    if (err) std::rethrow_exception(err);
  }
  for (int sd = 0; sd < 2; ++sd) TBF_CUDA(cudaStreamSynchronize(b->sstream[sd]));
  auto t1 = now();
  build_cores(*b);
  TBF_CUDA(cudaStreamSynchronize(b->stream));
  if (dbg) fprintf(stderr, "[oiobf] construct begin %.2f ms, cores %.2f ms\n", ms(t_begin, t_start), ms(t1, now()));
  b->t_ms[5] = ms(t_start, now());
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

std::unique_ptr<Plan> build_plan(oiobf_tbf& b, i64 nv, bool chunked, int parity = 0) {
  auto pl = std::make_unique<Plan>();
  pl->bfp = b.core_format == 1 && nv == 1;
  pl->nv = nv;
  pl->nchunk = chunked && b.world == 1 ? static_cast<int>(ipow(2, b.Lc)) : 1;
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
  // Record one box launch for descs (all of one side/level [/slab group]):
  // CTAs per box, amax bucket, input staging and shared-memory sizes; false
  // when a box does not fit on chip (the caller falls back to mode products).
  auto bl_split1 = [] {
    const char* e3 = std::getenv("OIOBF_BOX_SPLIT1");
    return !(e3 && std::strcmp(e3, "0") == 0);
  };
  auto commit_boxes = [&](std::vector<BoxDesc>& descs, int sd, int l, int in_buf, int out_buf, int transpose,
                          int group) -> bool {
    if (d < 2) return false;
    const int f = d - 1;
    // boxes with an empty output write nothing
    std::vector<BoxDesc> keep;
    for (const BoxDesc& x : descs) {
      bool empty = false;
      for (int k = 0; k < d; ++k) empty |= x.eout[k] == 0;
      if (!empty) keep.push_back(x);
    }
    descs.swap(keep);
    if (descs.empty()) return true;
    int cs_env = std::getenv("OIOBF_BOX_SPLIT") ? std::atoi(std::getenv("OIOBF_BOX_SPLIT")) : 0;
    // per-launch override for experiments: OIOBF_BOX_SPLIT_AT="side:level:cs"
    if (const char* e = std::getenv("OIOBF_BOX_SPLIT_AT")) {
      int es = -1, el = -1, ec = 0;
      if (std::sscanf(e, "%d:%d:%d", &es, &el, &ec) == 3 && es == sd && el == l) cs_env = ec;
    }
    // CTA size and input staging overrides (read per plan build: A/B sweeps)
    int nt_env = std::getenv("OIOBF_BOX_NT") ? std::atoi(std::getenv("OIOBF_BOX_NT")) : 0;
    if (const char* e = std::getenv("OIOBF_BOX_NT_AT")) {  // per-launch override: "side:level:nt"
      int es = -1, el = -1, en = 0;
      if (std::sscanf(e, "%d:%d:%d", &es, &el, &en) == 3 && es == sd && el == l) nt_env = en;
    }
    const int stage_env = std::getenv("OIOBF_BOX_STAGE") ? std::atoi(std::getenv("OIOBF_BOX_STAGE")) : -1;
    // many small boxes (config 3: 4096 per level): 128-thread CTAs, up to 6
    // per SM, and (without child sums) no input staging -- mode d-1 streams
    // its columns from L2 -- measured 1.49 -> 1.27 ms for the config-3 apply;
    // a few large boxes (config 2: 64 per level) keep 256 threads and staging
    const bool many = static_cast<i64>(descs.size()) >= 4 * static_cast<i64>(device_sms());
    const int box_nt = nt_env == 128 || nt_env == 256 ? nt_env : (many ? 128 : 256);
    const i64 nitems = static_cast<i64>(descs.size());
    int ef_min = 1 << 30, ef_max = 0;
    bool sums = false;
    for (const BoxDesc& x : descs) {
      ef_min = std::min(ef_min, x.eout[f]);
      ef_max = std::max(ef_max, x.eout[f]);
      sums |= x.nsum > 1;
    }
    // Output rows of mode d-1 per CTA: at most 8 (register accumulators of the
    // first mode), or 16 for staged boxes with few columns, whose first mode
    // splits the rows over threads in groups of 4 (first_mode_smem_split) --
    // then a P / U box is one CTA and its input (the ordered child sums) is
    // staged once instead of once per half
    int rs_max = 0;
    for (const BoxDesc& x : descs) {
      int rs = 1;
      for (int k = 0; k < f; ++k) rs *= x.ein[k];
      rs_max = std::max(rs_max, rs);
    }
    const char* a16env = std::getenv("OIOBF_BOX_A16");
    // (boxes without child sums -- the first P level, fed by the core GEMV --
    // qualify as well: with so few columns the input is a few KB and is staged)
    const bool a16 = !(a16env && std::strcmp(a16env, "0") == 0) && (sums || a16env == nullptr || std::strcmp(a16env, "1") != 0) &&
                     bl_split1() && ef_max > 8 && ef_max <= 16 && 2 * static_cast<i64>(rs_max) * nv <= box_nt &&
                     cs_env <= 0;
    const int amax_cap = a16 ? 16 : 8;
    struct Cfg {
      int cs = 0, amax_rows = 0;
      i64 smem_mat = 0, smem_in = 0, smem_t = 0, smem_t1 = 0;  // t0: modes f, f-2, ...; t1: f-1, f-3, ...
      bool stage = false, fits = false;
      i64 total() const { return smem_mat + smem_in + smem_t + smem_t1; }
    };
    auto size_for = [&](int cs) {
      Cfg c;
      c.cs = cs;
      c.amax_rows = (ef_max + cs - 1) / cs;
      for (const BoxDesc& x : descs) {
        i64 m = 0, in_sz = nv, rs = 1;
        for (int k = 0; k < d; ++k) {
          m += static_cast<i64>(x.ein[k]) * (k == f ? c.amax_rows : x.eout[k]);
          in_sz *= x.ein[k];
          if (k < f) rs *= x.ein[k];
        }
        c.smem_mat = std::max(c.smem_mat, m);
        c.smem_in = std::max(c.smem_in, in_sz);
        i64 t = rs * c.amax_rows * nv;  // after mode d-1 (buffer t0)
        c.smem_t = std::max(c.smem_t, t);
        int buf = 1;
        for (int k = f - 1; k >= 1; --k, buf ^= 1) {  // after mode k: the other buffer
          t = t / std::max(1, x.ein[k]) * x.eout[k];
          i64& slot = buf ? c.smem_t1 : c.smem_t;
          slot = std::max(slot, t);
        }
        // staging keeps a table of mode-0 row offsets (8 B each) in buffer t1
        c.smem_t1 = std::max(c.smem_t1, (in_sz / std::max(1, x.ein[0]) + 1) / 2);
      }
      // stage the input when two CTAs per SM still fit (always for child sums);
      // the rule keeps its measured calibration: it is evaluated on two
      // intermediate buffers of the larger size (staging a box that a single
      // CTA reads once only lowers occupancy)
      c.stage = sums || (c.smem_mat + c.smem_in + 2 * std::max(c.smem_t, c.smem_t1)) * 16 <= 112 * 1024;
      if ((stage_env == 0 || (stage_env < 0 && box_nt == 128)) && !sums) c.stage = false;
      if (stage_env == 1 || a16) c.stage = true;
      if (!c.stage) c.smem_in = 0;
      c.fits = c.amax_rows <= amax_cap && c.total() <= kMaxDynSmem / 16;
      return c;
    };
    auto bucket = [](int rows) { return rows <= 2 ? 2 : rows <= 4 ? 4 : 8; };
    // largest split that still runs in one wave (at least ceil(ef / amax_cap)
    // CTAs per box, at most one output row of mode d-1 per CTA)
    // (a CTA whose share of a narrow box is empty just exits early)
    const int cs_lo = std::max(1, (ef_max + amax_cap - 1) / amax_cap);
    Cfg best = size_for(cs_lo);
    if (!best.fits) return false;
    if (cs_env > 0) {
      best = size_for(std::max(cs_lo, std::min(cs_env, ef_max)));
      if (!best.fits) return false;
    } else {
      for (int cs = cs_lo + 1; cs <= std::min(std::max(ef_min, cs_lo), 16); ++cs) {
        const Cfg c = size_for(cs);
        if (!c.fits) break;
        const size_t bytes = 16 * static_cast<size_t>(c.total());
        const i64 cap = static_cast<i64>(box_ctas_per_sm(box_nt, c.stage ? 1 : 0, bytes)) * 148;
        if (nitems * cs > cap) break;
        best = c;
      }
    }
    const int cs = best.cs;
    const int amax_rows = best.amax_rows;
    const bool stage = best.stage;
    const i64 smem_mat = best.smem_mat, smem_in = best.smem_in, smem_t = best.smem_t, smem_t1 = best.smem_t1;
    BoxLaunch bl;
    bl.side = sd;
    bl.level = l;
    bl.in_buf = in_buf;
    bl.out_buf = out_buf;
    bl.item_begin = static_cast<i64>(pl->bdescs.size());
    bl.nitems = nitems;
    bl.info = BoxLaunchInfo{};
    bl.info.d = d;
    bl.info.nv = static_cast<int>(nv);
    bl.info.transpose = transpose;
    bl.info.cs = cs;
    bl.info.amax = bucket(amax_rows);
    bl.info.stage = stage ? 1 : 0;
    bl.info.nt = box_nt;
    {  // FP64 tensor-core phases (OIOBF_BOX_MMA=0: the CUDA-core loops)
      const char* e = std::getenv("OIOBF_BOX_MMA");
      // 0: CUDA-core loops; 1: first mode; 2: and mode 0 of the V / W side; 3: and mode 0 of both sides;
      // 4 (default): first mode, and the middle modes and mode 0 of the V / W side
      bl.info.mma = e ? std::atoi(e) : 4;
      const char* e2 = std::getenv("OIOBF_BOX_ASYNC_FAC");  // 0: blocking factor loads
      bl.info.afac = e2 && std::strcmp(e2, "0") == 0 ? 0 : 1;
      const char* e6 = std::getenv("OIOBF_BOX_STREAM_OUT");  // 0: default-policy stores to G
      bl.info.stream_out = out_buf == BUF_G && !(e6 && std::strcmp(e6, "0") == 0) ? 1 : 0;
      {  // 32-bit column table: offsets relative to the box origin
        bool ok = true;
        for (const BoxDesc& x : descs) {
          i64 span = 0;
          for (int k = 1; k <= d; ++k) span += static_cast<i64>(std::max(0, x.eout[k] - 1)) * std::llabs(x.out_stride[k]);
          ok = ok && span < (i64{1} << 31);
        }
        bl.info.tab_ok = ok ? 1 : 0;
      }
      // compile-time kernel variant (OIOBF_BOX_PATH=0: the all-variants kernel everywhere)
      {
        const char* e8 = std::getenv("OIOBF_BOX_PATH");
        const bool spec = !(e8 && std::strcmp(e8, "0") == 0) && box_nt == 128 && d == 3;
        bool vmma = spec && !stage && bl.info.mma >= 4 && !transpose;
        for (const BoxDesc& x : descs) {
          if (!vmma) break;
          i64 cc = static_cast<i64>(amax_rows) * nv;
          for (int k = 1; k < f; ++k) {
            vmma = vmma && x.ein[k] <= 16 && x.eout[k] <= 8;
            cc *= x.eout[k];
          }
          vmma = vmma && x.ein[f] <= 16 && x.ein[0] <= 16 && x.eout[0] <= 16 && cc <= 512 && bl.info.tab_ok;
        }
        // (the staged variant has CUDA-core middle modes and mode 0: what the P / U side runs unless
        // OIOBF_BOX_MMA=3, and the V / W side only below OIOBF_BOX_MMA=2)
        const bool staged = spec && stage && (transpose ? bl.info.mma != 3 : bl.info.mma < 2);
        bl.info.path = vmma ? 1 : staged ? 2 : 0;
      }
      const char* e3 = std::getenv("OIOBF_BOX_SPLIT1");  // 0: one thread per column in the staged first mode
      bl.info.split1 = e3 && std::strcmp(e3, "0") == 0 ? 0 : 1;
    }
    bl.info.smem_mat = static_cast<int>(smem_mat);
    bl.info.smem_in = static_cast<int>(smem_in);
    bl.info.smem_t = static_cast<int>(smem_t);
    bl.info.smem_t1 = static_cast<int>(smem_t1);
    // d = 2 boxes with enough work per box: the register-tiled GEMM kernel
    // (OIOBF_BOX2=0 disables, =force takes every d = 2 launch)
    {
      const char* b2env = std::getenv("OIOBF_BOX2");  // read per plan build (tests toggle it)
      const bool force = b2env && std::strcmp(b2env, "force") == 0;
      const bool off = b2env && std::strcmp(b2env, "0") == 0;
      if (d == 2 && !off) {
        int e0 = 0, o0 = 0, o1 = 0;
        i64 work = 0;  // mean input box size
        for (const BoxDesc& x : descs) {
          e0 = std::max(e0, x.ein[0]);
          o0 = std::max(o0, x.eout[0]);
          o1 = std::max(o1, x.eout[1]);
          work += static_cast<i64>(x.ein[0]) * x.ein[1];
        }
        work /= std::max<i64>(1, static_cast<i64>(descs.size()));
        const size_t sm2 = box2_smem_bytes(e0, o0, o1);
        if ((force || work >= 512) && sm2 <= 112 * 1024) {
          bl.box2 = 1;
          bl.smem2 = sm2;
        }
      }
    }
    if (std::getenv("OIOBF_DEBUG")) {
      i64 ein = 0, eout = 0;
      for (const BoxDesc& x : descs) {
        i64 a = 1, c = 1;
        for (int k = 0; k < d; ++k) {
          a *= x.ein[k];
          c *= x.eout[k];
        }
        ein = std::max(ein, a);
        eout = std::max(eout, c);
      }
      fprintf(stderr, "[oiobf] box side %d level %d: %lld boxes x cs %d (amax %d, stage %d, box2 %d, nt %d), "
              "smem mat/in/t0/t1 %lld/%lld/%lld/%lld el, "
              "max box in %lld out %lld, smem %lld B, ef %d..%d\n", sd, l, static_cast<long long>(nitems), cs,
              amax_rows, stage ? 1 : 0, bl.box2, bl.info.nt, static_cast<long long>(smem_mat),
              static_cast<long long>(smem_in), static_cast<long long>(smem_t), static_cast<long long>(smem_t1),
              static_cast<long long>(ein), static_cast<long long>(eout),
              static_cast<long long>(box_smem_bytes(bl.info)), ef_min, ef_max);
    }
    pl->bdescs.insert(pl->bdescs.end(), descs.begin(), descs.end());
    pl->ops.push_back(Op{3, static_cast<i64>(pl->boxes.size()), group});
    pl->boxes.push_back(bl);
    return true;
  };
  // chunked (host-pipelined) plans: slab group q = outer index of mode d-1;
  // the F / G rows of group q are one contiguous range
  const int Q = pl->nchunk;
  auto chunk_of = [&](i64 outer) { return Q > 1 ? static_cast<int>(outer / ipow(mpm, d - 1)) : 0; };
  auto tag_ops = [&](size_t from, int q) {
    for (size_t i = from; i < pl->ops.size(); ++i) pl->ops[i].chunk = q;
  };
  // ---- Step 1: V / W, then (Step 2) the core GEMV, per slab group
  std::vector<TRef> cur;  // per item (s, tau) of the current level
  const LevelData& ULc = b.side[1][static_cast<size_t>(b.Lc)];
  std::vector<TRef> gts(static_cast<size_t>(b.nmid * b.nmid));  // index t * nmid + s
  std::vector<TRef> wout(static_cast<size_t>(b.nmid * b.nmid));  // W output per (s, tau = t)
  const bool sharded = b.world > 1;
  pl->sharded = sharded;
  if (sharded)
    require(static_cast<i64>(b.send_off.size()) == b.nmid * b.nmid &&
                static_cast<i64>(b.recv_off.size()) == b.nmid * b.nmid,
            "sharded contract: exchange layout not set (oiobf_tbf_set_exchange)");
  const int* urank = sharded ? b.umid_rank.data() : ULc.h_rank.data();
  for (int q = 0; q < Q; ++q) {
    const size_t ops_mark = pl->ops.size();
    auto mine = [&](i64 outer) { return b.owns(outer) && chunk_of(outer) == q; };
    for (int l = 0; l <= b.Lc; ++l) {
      const LevelData& ld = b.side[0][static_cast<size_t>(l)];
      const i64 nin = ld.L.nin, nj = ld.L.nj;
      const i64 nitems = b.nmid * nin;
      std::vector<TRef> in(static_cast<size_t>(nitems));
      for (i64 it = 0; it < nitems; ++it) {
        const i64 s = it / nin, tau = it % nin;
        if (!mine(s)) continue;  // another rank's (or slab group's) column multi-set
        in[static_cast<size_t>(it)] =
            l == 0 ? global_slab(s)
                   : cur[static_cast<size_t>(s * ipow(2, static_cast<i64>(d) * (l - 1)) + parent_of(tau, l))];
      }
      // ---- fused boxes
      const i64 scratch_mark = scratch;
      std::vector<TRef> outs(static_cast<size_t>(nitems));
      std::vector<BoxDesc> descs;
      const i64 nbeta = ipow(nj, d);
      for (i64 it = 0; it < nitems; ++it) {
        const i64 s = it / nin, tau = it % nin;
        if (!mine(s)) continue;
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
          BoxDesc bd{};
          bd.in_off = x.off;
          bd.out_off = y.off;
          bd.nsum = 1;
          for (int k = 0; k < d; ++k) {
            const i64 j = (beta / ipow(nj, k)) % nj;
            i64 ci = 0, co = 0;
            for (i64 q2 = 0; q2 < j; ++q2) {
              ci += W[k][static_cast<size_t>(q2)];
              co += R[k][static_cast<size_t>(q2)];
            }
            bd.in_off += ci * x.stride[k];
            bd.out_off += co * y.stride[k];
            bd.ein[k] = W[k][static_cast<size_t>(j)];
            bd.eout[k] = R[k][static_cast<size_t>(j)];
            bd.mat_off[k] = MO[k][static_cast<size_t>(j)];
          }
          for (int p = 0; p < nd; ++p) {
            bd.in_stride[p] = x.stride[p];
            bd.out_stride[p] = y.stride[p];
          }
          bd.ein[d] = bd.eout[d] = static_cast<int>(nv);
          descs.push_back(bd);
        }
      }
      if (commit_boxes(descs, 0, l, l == 0 ? BUF_F : BUF_SCRATCH, BUF_SCRATCH, 0, 0)) {
        cur = outs;
        continue;
      }
      scratch = scratch_mark;  // fall back to per-mode launches for this level
      for (int k = 0; k < d; ++k) {
        std::vector<MPStep> mitems;
        std::vector<std::vector<Blk>> blocks;
        for (i64 it = 0; it < nitems; ++it) {
          const i64 s = it / nin, tau = it % nin;
          if (!mine(s)) continue;
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
    for (i64 s = 0; s < b.nmid; ++s)
      if (mine(s))
        for (i64 t = 0; t < b.nmid; ++t)
          wout[static_cast<size_t>(s * b.nmid + t)] = cur[static_cast<size_t>(s * b.nmid + t)];
    // ---- Step 2: cores.  x = F_{t,s} = W output (s, tau = t); y = G_{t,s}
    const i64 gemv_begin = static_cast<i64>(pl->gemv.size());
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
      if (!mine(s)) continue;
      const PairDesc& pd = b.h_pairs[static_cast<size_t>(p)];
      const TRef& x = wout[static_cast<size_t>(s * b.nmid + t)];
      TRef y;
      if (sharded && b.peer_mode()) {
        // fused exchange: the GEMV stores G_{t,s} into the receive buffer of
        // the owner q of t (peer memory), addressed relative to this rank's own
        // receive buffer of the same parity (the phase-1 output pointer)
        const i64 po = b.peer_off[static_cast<size_t>(t * b.nmid + s)];
        require(po >= 0, "sharded contract: missing peer offset");
        const int q = b.owner_of(t);
        const u64 mine_base = b.peer_base[static_cast<size_t>(parity * b.world + b.rank)];
        const u64 dest_base = b.peer_base[static_cast<size_t>(parity * b.world + q)];
        const i64 delta = static_cast<i64>(dest_base - mine_base);
        require(delta % 16 == 0, "sharded contract: receive buffers must be 16-byte aligned");
        y = packed(delta / 16 + po * nv, nd, gext);
      } else if (sharded) {  // GEMV output goes straight into the send buffer
        const i64 so = b.send_off[static_cast<size_t>(t * b.nmid + s)];
        require(so >= 0, "sharded contract: missing send offset");
        y = packed(so * nv, nd, gext);
      } else {
        y = alloc(nd, gext);
        gts[static_cast<size_t>(t * b.nmid + s)] = y;
      }
      if (R != pd.R || x.size() != static_cast<i64>(pd.C) * nv)
        throw std::runtime_error("internal: core shape mismatch");
      GemvDesc g;
      g.core_off = pl->bfp ? b.bfp_off[static_cast<size_t>(p)] : pd.core_off;
      g.x_off = x.off;
      g.y_off = y.off;
      g.R = pd.R;
      g.C = pd.C;
      pl->gemv.push_back(g);
    }
    if (static_cast<i64>(pl->gemv.size()) > gemv_begin) {
      finish_gemv(*pl, gemv_begin, static_cast<i64>(pl->gemv.size()), nv);
      pl->ops.push_back(Op{1, static_cast<i64>(pl->gemvs.size()) - 1, 1});
    }
    tag_ops(ops_mark, q);
  }  // slab groups (V/W + GEMV)
  // ---- Step 3: P (l = Lc..1), U (l = 0).  A P level writes one contribution
  // per child nu into consecutive equally-shaped buffers of its parent; the
  // consumer (next level down) reads their ordered sum (TRef::nsum) while
  // staging its input, so no separate summation pass is needed.
  for (int q = 0; q < Q; ++q) {
    const size_t ops_mark = pl->ops.size();
    auto mine = [&](i64 outer) { return b.owns(outer) && chunk_of(outer) == q; };
    std::vector<TRef> gcur = gts;  // per (t, nu) at level l: index t * nin + nu
    const int u_in0 = sharded ? BUF_RECV : BUF_SCRATCH;
    for (int l = b.Lc; l >= 0; --l) {
      const LevelData& ld = b.side[1][static_cast<size_t>(l)];
      const i64 nin = ld.L.nin, nj = ld.L.nj;
      const i64 pnin = l > 0 ? ipow(2, static_cast<i64>(d) * (l - 1)) : 1;
      const i64 nbeta = ipow(nj, d);
      const int u_in = l == b.Lc ? u_in0 : BUF_SCRATCH;
      std::vector<TRef> par(static_cast<size_t>(b.nmid * pnin));
      // kids of each parent, output widths, and the parents' child blocks
      auto kids_of = [&](i64 pnu) {
        std::vector<i64> kids;
        for (i64 nu = 0; nu < nin; ++nu)
          if (l == 0 || parent_of(nu, l) == pnu) kids.push_back(nu);
        return kids;
      };
      auto parent_shape = [&](i64 t, i64 nu0, int* oext, std::vector<std::vector<int>>& W) {
        W.assign(static_cast<size_t>(d), {});
        for (int k = 0; k < d; ++k) {
          int tw = 0;
          for (i64 j = 0; j < nj; ++j) {
            int r, w;
            i64 mo;
            slot_info(1, l, t, nu0, k, j, r, w, mo);
            W[static_cast<size_t>(k)].push_back(w);
            tw += w;
          }
          oext[k] = tw;
        }
        oext[d] = static_cast<int>(nv);
      };
      // child c's output buffer of parent (t, pnu): consecutive, parent-shaped
      std::vector<TRef> child_out(static_cast<size_t>(b.nmid * nin));
      for (i64 t = 0; t < b.nmid; ++t)
        for (i64 pnu = 0; pnu < pnin; ++pnu) {
          if (!mine(t)) continue;  // another rank's (or slab group's) row multi-set
          const std::vector<i64> kids = kids_of(pnu);
          int oext[kMaxTM];
          std::vector<std::vector<int>> W;
          parent_shape(t, kids[0], oext, W);
          if (l == 0) {
            const TRef y = global_slab(t);
            par[static_cast<size_t>(t * pnin + pnu)] = y;
            child_out[static_cast<size_t>(t * nin + kids[0])] = y;
            continue;
          }
          const TRef y0 = alloc(nd, oext);
          const i64 psize = y0.size();
          for (size_t c = 1; c < kids.size(); ++c) alloc(nd, oext);
          TRef pref = y0;
          pref.nsum = static_cast<int>(kids.size());
          pref.sum_stride = psize;
          par[static_cast<size_t>(t * pnin + pnu)] = pref;
          for (size_t c = 0; c < kids.size(); ++c) {
            TRef yc = y0;
            yc.off = y0.off + static_cast<i64>(c) * psize;
            child_out[static_cast<size_t>(t * nin + kids[c])] = yc;
          }
        }
      std::vector<BoxDesc> descs;
      for (i64 t = 0; t < b.nmid; ++t)
        for (i64 nu = 0; nu < nin; ++nu) {
          if (!mine(t)) continue;
          const TRef& x = gcur[static_cast<size_t>(t * nin + nu)];
          const TRef& yc = child_out[static_cast<size_t>(t * nin + nu)];
          for (i64 beta = 0; beta < nbeta; ++beta) {
            BoxDesc bd{};
            bd.out_off = yc.off;
            bd.in_off = x.off;
            bd.nsum = x.nsum;
            bd.sum_stride = x.sum_stride;
            for (int k = 0; k < d; ++k) {
              const int jb = static_cast<int>((beta / ipow(nj, k)) % nj);
              i64 co = 0, ci = 0;
              int r = 0, w = 0;
              i64 mo = 0;
              for (int q2 = 0; q2 < jb; ++q2) {
                slot_info(1, l, t, nu, k, q2, r, w, mo);
                ci += r;
                co += w;
              }
              slot_info(1, l, t, nu, k, jb, r, w, mo);
              bd.out_off += co * yc.stride[k];
              bd.in_off += ci * x.stride[k];
              bd.ein[k] = r;
              bd.eout[k] = w;
              bd.mat_off[k] = mo;
            }
            for (int p = 0; p < nd; ++p) {
              bd.out_stride[p] = yc.stride[p];
              bd.in_stride[p] = x.stride[p];
            }
            bd.ein[d] = bd.eout[d] = static_cast<int>(nv);
            descs.push_back(bd);
          }
        }
      if (commit_boxes(descs, 1, l, u_in, l == 0 ? BUF_G : BUF_SCRATCH, 1, 2)) {
        gcur = par;
        continue;
      }
      // ---- fall back: materialize summed inputs, then per-mode launches
      {
        SumLaunch sl;
        sl.begin = static_cast<i64>(pl->sums.size());
        i64 work = 0;
        std::map<i64, TRef> done;  // child block offset -> materialized parent
        for (i64 it = 0; it < b.nmid * nin; ++it) {
          const i64 t = it / nin;
          if (!mine(t)) continue;
          TRef& x = gcur[static_cast<size_t>(it)];
          if (x.nsum <= 1) continue;
          auto hit = done.find(x.off);
          if (hit != done.end()) {
            x = hit->second;
            continue;
          }
          SumDesc sdsc{};
          for (int c = 0; c < x.nsum; ++c) sdsc.child_off[sdsc.nchild++] = x.off + c * x.sum_stride;
          const TRef y = alloc(nd, x.ext);
          sdsc.out_off = y.off;
          sdsc.total = y.size();
          sdsc.work_off = work;
          work += sdsc.total;
          pl->sums.push_back(sdsc);
          done[x.off] = y;
          x = y;
        }
        sl.n = static_cast<i64>(pl->sums.size()) - sl.begin;
        sl.total = work;
        if (sl.n > 0) {
          pl->ops.push_back(Op{2, static_cast<i64>(pl->sum_launches.size()), 2});
          pl->sum_launches.push_back(sl);
        }
      }
      std::vector<TRef> x = gcur;
      for (int k = 0; k < d; ++k) {
        std::vector<MPStep> mitems;
        std::vector<std::vector<Blk>> blocks;
        for (i64 it = 0; it < b.nmid * nin; ++it) {
          const i64 t = it / nin;
          if (!mine(t)) continue;
          TRef& xi = x[static_cast<size_t>(it)];
          int oext[kMaxTM];
          for (int p = 0; p < nd; ++p) oext[p] = xi.ext[p];
          std::vector<Blk> bl;
          int ci = 0, co = 0;
          for (i64 j = 0; j < nj; ++j) {
            Blk B;
            int r, w;
            slot_info(1, l, t, it % nin, k, j, r, w, B.mat_off);
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
          // the last mode writes the child's block of its parent (or G)
          TRef y = k == d - 1 ? child_out[static_cast<size_t>(it)] : alloc(nd, oext);
          mitems.push_back(make_step(xi, y, k, 1));
          blocks.push_back(bl);
          xi = y;
        }
        const int in_buf = k == 0 ? u_in : BUF_SCRATCH;
        add_mp(*pl, 1, l, in_buf, (l == 0 && k == d - 1) ? BUF_G : BUF_SCRATCH, mitems, blocks, 2);
      }
      gcur = par;
    }
    tag_ops(ops_mark, q);
  }  // slab groups (P/U)
  pl->scratch_elems = scratch;
  cudaStream_t st = b.stream;
  pl->d_steps = to_device(pl->steps, st);
  pl->d_blks = to_device(pl->blks, st);
  pl->d_gemv = to_device(pl->gemv, st);
  pl->d_gemv_map = to_device(pl->gemv_map, st);
  pl->d_gemv_rb = to_device(pl->gemv_rb, st);
  pl->d_tma_map = to_device(pl->tma_map, st);
  pl->d_sums = to_device(pl->sums, st);
  pl->d_bdescs = to_device(pl->bdescs, st);
  pl->scratch.alloc(static_cast<size_t>(std::max<i64>(scratch, 1)));
  TBF_CUDA(cudaStreamSynchronize(st));
  return pl;
}

// ---- tiny-box engine plan (config 4 scale: ~1e8 boxes of <= kTinyBox elements)
// Largest box (input and output elements) of every level, both sides, and the
// widest core row: the tiny engine costs O(box) per output element.
bool tiny_eligible(const oiobf_tbf& b) {
  if (b.world > 1 || b.d < 1) return false;
  const int d = b.d;
  for (int sd = 0; sd < 2; ++sd)
    for (int l = 0; l <= b.Lc; ++l) {
      const LevelData& ld = b.side[sd][static_cast<size_t>(l)];
      const i64 nj = ld.L.nj;
      const i64 ngroups = ld.nslots / (d * nj);
      for (i64 g = 0; g < ngroups; ++g) {
        i64 bin = 1, bout = 1;
        for (int k = 0; k < d; ++k) {
          int mr = 0, mw = 0;
          for (i64 j = 0; j < nj; ++j) {
            const size_t sl = static_cast<size_t>((g * d + k) * nj + j);
            mr = std::max(mr, ld.h_rank[sl]);
            mw = std::max(mw, ld.h_width[sl]);
          }
          bin *= sd == 0 ? mw : mr;
          bout *= sd == 0 ? mr : mw;
        }
        if (bin > kTinyBox || bout > kTinyBox) return false;
      }
    }
  for (const PairDesc& pd : b.h_pairs)
    if (pd.C > kTinyBox) return false;
  return true;
}

// auto: the tiny engine when every box is tiny AND there are so many pairs that
// per-box descriptors / CTAs would dominate (>= 2^20 middle pairs)
bool use_tiny_engine(oiobf_tbf& b) {
  if (b.apply_engine == 1) return false;
  if (b.apply_engine == 2) return true;
  if (b.tiny_auto < 0)  // the eligibility scan walks every slot: once per handle
    b.tiny_auto = (b.nmid * b.nmid >= (i64{1} << 20) && tiny_eligible(b)) ? 1 : 0;
  return b.tiny_auto == 1;
}

std::unique_ptr<Plan> build_plan_tiny(oiobf_tbf& b, i64 nv) {
  require(b.world == 1, "tiny-box engine: sharded factorizations use the box engine");
  auto pl = std::make_unique<Plan>();
  pl->nv = nv;
  const int d = b.d;
  const i64 n = b.n, N = ipow(n, d);
  const i64 mid = n >> b.Lc, mpm = ipow(2, b.Lc);
  i64 scratch = 0;
  auto slab_off = [&](i64 outer) {
    i64 off = 0, st = 1;
    for (int p = 0; p < d; ++p) {
      off += ((outer / ipow(mpm, p)) % mpm) * mid * st;
      st *= n;
    }
    return off;
  };
  auto child_inner = [&](i64 pinner, int l, int c) {
    i64 inner = 0;
    for (int p = d - 1; p >= 0; --p) {
      const i64 pc = (pinner >> ((l - 1) * p)) & ((i64{1} << (l - 1)) - 1);
      inner = (inner << l) | (2 * pc + ((c >> p) & 1));
    }
    return inner;
  };
  // sum over blocks j of the rank (what = 0) or width (what = 1) of slot group (outer, inner, k)
  auto ext_of = [&](const LevelData& ld, i64 outer, i64 inner, int k, int what) {
    const i64 nin = ld.L.nin, nj = ld.L.nj;
    i64 e = 0;
    for (i64 j = 0; j < nj; ++j) {
      const size_t sl = static_cast<size_t>(((outer * nin + inner) * d + k) * nj + j);
      e += what == 0 ? ld.h_rank[sl] : ld.h_width[sl];
    }
    return e;
  };
  // largest factor block set of one (outer, inner, k): sum over j of r * w
  auto fac_of = [&](const LevelData& ld, i64 outer, i64 inner) {
    const i64 nin = ld.L.nin, nj = ld.L.nj;
    i64 m = 0;
    for (int k = 0; k < d; ++k) {
      i64 e = 0;
      for (i64 j = 0; j < nj; ++j) {
        const size_t sl = static_cast<size_t>(((outer * nin + inner) * d + k) * nj + j);
        e += static_cast<i64>(ld.h_rank[sl]) * ld.h_width[sl];
      }
      m = std::max(m, e);
    }
    return m;
  };
  i64 fstride = 0, xstride = 0, ostride = 0, maxo = 1;  // of the level being planned
  auto add_level = [&](int sd, int l, const LevelData& ld, int nch, int in_buf, int out_buf, int in_global,
                       int out_global, i64 group_begin, i64 off_begin, i64 max_in) {
    Plan::TinyLevel tl;
    tl.side = sd;
    tl.l = l;
    tl.in_buf = in_buf;
    tl.out_buf = out_buf;
    tl.group_begin = group_begin;
    tl.off_begin = off_begin;
    TinyLevelArgs& a = tl.args;
    a = TinyLevelArgs{};
    a.side = sd;
    a.l = l;
    a.d = d;
    a.nv = static_cast<int>(nv);
    a.in_global = in_global;
    a.out_global = out_global;
    a.nch = nch;
    a.nin = ld.L.nin;
    a.nj = ld.L.nj;
    a.ngroups = static_cast<i64>(pl->tiny_groups.size()) - group_begin;
    a.max_in = max_in;
    a.fstride = fstride;
    a.xstride = xstride;
    a.ostride = ostride;
    a.maxo = maxo;
    if (tiny_smem_bytes(a) > static_cast<size_t>(kMaxDynSmem)) a.fstride = 0;  // factors from global memory
    // CTA size from the group's output count (small groups: small CTAs, more resident)
    {
      const i64 outs = sd == 0 ? nch * ostride : 0;
      i64 mx = outs;
      if (sd == 1) {  // parent output size
        for (i64 gi = group_begin; gi < static_cast<i64>(pl->tiny_groups.size()); ++gi) {
          const TinyGroup& tg = pl->tiny_groups[static_cast<size_t>(gi)];
          i64 size = nv;
          const i64 first = l > 0 ? child_inner(tg.pinner, l, 0) : 0;
          for (int k = 0; k < d; ++k) size *= ext_of(ld, tg.outer, first, k, 1);
          mx = std::max(mx, size);
          if (gi - group_begin > 4096) break;  // a sample: the CTA size only affects speed
        }
      }
      int th = 32;
      while (th < 256 && th < mx) th *= 2;
      a.threads = th;
    }
    {
      i64 st = 1;
      for (int p = 0; p < d; ++p) {
        a.gstride[p] = st;
        st *= n;
      }
      a.gstride[d] = N;
    }
    require(tiny_smem_bytes(a) <= static_cast<size_t>(kMaxDynSmem), "tiny engine: a box group does not fit on chip");
    pl->ops.push_back(Op{6, static_cast<i64>(pl->tiny_levels.size()), sd == 0 ? 0 : 2});
    pl->tiny_levels.push_back(tl);
  };
  // ---- V / W: group = parent (s, p_tau); its 2^d children tau read the parent output
  std::vector<i64> prev;  // output offset per (s, tau) of the previous level
  for (int l = 0; l <= b.Lc; ++l) {
    const LevelData& ld = b.side[0][static_cast<size_t>(l)];
    const i64 nin = ld.L.nin;
    const i64 pnin = l > 0 ? ipow(2, static_cast<i64>(d) * (l - 1)) : 1;
    const int nch = l > 0 ? (1 << d) : 1;
    const i64 group_begin = static_cast<i64>(pl->tiny_groups.size());
    const i64 off_begin = static_cast<i64>(pl->tiny_off.size());
    pl->tiny_off.resize(static_cast<size_t>(off_begin + b.nmid * nin));
    i64 max_in = 1;
    fstride = 0;
    ostride = 1;
    maxo = 1;
    for (i64 s = 0; s < b.nmid; ++s)
      for (i64 ptau = 0; ptau < pnin; ++ptau) {
        const i64 first = l > 0 ? child_inner(ptau, l, 0) : 0;
        i64 in_sz = nv;
        for (int k = 0; k < d; ++k) in_sz *= ext_of(ld, s, first, k, 1);
        max_in = std::max(max_in, in_sz);
        pl->tiny_groups.push_back(TinyGroup{s, ptau, l == 0 ? slab_off(s) : prev[static_cast<size_t>(s * pnin + ptau)]});
        for (int c = 0; c < nch; ++c) {
          const i64 tau = l > 0 ? child_inner(ptau, l, c) : 0;
          fstride = std::max(fstride, fac_of(ld, s, tau));
          i64 size = nv;
          for (int k = 0; k < d; ++k) {
            const i64 e = ext_of(ld, s, tau, k, 0);
            maxo = std::max(maxo, e);
            size *= e;
          }
          ostride = std::max(ostride, size);
          pl->tiny_off[static_cast<size_t>(off_begin + s * nin + tau)] = scratch;
          scratch += size;
        }
      }
    add_level(0, l, ld, nch, l == 0 ? BUF_F : BUF_SCRATCH, BUF_SCRATCH, l == 0 ? 1 : 0, 0, group_begin, off_begin,
              max_in);
    prev.assign(pl->tiny_off.begin() + off_begin, pl->tiny_off.end());
  }
  // ---- cores: G_{t,s} = K(tbar, sbar) F_{t,s}, F_{t,s} = W output (s, tau = t)
  std::vector<i64> gts(static_cast<size_t>(b.nmid * b.nmid));
  {
    i64 rows = 0;
    for (i64 p = 0; p < b.nmid * b.nmid; ++p) {
      const i64 s = p / b.nmid, t = p % b.nmid;
      const PairDesc& pd = b.h_pairs[static_cast<size_t>(p)];
      GemvDesc g;
      g.core_off = pd.core_off;
      g.x_off = prev[static_cast<size_t>(s * b.nmid + t)];
      g.y_off = scratch;
      g.R = pd.R;
      g.C = pd.C;
      g.cta_off = rows;
      rows += pd.R;
      gts[static_cast<size_t>(t * b.nmid + s)] = scratch;
      scratch += static_cast<i64>(pd.R) * nv;
      pl->gemv.push_back(g);
    }
    GemvLaunch gl;
    gl.desc_begin = 0;
    gl.ndesc = static_cast<i64>(pl->gemv.size());
    gl.total_rows = rows;
    pl->gemvs.push_back(gl);
    pl->ops.push_back(Op{7, 0, 1});
  }
  // ---- P / U: group = parent (t, p_nu); its 2^d children nu (ascending) add into it
  std::vector<i64> pin = gts;  // input offset per (t, nu) of the current level
  for (int l = b.Lc; l >= 0; --l) {
    const LevelData& ld = b.side[1][static_cast<size_t>(l)];
    const i64 nin = ld.L.nin;
    const i64 pnin = l > 0 ? ipow(2, static_cast<i64>(d) * (l - 1)) : 1;
    const int nch = l > 0 ? (1 << d) : 1;
    const i64 group_begin = static_cast<i64>(pl->tiny_groups.size());
    const i64 off_begin = static_cast<i64>(pl->tiny_off.size());
    pl->tiny_off.insert(pl->tiny_off.end(), pin.begin(), pin.end());
    std::vector<i64> out(static_cast<size_t>(b.nmid * pnin));
    fstride = 0;
    xstride = 1;
    maxo = 1;
    for (i64 t = 0; t < b.nmid; ++t)
      for (i64 pnu = 0; pnu < pnin; ++pnu) {
        const i64 first = l > 0 ? child_inner(pnu, l, 0) : 0;
        for (int c = 0; c < nch; ++c) {
          const i64 nu = l > 0 ? child_inner(pnu, l, c) : 0;
          i64 cs = nv;
          for (int k = 0; k < d; ++k) cs *= ext_of(ld, t, nu, k, 0);
          xstride = std::max(xstride, cs);
          fstride = std::max(fstride, fac_of(ld, t, nu));
        }
        i64 size = nv;
        for (int k = 0; k < d; ++k) {
          const i64 e = ext_of(ld, t, first, k, 1);
          maxo = std::max(maxo, e);
          size *= e;
        }
        const i64 off = l == 0 ? slab_off(t) : scratch;
        pl->tiny_groups.push_back(TinyGroup{t, pnu, off});
        out[static_cast<size_t>(t * pnin + pnu)] = off;
        if (l > 0) scratch += size;
      }
    add_level(1, l, ld, nch, BUF_SCRATCH, l == 0 ? BUF_G : BUF_SCRATCH, 0, l == 0 ? 1 : 0, group_begin, off_begin,
              nch * xstride);
    pin.swap(out);
  }
  pl->scratch_elems = scratch;
  cudaStream_t st = b.stream;
  pl->d_gemv = to_device(pl->gemv, st);
  pl->d_tiny_groups = to_device(pl->tiny_groups, st);
  pl->d_tiny_off = to_device(pl->tiny_off, st);
  pl->scratch.alloc(static_cast<size_t>(std::max<i64>(scratch, 1)));
  TBF_CUDA(cudaStreamSynchronize(st));
  return pl;
}

// ---- rank-one engine (r1_kernels.cu): every ID of rank 1 (DFT with two-sided
// bit reversal), so factor blocks, intermediates and cores are regular.
// Eligible when, on both sides and every level, each slot has rank 1 and
// width W_l (the leaf size <= 2 at l = 0, 2 above) with its block at slot * W_l
// in the interp arena, and every core is 1 x 1 at its pair index.
// Sharded (world > 1): the same for the OWNED slots and pairs, whose blocks
// are packed in local order (slots of other ranks have rank 0 and no block);
// every rank must own the same power-of-two number of middle multi-sets.
std::vector<int> owned_list(const oiobf_tbf& b) {
  std::vector<int> own;
  for (i64 o = 0; o < b.nmid; ++o)
    if (b.owns(o)) own.push_back(static_cast<int>(o));
  return own;
}

bool r1_eligible(const oiobf_tbf& b) {
  if (b.d < 1 || b.d > kMaxD || (b.n & (b.n - 1)) != 0) return false;
  const i64 leaf = b.n >> b.L;
  if (leaf < 1 || leaf > 2) return false;
  const bool sharded = b.world > 1;
  std::vector<i64> pos(static_cast<size_t>(b.nmid), -1);  // local index of an owned middle multi-set
  i64 nown = 0;
  for (i64 o = 0; o < b.nmid; ++o)
    if (b.owns(o)) pos[static_cast<size_t>(o)] = nown++;
  if (sharded) {
    if (nown * b.world != b.nmid || (nown & (nown - 1)) != 0) return false;
    if (b.peer_mode()) return false;  // the fused exchange is the box engine's GEMV epilogue
    if (static_cast<i64>(b.send_off.size()) != b.nmid * b.nmid) return false;
  }
  for (int sd = 0; sd < 2; ++sd) {
    if (b.side[sd].size() != static_cast<size_t>(b.Lc + 1)) return false;
    for (int l = 0; l <= b.Lc; ++l) {
      const LevelData& ld = b.side[sd][static_cast<size_t>(l)];
      const int w = l == 0 ? static_cast<int>(leaf) : 2;
      if (static_cast<i64>(ld.h_rank.size()) != ld.nslots || static_cast<i64>(ld.h_interp_off.size()) != ld.nslots)
        return false;
      const i64 per_outer = ld.nslots / b.nmid;  // slots of one outer multi-set (contiguous)
      std::vector<char> bad(parallel_nchunks(static_cast<size_t>(ld.nslots)), 0);
      parallel_chunks(static_cast<size_t>(ld.nslots), [&](size_t c, size_t lo, size_t hi) {
        for (size_t i = lo; i < hi && !bad[c]; ++i) {
          const i64 outer = static_cast<i64>(i) / per_outer;
          const i64 li = pos[static_cast<size_t>(outer)];
          if (li < 0) {
            bad[c] = ld.h_rank[i] != 0;
          } else {
            const i64 local = li * per_outer + (static_cast<i64>(i) - outer * per_outer);
            bad[c] = ld.h_rank[i] != 1 || ld.h_width[i] != w || ld.h_interp_off[i] != local * w;
          }
        }
      });
      for (char x : bad)
        if (x) return false;
    }
  }
  const i64 P = b.nmid * b.nmid;
  if (static_cast<i64>(b.h_pairs.size()) != P) return false;
  std::vector<char> bad(parallel_nchunks(static_cast<size_t>(P)), 0);
  parallel_chunks(static_cast<size_t>(P), [&](size_t c, size_t lo, size_t hi) {
    for (size_t p = lo; p < hi && !bad[c]; ++p) {
      const PairDesc& pd = b.h_pairs[p];
      const i64 sq = static_cast<i64>(p) / b.nmid, t = static_cast<i64>(p) - sq * b.nmid;
      const i64 li = pos[static_cast<size_t>(sq)];
      if (li < 0) {
        bad[c] = pd.C != 0;
      } else {
        bad[c] = pd.R != 1 || pd.C != 1 || pd.core_off != li * b.nmid + t;
        if (sharded)  // every block G_{t,s} is one element: the exchange tables must say so
          bad[c] = bad[c] || b.send_off[static_cast<size_t>(t * b.nmid + sq)] < 0;
      }
    }
  });
  for (char x : bad)
    if (x) return false;
  return true;
}

bool use_r1_engine(oiobf_tbf& b) {
  if (b.apply_engine != 0 && b.apply_engine != 4) return false;
  if (b.r1_ok < 0) b.r1_ok = r1_eligible(b) ? 1 : 0;  // one scan of every slot per handle
  if (b.apply_engine == 4)
    require(b.r1_ok == 1, "tbf_set_apply_engine: the rank-one engine needs every ID of rank 1 (leaf <= 2)");
  return b.r1_ok == 1;
}

std::unique_ptr<Plan> build_plan_r1(oiobf_tbf& b, i64 nv) {
  auto pl = std::make_unique<Plan>();
  pl->nv = nv;
  const int d = b.d;
  const i64 n = b.n;
  // sharded: the nown owned middle multi-sets in local order (r1_eligible)
  const std::vector<int> own = b.world > 1 ? owned_list(b) : std::vector<int>();
  const i64 nown = b.world > 1 ? static_cast<i64>(own.size()) : b.nmid;
  if (b.world > 1) {
    pl->sharded = true;
    pl->d_r1_own = to_device(own, b.stream);
    pl->d_r1_send_off = to_device(b.send_off, b.stream);
    pl->d_r1_recv_off = to_device(b.recv_off, b.stream);
    TBF_CUDA(cudaStreamSynchronize(b.stream));
  }
  const i64 P = nown * b.nmid;  // elements of every intermediate (per vector)
  const i64 leaf = n >> b.L;
  auto base = [&](int sd, int l) {
    const LevelData& ld = b.side[sd][static_cast<size_t>(l)];
    R1LevelArgs a{};
    a.side = sd;
    a.l = l;
    a.d = d;
    a.W = l == 0 ? static_cast<int>(leaf) : 2;
    a.nv = static_cast<int>(nv);
    a.Lc = b.Lc;
    a.nch = l > 0 ? (1 << d) : 1;
    a.n = n;
    a.nmid = b.nmid;
    a.mpm = ipow(2, b.Lc);
    a.mid = n >> b.Lc;
    a.nin = ld.L.nin;
    a.nj = ld.L.nj;
    a.njd = ipow(a.nj, d);
    a.pnin = l > 0 ? ipow(2, static_cast<i64>(d) * (l - 1)) : 1;
    a.ngroups = nown * a.pnin;
    a.E = a.nj * a.W;
    a.ED = ipow(a.E, d);
    a.fblk = static_cast<int>(d * a.nj * a.W);
    a.FS = a.fblk | 1;
    auto lg = [](i64 x) {
      int r = 0;
      while ((i64{1} << r) < x) ++r;
      require((i64{1} << r) == x, "rank-one engine: extents must be powers of two");
      return r;
    };
    a.lg_n = lg(n);
    a.lg_mid = lg(a.mid);
    a.lg_nmid = lg(a.nmid);
    a.lg_nown = lg(nown);
    a.own = b.world > 1 ? pl->d_r1_own.p : nullptr;
    a.lg_nin = lg(a.nin);
    a.lg_nj = lg(a.nj);
    a.lg_njd = lg(a.njd);
    a.lg_pnin = lg(a.pnin);
    a.lg_nch = lg(a.nch);
    a.lg_E = lg(a.E);
    a.lg_ED = lg(a.ED);
    return a;
  };
  const int th = r1_threads();
  // ping-pong: level outputs alternate between scratch halves [0, P nv) and [P nv, 2 P nv)
  int cur = 0;  // half holding the current intermediate (-1: F)
  auto add = [&](R1LevelArgs a, int in_half, int out_half) {
    Plan::R1Level rl;
    a.magic = static_cast<unsigned>(((u64{1} << 32) + a.fblk - 1) / a.fblk);
    rl.args = a;
    rl.in_off = in_half < 0 ? -1 : in_half * P * nv;
    rl.out_off = out_half < 0 ? -1 : out_half * P * nv;
    require(r1_smem_bytes(a) <= static_cast<size_t>(kMaxDynSmem), "rank-one engine: a group does not fit on chip");
    pl->ops.push_back(Op{8, static_cast<i64>(pl->r1_levels.size()), a.side == 0 ? (a.core_mul ? 1 : 0) : 2});
    pl->r1_levels.push_back(rl);
  };
  auto parent_of = [&](i64 inner, int l) {
    i64 p = 0;
    for (int q = 0; q < d; ++q) p |= (((inner >> (l * q)) & ((i64{1} << l) - 1)) >> 1) << ((l - 1) * q);
    return p;
  };
  for (int l = 0; l <= b.Lc; ++l) {
    R1LevelArgs a = base(0, l);
    a.in_global = l == 0;
    a.core_mul = l == b.Lc;
    // T consecutive tau per CTA: their factor blocks (T * FS elements) <= 32 KB
    a.lg_T = 0;
    while (a.lg_T < a.lg_nin && (i64{2} << a.lg_T) * a.FS * 16 <= 32 * 1024) ++a.lg_T;
    a.Pc = l > 0 ? static_cast<int>(parent_of((i64{1} << a.lg_T) - 1, l) + 1) : 1;
    a.XS = static_cast<int>(a.ED | 1);
    if (l >= 1 && a.njd == 1 && a.lg_nin >= 5) {  // middle level: warp tiles of 32 tau
      a.warp_tiles = 1;
      a.Pc = static_cast<int>(parent_of(31, l) + 1);
    }
    const int out_half = l == 0 ? 0 : 1 - cur;
    add(a, l == 0 ? -1 : cur, out_half);
    cur = out_half;
  }
  if (b.world > 1) {
    // exchange: pack the level-Lc V/W output into the send buffer (phase 1);
    // unpack the receive buffer into the level-Lc P/U input (phase 2)
    Plan::R1Level pk;
    pk.args = base(0, b.Lc);
    pk.in_off = cur * P * nv;
    pk.out_off = -1;
    pl->ops.push_back(Op{9, static_cast<i64>(pl->r1_levels.size()), 1});
    pl->r1_levels.push_back(pk);
    Plan::R1Level up = pk;
    up.in_off = -1;
    up.out_off = cur * P * nv;
    pl->ops.push_back(Op{10, static_cast<i64>(pl->r1_levels.size()), 2});
    pl->r1_levels.push_back(up);
  }
  for (int l = b.Lc; l >= 0; --l) {
    R1LevelArgs a = base(1, l);
    a.in_transposed = l == b.Lc;
    a.out_global = l == 0;
    a.nunits = a.ngroups * a.njd;
    i64 nx = 1;
    for (int k = 0; k < d; ++k) nx *= a.W;
    a.warp_tiles = l >= 1;  // one warp per (group, block tuple) unit
    if (!a.warp_tiles) {
      a.gpb = static_cast<int>(std::max<i64>(1, th / std::max<i64>(nx, a.nch)));  // units: <= one thread per child
      while (a.gpb > 1 && r1_smem_bytes(a) > 72 * 1024) a.gpb /= 2;
    }
    const int out_half = l == 0 ? -1 : 1 - cur;
    add(a, cur, out_half);
    cur = out_half;
  }
  pl->scratch_elems = 2 * P * nv;
  pl->scratch.alloc(static_cast<size_t>(std::max<i64>(pl->scratch_elems, 1)));
  return pl;
}

// chunked = true: the host-pipelined plan (ops per slab group, see
// contract_host); the device-buffer path uses the unchunked plan
// parity: fused-exchange plans (receive buffers alternate between steps)
Plan& get_plan(oiobf_tbf& b, i64 nv, bool chunked = false, int parity = 0) {
  const bool r1 = use_r1_engine(b);
  const bool tiny = !r1 && use_tiny_engine(b);
  if (tiny || r1) chunked = false;  // one slab group: these plans are not split
  const i64 key = 4 * nv + 2 * parity + (chunked ? 1 : 0);
  auto it = b.plans.find(key);
  if (it != b.plans.end()) return *it->second;
  auto& slot = b.plans[key];
  slot = r1 ? build_plan_r1(b, nv) : tiny ? build_plan_tiny(b, nv) : build_plan(b, nv, chunked, parity);
  return *slot;
}


struct OpBuffers {
  const double2* F = nullptr;
  double2* G = nullptr;
  double2* send = nullptr;
  const double2* recv = nullptr;
  double2* scratch = nullptr;  // null: the plan's own scratch
};

// phase: 0 = whole contraction, 1 = V/W + core GEMV, 2 = P/U (sharded, or
// one slab group of a pipelined plan); chunk >= 0: that slab group only
void run_ops(oiobf_tbf& b, Plan& pl, const OpBuffers& io, cudaStream_t st, int group_filter = -1, int phase = 0,
             int chunk = -1) {
  // OIOBF_ABLATE=<digits>: skip these op kinds (timing experiments only; the
  // result is wrong when set)
  static const char* ablate = std::getenv("OIOBF_ABLATE");
  double2* const scr = io.scratch ? io.scratch : pl.scratch.p;
  auto in_ptr = [&](int id) -> const double2* {
    return id == BUF_F ? io.F : id == BUF_RECV ? io.recv : scr;
  };
  auto out_ptr = [&](int id) -> double2* { return id == BUF_G ? io.G : id == BUF_SEND ? io.send : scr; };
  for (const Op& op : pl.ops) {
    if (group_filter >= 0 && op.group != group_filter) continue;
    if (phase == 1 && op.group == 2) continue;
    if (phase == 2 && op.group != 2) continue;
    if (chunk >= 0 && op.chunk != chunk) continue;
    if (ablate && std::strchr(ablate, '0' + op.kind)) continue;
    if (op.kind == 0) {
      const MPLaunch& m = pl.mps[static_cast<size_t>(op.idx)];
      const LevelData& ld = b.side[m.side][static_cast<size_t>(m.level)];
      launch_mode_product(m.nsteps, pl.d_steps.p + m.step_begin, m.total_out, pl.d_blks.p, ld.interp.p,
                          in_ptr(m.in_buf), out_ptr(m.out_buf), st);
    } else if (op.kind == 1) {
      double2* y = pl.sharded ? io.send : scr;
      const GemvLaunch& gl = pl.gemvs[static_cast<size_t>(op.idx)];
      const GemvDesc* gd = pl.d_gemv.p + gl.desc_begin;
      if (pl.bfp)
        launch_gemv_bfp(pl.d_gemv_map.p + gl.map_begin, gd, gl.ctas, gl.total_rows, pl.d_gemv_rb.p + gl.rb_begin,
                        b.bfp_q.p, b.bfp_e.p, scr, y, gl.max_c, st);
      else if (gl.tma)
        launch_gemv_tma(pl.d_tma_map.p + gl.tma_map_begin, gd, gl.tma_ctas, gl.total_rows,
                        pl.d_gemv_rb.p + gl.tma_rb_begin, static_cast<int>(pl.nv), gl.tma_stages,
                        gl.tma_stage_elems, gl.tma_xcap, b.cores.p, scr, y, st);
      else
        launch_gemv(pl.d_gemv_map.p + gl.map_begin, gd, gl.ctas, gl.total_rows, pl.d_gemv_rb.p + gl.rb_begin,
                    static_cast<int>(pl.nv), b.cores.p, scr, y, gl.max_c, st);
    } else if (op.kind == 6) {
      const Plan::TinyLevel& tl = pl.tiny_levels[static_cast<size_t>(op.idx)];
      const LevelData& ld = b.side[tl.side][static_cast<size_t>(tl.l)];
      launch_tiny_level(tl.args, pl.d_tiny_groups.p + tl.group_begin, pl.d_tiny_off.p + tl.off_begin, ld.rank.p,
                        ld.width.p, ld.interp_off.p, ld.interp.p, in_ptr(tl.in_buf), out_ptr(tl.out_buf), st);
    } else if (op.kind == 8) {
      const Plan::R1Level& rl = pl.r1_levels[static_cast<size_t>(op.idx)];
      const LevelData& ld = b.side[rl.args.side][static_cast<size_t>(rl.args.l)];
      launch_r1_level(rl.args, ld.interp.p, b.cores.p, rl.in_off < 0 ? io.F : scr + rl.in_off,
                      rl.out_off < 0 ? io.G : scr + rl.out_off, st);
    } else if (op.kind == 9 || op.kind == 10) {
      const Plan::R1Level& rl = pl.r1_levels[static_cast<size_t>(op.idx)];
      if (op.kind == 9)
        launch_r1_exchange(rl.args, 0, reinterpret_cast<const long long*>(pl.d_r1_send_off.p), scr + rl.in_off,
                           io.send, st);
      else
        launch_r1_exchange(rl.args, 1, reinterpret_cast<const long long*>(pl.d_r1_recv_off.p), io.recv,
                           scr + rl.out_off, st);
    } else if (op.kind == 7) {
      const GemvLaunch& gl = pl.gemvs[static_cast<size_t>(op.idx)];
      launch_tiny_gemv(pl.d_gemv.p + gl.desc_begin, gl.ndesc, gl.total_rows, static_cast<int>(pl.nv), b.cores.p,
                       scr, scr, st);
    } else if (op.kind == 3) {
      const BoxLaunch& bx = pl.boxes[static_cast<size_t>(op.idx)];
      const LevelData& ld = b.side[bx.side][static_cast<size_t>(bx.level)];
      if (bx.box2)
        launch_box2(bx.nitems, pl.d_bdescs.p + bx.item_begin, bx.info, bx.smem2, ld.interp.p, in_ptr(bx.in_buf),
                    out_ptr(bx.out_buf), st);
      else
        launch_box(bx.nitems, pl.d_bdescs.p + bx.item_begin, bx.info, ld.interp.p, in_ptr(bx.in_buf),
                   out_ptr(bx.out_buf), st);
    } else {
      const SumLaunch& s = pl.sum_launches[static_cast<size_t>(op.idx)];
      launch_sum_children(s.n, pl.d_sums.p + s.begin, s.total, scr, scr, st);
    }
  }
}

void run_ops(oiobf_tbf& b, Plan& pl, const double2* F, double2* G, cudaStream_t st, int group_filter = -1) {
  OpBuffers io;
  io.F = F;
  io.G = G;
  run_ops(b, pl, io, st, group_filter, 0);
}

bool is_pinned(const void* p);

// Right-hand sides per contraction: beyond 4 vectors the box levels no longer
// stage their inputs on chip and the GEMV re-reads the cores per group of 4,
// so wider n_v runs as consecutive 4-vector contractions (F and G are
// n^d x n_v with vector stride n^d: each group is a contiguous slice).
// Measured (config 2, L2 flushed): 96 / 71 / 48 us per vector at n_v = 1 / 2 /
// 4; 65 / 64 / 61 at n_v = 8 / 16 / 32 as one plan.  OIOBF_NV_CHUNK overrides.
i64 nv_chunk() {
  static const i64 c = std::getenv("OIOBF_NV_CHUNK") ? std::atoll(std::getenv("OIOBF_NV_CHUNK")) : 4;
  return c > 0 ? c : 4;
}

// the plan's launches for io (phase 0: whole contraction, 1 / 2: sharded
// phases) captured into an instantiated graph
cudaGraphExec_t capture_io(oiobf_tbf& b, Plan& pl, const OpBuffers& io, int phase) {
  cudaStream_t cap;
  TBF_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  cudaGraph_t g;
  TBF_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
  try {
    run_ops(b, pl, io, cap, -1, phase);
  } catch (...) {
    cudaStreamEndCapture(cap, &g);
    cudaStreamDestroy(cap);
    throw;
  }
  TBF_CUDA(cudaStreamEndCapture(cap, &g));
  cudaGraphExec_t ex;
  TBF_CUDA(cudaGraphInstantiate(&ex, g, 0));
  TBF_CUDA(cudaGraphDestroy(g));
  TBF_CUDA(cudaStreamDestroy(cap));
  return ex;
}

cudaGraphExec_t capture_ops(oiobf_tbf& b, Plan& pl, const double2* F, double2* G, double2* scratch = nullptr) {
  cudaStream_t cap;
  TBF_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  cudaGraph_t g;
  TBF_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
  try {
    OpBuffers io;
    io.F = F;
    io.G = G;
    io.scratch = scratch;
    run_ops(b, pl, io, cap);
  } catch (...) {
    cudaStreamEndCapture(cap, &g);
    cudaStreamDestroy(cap);
    throw;
  }
  TBF_CUDA(cudaStreamEndCapture(cap, &g));
  cudaGraphExec_t ex;
  TBF_CUDA(cudaGraphInstantiate(&ex, g, 0));
  TBF_CUDA(cudaGraphDestroy(g));
  TBF_CUDA(cudaStreamDestroy(cap));
  return ex;
}

void contract_device(oiobf_tbf& b, const double2* F, double2* G, i64 nv, cudaStream_t st) {
  require(nv >= 1, "tbf_contract: nv must be >= 1");
  TBF_CUDA(cudaSetDevice(b.device));
  if (nv > nv_chunk() && b.world == 1) {
    const i64 N = ipow(b.n, b.d);
    Plan& pc = get_plan(b, nv_chunk());
    pc.dev_graphs.cap = std::max<size_t>(pc.dev_graphs.cap, static_cast<size_t>(2 * ((nv + nv_chunk() - 1) / nv_chunk())));
    for (i64 v0 = 0; v0 < nv; v0 += nv_chunk())
      contract_device(b, F + v0 * N, G + v0 * N, std::min(nv_chunk(), nv - v0), st);
    return;
  }
  Plan& pl = get_plan(b, nv);
  static const bool no_graph = std::getenv("OIOBF_NO_GRAPH") != nullptr;  // profiling aid
  if (no_graph) {
    run_ops(b, pl, F, G, st);
    return;
  }
  cudaGraphExec_t ex = pl.dev_graphs.find(F, G, st);
  if (!ex) {
    ex = capture_ops(b, pl, F, G);
    pl.dev_graphs.put(F, G, st, ex);
  }
  if (!pl.dev_done) TBF_CUDA(cudaEventCreateWithFlags(&pl.dev_done, cudaEventDisableTiming));
  if (pl.dev_used && pl.dev_last != st) TBF_CUDA(cudaStreamWaitEvent(st, pl.dev_done, 0));
  TBF_CUDA(cudaGraphLaunch(ex, st));
  TBF_CUDA(cudaEventRecord(pl.dev_done, st));
  pl.dev_last = st;
  pl.dev_used = true;
}

// Stream-ordered host-buffer contraction (pinned F and G): slot k of the plan
//   copy-in stream     [slot's previous compute done] H2D F -> slot.F  -> in
//   slot's compute     wait in, [slot's previous D2H done]; graph       -> done
//   copy-out stream    wait done; D2H slot.G -> G                        -> out
//   caller's stream    waits out
// Consecutive calls alternate slots, so the H2D of call k+1 overlaps the
// contraction of call k and the D2H of call k-1 (PCIe is full duplex).  Each
// slot has its own compute stream and scratch, so two contractions may also
// overlap each other (their box levels are latency-bound and leave the GPU
// mostly idle).  The caller's stream is never waited on before the copies
// (F is host memory the caller has finished writing when it makes the call).
void contract_host_async(oiobf_tbf& b, const double* F, double* G, i64 nv, cudaStream_t user) {
  require(nv >= 1, "tbf_contract_async: nv must be >= 1");
  TBF_CUDA(cudaSetDevice(b.device));
  if (nv > nv_chunk()) {
    const i64 N = ipow(b.n, b.d);
    for (i64 v0 = 0; v0 < nv; v0 += nv_chunk())
      contract_host_async(b, F + 2 * v0 * N, G + 2 * v0 * N, std::min(nv_chunk(), nv - v0), user);
    return;
  }
  require(is_pinned(F) && is_pinned(G),
          "tbf_contract_async: F and G must be pinned host memory (cudaHostAlloc / cudaHostRegister)");
  Plan& pl = get_plan(b, nv);
  if (!b.s_in) {
    TBF_CUDA(cudaStreamCreateWithFlags(&b.s_in, cudaStreamNonBlocking));
    TBF_CUDA(cudaStreamCreateWithFlags(&b.s_out, cudaStreamNonBlocking));
  }
  const int slot = pl.anext;
  AsyncSet& A = pl.aset[slot];
  pl.anext ^= 1;
  if (!b.s_cmp[slot]) TBF_CUDA(cudaStreamCreateWithFlags(&b.s_cmp[slot], cudaStreamNonBlocking));
  const size_t tot = static_cast<size_t>(ipow(b.n, b.d) * nv);
  if (A.F.n != tot) {
    if (A.used) TBF_CUDA(cudaEventSynchronize(A.out));
    if (A.gexec) {
      cudaGraphExecDestroy(A.gexec);
      A.gexec = nullptr;
    }
    A.F.alloc(tot);
    A.G.alloc(tot);
    A.scratch.alloc(static_cast<size_t>(std::max<i64>(pl.scratch_elems, 1)));
    A.used = false;
  }
  if (!A.in)
    for (cudaEvent_t* e : {&A.in, &A.done, &A.out, &A.user})
      TBF_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  // work the caller already enqueued on its stream (e.g. a consumer of the G
  // of an earlier call) precedes this call's D2H into G
  TBF_CUDA(cudaEventRecord(A.user, user));
  if (!A.gexec) A.gexec = capture_ops(b, pl, A.F.p, A.G.p, A.scratch.p);
  cudaStream_t cst = b.s_cmp[slot];
  if (A.used) TBF_CUDA(cudaStreamWaitEvent(b.s_in, A.done, 0));
  TBF_CUDA(cudaMemcpyAsync(A.F.p, F, tot * sizeof(double2), cudaMemcpyHostToDevice, b.s_in));
  TBF_CUDA(cudaEventRecord(A.in, b.s_in));
  TBF_CUDA(cudaStreamWaitEvent(cst, A.in, 0));
  if (A.used) TBF_CUDA(cudaStreamWaitEvent(cst, A.out, 0));
  TBF_CUDA(cudaGraphLaunch(A.gexec, cst));
  TBF_CUDA(cudaEventRecord(A.done, cst));
  TBF_CUDA(cudaStreamWaitEvent(b.s_out, A.done, 0));
  TBF_CUDA(cudaStreamWaitEvent(b.s_out, A.user, 0));
  TBF_CUDA(cudaMemcpyAsync(G, A.G.p, tot * sizeof(double2), cudaMemcpyDeviceToHost, b.s_out));
  TBF_CUDA(cudaEventRecord(A.out, b.s_out));
  TBF_CUDA(cudaStreamWaitEvent(user, A.out, 0));
  A.used = true;
}

// Host-buffer contraction, pipelined over the slab groups of mode d-1 (each
// group is one contiguous range of F and of G):
//   copy-in stream   H2D F[q]                      -> event in[q]
//   compute stream   wait in[q]; V/W + GEMV of group q   (q = 0 .. Q-1)
//                    P/U of group q               -> event out[q]
//   copy-out stream  wait out[q]; D2H G[q]
// so the PCIe copies overlap the V/W side and GEMV of earlier groups and the
// P/U side of later ones.  Pinned host buffers: captured once into a graph
// (copy nodes included) and replayed while the pointers stay the same.
void issue_pipeline(oiobf_tbf& b, Plan& pl, const double* F, double* G, cudaStream_t st) {
  const int Q = pl.nchunk;
  const i64 N = ipow(b.n, b.d);
  const size_t chunk_bytes = static_cast<size_t>(N / Q) * sizeof(double2);
  const size_t pitch = static_cast<size_t>(N) * sizeof(double2);
  const size_t nv = static_cast<size_t>(pl.nv);
  cudaEvent_t* ev = b.ev.data();  // [0] fork, [1] join, [2 + q] in, [2 + Q + q] out
  TBF_CUDA(cudaEventRecord(ev[0], st));
  TBF_CUDA(cudaStreamWaitEvent(b.s_in, ev[0], 0));
  TBF_CUDA(cudaStreamWaitEvent(b.s_out, ev[0], 0));
  char* dF = reinterpret_cast<char*>(pl.stage_F.p);
  char* dG = reinterpret_cast<char*>(pl.stage_G.p);
  for (int q = 0; q < Q; ++q) {
    TBF_CUDA(cudaMemcpy2DAsync(dF + q * chunk_bytes, pitch, reinterpret_cast<const char*>(F) + q * chunk_bytes, pitch,
                               chunk_bytes, nv, cudaMemcpyHostToDevice, b.s_in));
    TBF_CUDA(cudaEventRecord(ev[2 + q], b.s_in));
  }
  OpBuffers io;
  io.F = pl.stage_F.p;
  io.G = pl.stage_G.p;
  for (int q = 0; q < Q; ++q) {
    TBF_CUDA(cudaStreamWaitEvent(st, ev[2 + q], 0));
    run_ops(b, pl, io, st, -1, 1, q);
  }
  for (int q = 0; q < Q; ++q) {
    run_ops(b, pl, io, st, -1, 2, q);
    TBF_CUDA(cudaEventRecord(ev[2 + Q + q], st));
    TBF_CUDA(cudaStreamWaitEvent(b.s_out, ev[2 + Q + q], 0));
    TBF_CUDA(cudaMemcpy2DAsync(reinterpret_cast<char*>(G) + q * chunk_bytes, pitch, dG + q * chunk_bytes, pitch,
                               chunk_bytes, nv, cudaMemcpyDeviceToHost, b.s_out));
  }
  TBF_CUDA(cudaEventRecord(ev[1], b.s_out));
  TBF_CUDA(cudaStreamWaitEvent(st, ev[1], 0));
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void contract_host(oiobf_tbf& b, const double* F, double* G, i64 nv) {
  TBF_CUDA(cudaSetDevice(b.device));
  if (nv > nv_chunk()) {
    const i64 N = ipow(b.n, b.d);
    for (i64 v0 = 0; v0 < nv; v0 += nv_chunk())
      contract_host(b, F + 2 * v0 * N, G + 2 * v0 * N, std::min(nv_chunk(), nv - v0));
    return;
  }
  Plan& pl = get_plan(b, nv, true);
  const size_t N = static_cast<size_t>(ipow(b.n, b.d) * nv);
  if (pl.stage_F.n != N) {  // staging buffers persist so the captured graph is reused
    pl.stage_F.alloc(N);
    pl.stage_G.alloc(N);
  }
  if (!b.s_in) {
    TBF_CUDA(cudaStreamCreateWithFlags(&b.s_in, cudaStreamNonBlocking));
    TBF_CUDA(cudaStreamCreateWithFlags(&b.s_out, cudaStreamNonBlocking));
  }
  const size_t nev = 2 + 2 * static_cast<size_t>(pl.nchunk);
  while (b.ev.size() < nev) {
    cudaEvent_t e;
    TBF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    b.ev.push_back(e);
  }
  static const bool no_graph = std::getenv("OIOBF_NO_GRAPH") != nullptr;
  if (no_graph || !is_pinned(F) || !is_pinned(G)) {  // pageable memory cannot be captured
    issue_pipeline(b, pl, F, G, b.stream);
    TBF_CUDA(cudaStreamSynchronize(b.stream));
    return;
  }
  cudaGraphExec_t ex = pl.host_graphs.find(F, G, nullptr);
  if (!ex) {
    cudaGraph_t g;
    // global mode: the fork/join events pull the copy streams into the capture
    TBF_CUDA(cudaStreamBeginCapture(b.stream, cudaStreamCaptureModeThreadLocal));
    try {
      issue_pipeline(b, pl, F, G, b.stream);
    } catch (...) {
      cudaStreamEndCapture(b.stream, &g);
      throw;
    }
    TBF_CUDA(cudaStreamEndCapture(b.stream, &g));
    TBF_CUDA(cudaGraphInstantiate(&ex, g, 0));
    TBF_CUDA(cudaGraphDestroy(g));
    pl.host_graphs.put(F, G, nullptr, ex);
  }
  TBF_CUDA(cudaGraphLaunch(ex, b.stream));
  TBF_CUDA(cudaStreamSynchronize(b.stream));
}

// ---- TBF1 serialization: self-describing little-endian
// file: header (magic "TBF1", version, kernel spec, L, tol, proxy strategy,
// seed), then the factor blocks in canonical tree order (V/W levels 0..Lc,
// U/P levels 0..Lc: r_est, slot count, proxy rows, widest ID, ranks, widths,
// pivots, sorted skeletons, interps), then the cores (per pair R, C and the
// row-major R x C entries), then an FNV-1a 64-bit checksum of everything
// before it.  Round trips are bit-exact (tests/test_gpu_parity.py).
constexpr uint32_t kTbfVersion = 1;

struct TbfWriter {
  FILE* f;
  u64 h = 1469598103934665603ULL;
  void put(const void* p, size_t n) {
    const unsigned char* c = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ULL;
    if (n && std::fwrite(p, 1, n, f) != n) throw std::runtime_error("tbf_save: write failed");
  }
  template <class T>
  void v(T x) { put(&x, sizeof(T)); }
};

struct TbfReader {
  FILE* f;
  u64 h = 1469598103934665603ULL;
  void get(void* p, size_t n) {
    if (n && std::fread(p, 1, n, f) != n) throw InvalidArg("tbf_load: truncated file");
    const unsigned char* c = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ULL;
  }
  template <class T>
  T v() {
    T x;
    get(&x, sizeof(T));
    return x;
  }
};

void tbf_save(const oiobf_tbf& b, const char* path) {
  require(b.world == 1, "tbf_save: sharded factorizations are not serializable");
  FILE* f = std::fopen(path, "wb");
  if (!f) throw std::runtime_error(std::string("tbf_save: cannot open ") + path);
  TbfWriter w{f};
  try {
    cudaStream_t st = b.stream;
    w.put("TBF1", 4);
    w.v<uint32_t>(kTbfVersion);
    w.v<int32_t>(b.spec.kind);
    w.v<int32_t>(b.spec.d);
    w.v<int64_t>(b.spec.n);
    w.v<int32_t>(b.spec.bitrev);
    w.v<uint32_t>(b.spec.seed);
    w.v<double>(b.spec.kappa);
    for (int i = 0; i < 3; ++i) w.v<double>(b.spec.offset[i]);
    w.v<int32_t>(b.L);
    w.v<double>(b.tol);
    w.v<int32_t>(b.strat.mode);
    w.v<int64_t>(b.strat.q);
    w.v<int64_t>(b.strat.max_retries);
    w.v<int64_t>(b.strat.row_cap);
    w.v<uint64_t>(b.seed);
    for (int sd = 0; sd < 2; ++sd)
      for (int l = 0; l <= b.Lc; ++l) {
        const LevelData& ld = b.side[sd][static_cast<size_t>(l)];
        const i64 ns = ld.nslots;
        w.v<int64_t>(b.r_est[sd][static_cast<size_t>(l)]);
        w.v<int64_t>(ns);
        w.v<int64_t>(ld.L.m);
        w.v<int64_t>(ld.L.wmax);
        w.v<int64_t>(ld.total_skel);
        w.v<int64_t>(ld.total_interp);
        std::vector<int> perm(static_cast<size_t>(ns * ld.L.wmax)), skel(static_cast<size_t>(ld.total_skel));
        std::vector<double2> interp(static_cast<size_t>(ld.total_interp));
        ld.perm.download(perm.data(), perm.size(), st);
        ld.skel.download(skel.data(), skel.size(), st);
        ld.interp.download(interp.data(), interp.size(), st);
        TBF_CUDA(cudaStreamSynchronize(st));
        w.put(ld.h_rank.data(), sizeof(int) * static_cast<size_t>(ns));
        w.put(ld.h_width.data(), sizeof(int) * static_cast<size_t>(ns));
        w.put(perm.data(), sizeof(int) * perm.size());
        w.put(skel.data(), sizeof(int) * skel.size());
        w.put(interp.data(), sizeof(double2) * interp.size());
      }
    const i64 P = static_cast<i64>(b.h_pairs.size());
    w.v<int64_t>(P);
    w.v<int64_t>(b.total_core);
    for (const PairDesc& pd : b.h_pairs) {
      w.v<int32_t>(pd.R);
      w.v<int32_t>(pd.C);
    }
    std::vector<double2> cores(static_cast<size_t>(b.total_core));
    b.cores.download(cores.data(), cores.size(), st);
    TBF_CUDA(cudaStreamSynchronize(st));
    w.put(cores.data(), sizeof(double2) * cores.size());
    const u64 sum = w.h;
    if (std::fwrite(&sum, sizeof(sum), 1, f) != 1) throw std::runtime_error("tbf_save: write failed");
  } catch (...) {
    std::fclose(f);
    throw;
  }
  if (std::fclose(f) != 0) throw std::runtime_error("tbf_save: close failed");
}

oiobf_tbf* tbf_load(const char* path) {
  FILE* f = std::fopen(path, "rb");
  if (!f) throw InvalidArg(std::string("tbf_load: cannot open ") + path);
  TbfReader r{f};
  std::unique_ptr<oiobf_tbf> b;
  try {
    char magic[4];
    r.get(magic, 4);
    require(std::memcmp(magic, "TBF1", 4) == 0, "tbf_load: not a TBF1 file");
    require(r.v<uint32_t>() == kTbfVersion, "tbf_load: unsupported TBF1 version");
    oiobf_kernel_spec spec{};
    spec.kind = r.v<int32_t>();
    spec.d = r.v<int32_t>();
    spec.n = r.v<int64_t>();
    spec.bitrev = r.v<int32_t>();
    spec.seed = r.v<uint32_t>();
    spec.kappa = r.v<double>();
    for (int i = 0; i < 3; ++i) spec.offset[i] = r.v<double>();
    const int L = r.v<int32_t>();
    const double tol = r.v<double>();
    oiobf_proxy_strategy ps{};
    ps.mode = r.v<int32_t>();
    ps.q = r.v<int64_t>();
    ps.max_retries = r.v<int64_t>();
    ps.row_cap = r.v<int64_t>();
    const u64 seed = r.v<uint64_t>();
    b = construct_begin(spec, L, tol, ps, seed, 0, 1);
    cudaStream_t st = b->stream;
    for (int sd = 0; sd < 2; ++sd)
      for (int l = 0; l <= b->Lc; ++l) {
        const i64 r_est = r.v<int64_t>(), ns = r.v<int64_t>(), m = r.v<int64_t>(), wmax = r.v<int64_t>();
        const i64 tsk = r.v<int64_t>(), tip = r.v<int64_t>();
        LevelData& ld = b->side[sd][static_cast<size_t>(l)];
        ld.L = make_level(*b, sd, l, r_est, wmax);
        require(ld.L.nslots == ns && ld.L.m == m && wmax >= 1 && wmax <= kMaxW, "tbf_load: level shape mismatch");
        b->r_est[sd].push_back(r_est);
        ld.nslots = ns;
        ld.h_rank.resize(static_cast<size_t>(ns));
        ld.h_width.resize(static_cast<size_t>(ns));
        ld.h_sat.assign(static_cast<size_t>(ns), 0);
        std::vector<int> perm(static_cast<size_t>(ns * wmax)), skel(static_cast<size_t>(tsk));
        std::vector<double2> interp(static_cast<size_t>(tip));
        r.get(ld.h_rank.data(), sizeof(int) * static_cast<size_t>(ns));
        r.get(ld.h_width.data(), sizeof(int) * static_cast<size_t>(ns));
        r.get(perm.data(), sizeof(int) * perm.size());
        r.get(skel.data(), sizeof(int) * skel.size());
        r.get(interp.data(), sizeof(double2) * interp.size());
        ld.h_skel_off.resize(static_cast<size_t>(ns));
        ld.h_interp_off.resize(static_cast<size_t>(ns));
        i64 so = 0, io = 0;
        ld.max_rank = 0;
        for (i64 i = 0; i < ns; ++i) {
          const int rk = ld.h_rank[static_cast<size_t>(i)], wd = ld.h_width[static_cast<size_t>(i)];
          require(rk >= 0 && wd >= rk && wd <= wmax, "tbf_load: bad rank / width");
          ld.h_skel_off[static_cast<size_t>(i)] = so;
          ld.h_interp_off[static_cast<size_t>(i)] = io;
          so += rk;
          io += static_cast<i64>(rk) * wd;
          ld.max_rank = std::max(ld.max_rank, rk);
        }
        require(so == tsk && io == tip, "tbf_load: skeleton / interp sizes disagree with the ranks");
        ld.total_skel = tsk;
        ld.total_interp = tip;
        ld.rank = to_device(ld.h_rank, st);
        ld.width = to_device(ld.h_width, st);
        ld.perm = to_device(perm, st);
        ld.gaps.alloc(static_cast<size_t>(ns));
        ld.skel_off = to_device(ld.h_skel_off, st);
        ld.interp_off = to_device(ld.h_interp_off, st);
        ld.skel.alloc(static_cast<size_t>(std::max<i64>(tsk, 1)));
        ld.skel.upload(skel.data(), skel.size(), st);
        ld.interp.alloc(static_cast<size_t>(std::max<i64>(tip, 1)));
        ld.interp.upload(interp.data(), interp.size(), st);
        TBF_CUDA(cudaStreamSynchronize(st));
      }
    const i64 P = r.v<int64_t>(), tc = r.v<int64_t>();
    const i64 off = layout_pairs(*b);
    require(P == static_cast<i64>(b->h_pairs.size()) && tc == off, "tbf_load: core layout mismatch");
    for (const PairDesc& pd : b->h_pairs) {
      const int R = r.v<int32_t>(), C = r.v<int32_t>();
      require(R == pd.R && C == pd.C, "tbf_load: core shape mismatch");
    }
    std::vector<double2> cores(static_cast<size_t>(tc));
    r.get(cores.data(), sizeof(double2) * cores.size());
    const u64 expect = r.h;
    u64 sum = 0;
    if (std::fread(&sum, sizeof(sum), 1, f) != 1) throw InvalidArg("tbf_load: truncated file");
    require(sum == expect, "tbf_load: checksum mismatch");
    b->cores.alloc(static_cast<size_t>(std::max<i64>(tc, 1)));
    b->cores.upload(cores.data(), cores.size(), st);
    TBF_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    std::fclose(f);
    throw;
  }
  std::fclose(f);
  return b.release();
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
  std::vector<int> tmp(static_cast<size_t>(mode == OIOBF_PROXY_ALL ? extent : c));
  i64 got = 0;
  if (mode == OIOBF_PROXY_UNIFORM_RANDOM && c > kMaxProxy) {  // full pool (id.cpp:171-181)
    std::vector<int> pool(static_cast<size_t>(extent));
    for (i64 i = 0; i < extent; ++i) pool[static_cast<size_t>(i)] = static_cast<int>(i + 1);
    u64 st = seed;
    for (i64 i = 0; i < c; ++i) {
      const i64 j = i + static_cast<i64>(splitmix_bounded(st, static_cast<u64>(extent - i)));
      std::swap(pool[static_cast<size_t>(i)], pool[static_cast<size_t>(j)]);
    }
    std::copy(pool.begin(), pool.begin() + c, tmp.begin());
    std::sort(tmp.begin(), tmp.end());
    got = c;
  } else {
    got = select_proxies(extent, count, mode, seed, tmp.data());
  }
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

int oiobf_tbf_shard_set_owners(oiobf_tbf* h, const int32_t* owners) {
  CAPI_BEGIN
  require(h && owners, "tbf_shard_set_owners: null argument");
  require(h->r_est[0].empty() && h->r_est[1].empty(), "tbf_shard_set_owners: call before the first level is built");
  std::vector<int> own(static_cast<size_t>(h->nmid));
  for (i64 o = 0; o < h->nmid; ++o) {
    require(owners[o] >= 0 && owners[o] < h->world, "tbf_shard_set_owners: owner out of range");
    own[static_cast<size_t>(o)] = owners[o];
  }
  TBF_CUDA(cudaSetDevice(h->device));
  h->d_owner = to_device(own, h->stream);
  TBF_CUDA(cudaStreamSynchronize(h->stream));
  h->owner = std::move(own);
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
  h->sync_all();
  h->plans.clear();
  h->r1_ok = -1;  // the sharded rank-one engine needs the exchange tables
  CAPI_END
}

int oiobf_tbf_set_peer_exchange(oiobf_tbf* h, const int64_t* peer_off, const uint64_t* recv_base, int32_t world,
                                int64_t nv_max) {
  CAPI_BEGIN
  require(h, "tbf_set_peer_exchange: null handle");
  if (!recv_base) {  // back to the send buffer + all-to-all path
    std::lock_guard<std::mutex> lk(h->mu);
    h->sync_all();
    h->plans.clear();
    h->r1_ok = -1;
    h->peer_off.clear();
    h->peer_base.clear();
    h->peer_nv_max = 0;
    return OIOBF_OK;
  }
  require(peer_off, "tbf_set_peer_exchange: null argument");
  require(world == h->world && world > 1, "tbf_set_peer_exchange: world must match the sharded factorization");
  require(nv_max >= 1, "tbf_set_peer_exchange: nv_max must be >= 1");
  std::lock_guard<std::mutex> lk(h->mu);
  const i64 P = h->nmid * h->nmid;
  h->sync_all();
  h->plans.clear();
  h->peer_off.assign(peer_off, peer_off + P);
  h->peer_base.assign(recv_base, recv_base + 2 * world);
  h->peer_nv_max = nv_max;
  for (u64 a : h->peer_base) require(a != 0 && a % 16 == 0, "tbf_set_peer_exchange: bad receive buffer address");
  CAPI_END
}

int oiobf_device_alloc(int64_t bytes, void** out) {
  CAPI_BEGIN
  require(out && bytes > 0, "device_alloc: bad argument");
  ensure_device();
  TBF_CUDA(cudaMalloc(out, static_cast<size_t>(bytes)));
  CAPI_END
}

int oiobf_device_free(void* p) {
  CAPI_BEGIN
  if (p) TBF_CUDA(cudaFree(p));
  CAPI_END
}

int oiobf_ipc_handle(void* p, uint8_t handle[64]) {
  CAPI_BEGIN
  require(p && handle, "ipc_handle: null argument");
  cudaIpcMemHandle_t hd;
  TBF_CUDA(cudaIpcGetMemHandle(&hd, p));
  static_assert(sizeof(hd) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle, &hd, 64);
  CAPI_END
}

int oiobf_ipc_open(const uint8_t handle[64], void** out) {
  CAPI_BEGIN
  require(handle && out, "ipc_open: null argument");
  ensure_device();
  cudaIpcMemHandle_t hd;
  std::memcpy(&hd, handle, 64);
  TBF_CUDA(cudaIpcOpenMemHandle(out, hd, cudaIpcMemLazyEnablePeerAccess));
  CAPI_END
}

int oiobf_ipc_close(void* p) {
  CAPI_BEGIN
  if (p) TBF_CUDA(cudaIpcCloseMemHandle(p));
  CAPI_END
}

int oiobf_memcpy(void* dst, const void* src, int64_t bytes) {
  CAPI_BEGIN
  require(bytes >= 0 && (bytes == 0 || (dst && src)), "memcpy: bad argument");
  ensure_device();
  if (bytes) TBF_CUDA(cudaMemcpy(dst, src, static_cast<size_t>(bytes), cudaMemcpyDefault));
  CAPI_END
}

int oiobf_tbf_copy_owned(oiobf_tbf* h, int32_t dir, const void* src, void* dst, int64_t nv, void* stream) {
  CAPI_BEGIN
  require(h && src && dst, "tbf_copy_owned: null argument");
  require(dir == 0 || dir == 1, "tbf_copy_owned: dir must be 0 (F in) or 1 (G out)");
  require(nv >= 1, "tbf_copy_owned: nv must be >= 1");
  TBF_CUDA(cudaSetDevice(h->device));
  const int d = h->d;
  const i64 n = h->n, mpm = ipow(2, h->Lc), mid = n >> h->Lc, N = ipow(n, d);
  // modes 0..2 as one 3D copy (x = mode 0 contiguous), the rest looped
  const int d3 = std::min(d, 3);
  i64 outer_cnt = nv;
  for (int k = 3; k < d; ++k) outer_cnt *= mid;
  for (i64 o = 0; o < h->nmid; ++o) {
    if (!h->owns(o)) continue;
    i64 base = 0, st = 1;
    for (int k = 0; k < d; ++k) {
      base += ((o / ipow(mpm, k)) % mpm) * mid * st;
      st *= n;
    }
    for (i64 q = 0; q < outer_cnt; ++q) {
      i64 off = base, rem = q;
      for (int k = 3; k < d; ++k) {
        off += (rem % mid) * ipow(n, k);
        rem /= mid;
      }
      off += rem * N;  // vector index
      cudaMemcpy3DParms p = {};
      const size_t pitch = static_cast<size_t>(n) * 16;
      p.srcPtr = make_cudaPitchedPtr(const_cast<char*>(static_cast<const char*>(src)) + 16 * off, pitch,
                                     static_cast<size_t>(n), static_cast<size_t>(d > 1 ? n : 1));
      p.dstPtr = make_cudaPitchedPtr(static_cast<char*>(dst) + 16 * off, pitch, static_cast<size_t>(n),
                                     static_cast<size_t>(d > 1 ? n : 1));
      p.extent = make_cudaExtent(static_cast<size_t>(mid) * 16, static_cast<size_t>(d3 > 1 ? mid : 1),
                                 static_cast<size_t>(d3 > 2 ? mid : 1));
      p.kind = cudaMemcpyDefault;
      TBF_CUDA(cudaMemcpy3DAsync(&p, static_cast<cudaStream_t>(stream)));
    }
  }
  CAPI_END
}

int oiobf_synchronize(void) {
  CAPI_BEGIN
  ensure_device();
  TBF_CUDA(cudaDeviceSynchronize());
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
  int parity = 0;
  if (h->peer_mode() && phase == 1) {  // dOut names the parity: this rank's own receive buffer
    const u64 a = reinterpret_cast<u64>(dOut);
    const u64 own0 = h->peer_base[static_cast<size_t>(h->rank)];
    const u64 own1 = h->peer_base[static_cast<size_t>(h->world + h->rank)];
    require(a == own0 || a == own1,
            "tbf_contract_phase: with a fused exchange, phase 1 writes this rank's own receive buffer");
    require(nv <= h->peer_nv_max, "tbf_contract_phase: nv exceeds the receive buffers (nv_max)");
    parity = a == own0 ? 0 : 1;
  }
  Plan& pl = get_plan(*h, nv, false, parity);
  OpBuffers io;
  if (phase == 1) {
    io.F = static_cast<const double2*>(dIn);
    io.send = static_cast<double2*>(dOut);
  } else {
    io.recv = static_cast<const double2*>(dIn);
    io.G = static_cast<double2*>(dOut);
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  static const bool no_graph = std::getenv("OIOBF_NO_GRAPH") != nullptr;  // profiling aid
  if (no_graph) {
    run_ops(*h, pl, io, st, -1, phase);
  } else {  // one captured graph per (phase, input, output, stream)
    auto& gc = pl.phase_graphs[phase - 1];
    cudaGraphExec_t ex = gc.find(dIn, dOut, st);
    if (!ex) {
      ex = capture_io(*h, pl, io, phase);
      gc.put(dIn, dOut, st, ex);
    }
    if (!pl.dev_done) TBF_CUDA(cudaEventCreateWithFlags(&pl.dev_done, cudaEventDisableTiming));
    if (pl.dev_used && pl.dev_last != st) TBF_CUDA(cudaStreamWaitEvent(st, pl.dev_done, 0));
    TBF_CUDA(cudaGraphLaunch(ex, st));
    TBF_CUDA(cudaEventRecord(pl.dev_done, st));
    pl.dev_last = st;
    pl.dev_used = true;
  }
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
  require(h->world == 1, "tbf_contract: sharded factorization -- use oiobf_tbf_contract_phase");
  std::lock_guard<std::mutex> lk(h->mu);
  contract_host(*h, F, G, nv);
  CAPI_END
}

int oiobf_tbf_contract_async(oiobf_tbf* h, const double* F, double* G, int64_t nv, void* stream) {
  CAPI_BEGIN
  require(h && F && G, "tbf_contract_async: null argument");
  require(h->world == 1, "tbf_contract_async: sharded factorization -- use oiobf_tbf_contract_phase");
  std::lock_guard<std::mutex> lk(h->mu);
  contract_host_async(*h, F, G, nv, static_cast<cudaStream_t>(stream));
  CAPI_END
}

int oiobf_tbf_save(const oiobf_tbf* h, const char* path) {
  CAPI_BEGIN
  require(h && path, "tbf_save: null argument");
  std::lock_guard<std::mutex> lk(const_cast<oiobf_tbf*>(h)->mu);
  TBF_CUDA(cudaSetDevice(h->device));
  tbf_save(*h, path);
  CAPI_END
}

int oiobf_tbf_load(const char* path, oiobf_tbf** out) {
  CAPI_BEGIN
  require(path && out, "tbf_load: null argument");
  *out = tbf_load(path);
  CAPI_END
}

namespace {
// Block-floating-point copy of the cores (k_bfp_compress, one warp per block
// of 32 entries of a row).  Pairs this rank does not own have C = 0.
void compress_cores_bfp(oiobf_tbf& b) {
  cudaStream_t st = b.stream;
  const i64 P = b.nmid * b.nmid;
  std::vector<long long> blk_prefix(static_cast<size_t>(P)), q_off(static_cast<size_t>(P));
  std::vector<GemvDesc> raw(static_cast<size_t>(P));
  b.bfp_off.assign(static_cast<size_t>(P), 0);
  i64 blocks = 0;
  for (i64 p = 0; p < P; ++p) {
    const PairDesc& pd = b.h_pairs[static_cast<size_t>(p)];
    GemvDesc g{};
    g.core_off = pd.core_off;
    g.R = pd.R;
    g.C = pd.C;
    raw[static_cast<size_t>(p)] = g;
    blk_prefix[static_cast<size_t>(p)] = blocks;
    q_off[static_cast<size_t>(p)] = blocks * 32;
    b.bfp_off[static_cast<size_t>(p)] = blocks * 32;
    if (pd.C > 0) blocks += static_cast<i64>(pd.R) * ((pd.C + 31) / 32);
  }
  b.bfp_entries = blocks * 32;
  b.bfp_q.alloc(static_cast<size_t>(std::max<i64>(b.bfp_entries, 32)));
  b.bfp_e.alloc(static_cast<size_t>(std::max<i64>(blocks, 1)));
  DevBuf<long long> d_prefix = to_device(blk_prefix, st), d_qoff = to_device(q_off, st);
  DevBuf<GemvDesc> d_raw = to_device(raw, st);
  launch_bfp_compress(d_prefix.p, P, d_raw.p, d_qoff.p, blocks, b.cores.p, b.bfp_q.p, b.bfp_e.p, st);
  TBF_CUDA(cudaStreamSynchronize(st));
}
}  // namespace

// 0 = FP64 cores (exact; default), 1 = block floating point (32-bit mantissas,
// one 16-bit exponent per 32 entries of a core row: half the core bytes, each
// entry within 2^-31 of its block's largest component; used by the n_v = 1
// core GEMV).  The FP64 cores stay resident; switching rebuilds the plans.
int oiobf_tbf_set_core_format(oiobf_tbf* h, int32_t format) {
  CAPI_BEGIN
  require(h, "tbf_set_core_format: null handle");
  require(format == 0 || format == 1, "tbf_set_core_format: format must be 0 (fp64) or 1 (block floating point)");
  std::lock_guard<std::mutex> lk(h->mu);
  TBF_CUDA(cudaSetDevice(h->device));
  if (format == h->core_format) return OIOBF_OK;
  h->sync_all();
  if (format == 1) {
    require(!use_r1_engine(*h), "tbf_set_core_format: the rank-one engine keeps its 1 x 1 cores in FP64");
    if (h->bfp_off.empty()) compress_cores_bfp(*h);
  }
  h->plans.clear();
  h->core_format = format;
  CAPI_END
}

int oiobf_tbf_set_apply_engine(oiobf_tbf* h, int32_t engine) {
  CAPI_BEGIN
  require(h, "tbf_set_apply_engine: null handle");
  require(engine >= 0 && engine <= 4 && engine != 3,
          "tbf_set_apply_engine: engine must be 0 (auto), 1 (box), 2 (tiny) or 4 (rank-one)");
  std::lock_guard<std::mutex> lk(h->mu);
  if (h->apply_engine != engine) {
    h->sync_all();
    h->plans.clear();
    h->apply_engine = engine;
  }
  CAPI_END
}

int oiobf_tbf_apply_engine(oiobf_tbf* h, int32_t* engine) {
  CAPI_BEGIN
  require(h && engine, "tbf_apply_engine: null argument");
  std::lock_guard<std::mutex> lk(h->mu);
  if (use_r1_engine(*h)) {
    *engine = 4;
  } else if (use_tiny_engine(*h)) {
    *engine = 2;
  } else {
    TBF_CUDA(cudaSetDevice(h->device));
    *engine = 1;
  }
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
    std::vector<double2> hc(cores ? static_cast<size_t>(h->total_core) : 0);
    if (cores) h->cores.download(hc.data(), hc.size(), st);
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

// Cores of selected middle pairs only (sorted pair indices p = s * nmid + t):
// core_rows / core_cols for every pair, with core_cols = 0 for pairs not
// selected, and the selected cores in the reference's column-major
// matricization, packed in pair order -- a valid tbf_import core set for an
// input supported on the selected pairs' column blocks (config 5's 95 GB of
// cores are checked block-wise this way).
int oiobf_tbf_export_cores(const oiobf_tbf* h, int64_t nsel, const int64_t* sel, double* cores, int64_t* core_rows,
                           int64_t* core_cols) {
  CAPI_BEGIN
  require(h && sel && cores && core_rows && core_cols, "tbf_export_cores: null argument");
  TBF_CUDA(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  const i64 P = static_cast<i64>(h->h_pairs.size());
  for (i64 p = 0; p < P; ++p) {
    core_rows[p] = h->h_pairs[static_cast<size_t>(p)].R;
    core_cols[p] = 0;
  }
  i64 o = 0;
  std::vector<double2> hc;
  for (i64 q = 0; q < nsel; ++q) {
    const i64 p = sel[q];
    require(p >= 0 && p < P && (q == 0 || p > sel[q - 1]), "tbf_export_cores: pair list must be sorted and in range");
    const PairDesc& pd = h->h_pairs[static_cast<size_t>(p)];
    core_cols[p] = pd.C;
    hc.resize(static_cast<size_t>(pd.R) * pd.C);
    TBF_CUDA(cudaMemcpyAsync(hc.data(), h->cores.p + pd.core_off, hc.size() * sizeof(double2), cudaMemcpyDeviceToHost,
                             st));
    TBF_CUDA(cudaStreamSynchronize(st));
    for (int r = 0; r < pd.R; ++r)
      for (int c = 0; c < pd.C; ++c) {
        const double2 v = hc[static_cast<size_t>(r) * pd.C + c];
        const i64 e = o + r + static_cast<i64>(c) * pd.R;
        cores[2 * e] = v.x;
        cores[2 * e + 1] = v.y;
      }
    o += static_cast<i64>(pd.R) * pd.C;
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
  // cores as the GEMV reads them: FP64, or 8 B per entry + 2 B per 32-entry block
  const i64 core_bytes = pl.bfp ? 8 * h->bfp_entries + 2 * (h->bfp_entries / 32) : 16 * h->total_core;
  out[0] = 16 * (2 * N + fac) + core_bytes;
  out[1] = core_bytes;
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

// FP64 peaks of this device (bench roofline denominators): out[0] DFMA
// TFLOP/s, out[1] DMMA (mma.sync f64) TFLOP/s, out[2] SMs, out[3] SM MHz
int oiobf_fp64_peak(double* out) {
  CAPI_BEGIN
  require(out, "fp64_peak: null argument");
  ensure_device();
  measure_fp64_peak(out);
  CAPI_END
}

// Cold-L2 timing of the core-contraction phase alone: before each of `reps`
// single launches the caller's flush buffer (larger than the 126 MB L2) is
// overwritten on the same stream; out = mean launch time in ms.
int oiobf_tbf_profile_core_cold(oiobf_tbf* h, const void* dF, void* dG, int32_t reps, void* stream, void* flush,
                                int64_t flush_bytes, double* out) {
  CAPI_BEGIN
  require(h && dF && dG && flush && out && reps >= 1 && flush_bytes > 0, "tbf_profile_core_cold: bad argument");
  std::lock_guard<std::mutex> lk(h->mu);
  TBF_CUDA(cudaSetDevice(h->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Plan& pl = get_plan(*h, 1);
  for (int g = 0; g < 3; ++g)  // full warm pass: the core phase's input is the V/W output in scratch
    run_ops(*h, pl, static_cast<const double2*>(dF), static_cast<double2*>(dG), st, g);
  double tot = 0;
  for (int r = 0; r < reps; ++r) {
    TBF_CUDA(cudaMemsetAsync(flush, r & 0xff, static_cast<size_t>(flush_bytes), st));
    EventTimer t(st);
    run_ops(*h, pl, static_cast<const double2*>(dF), static_cast<double2*>(dG), st, 1);
    tot += t.stop();
  }
  *out = tot / reps;
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
  // matrices of up to kMaxW columns: TSQR + reference pivoting on R in shared
  // memory (k_matrix_panel / k_finish); wider ones: the pivoted Householder QR
  // in global memory (k_qrcp_wide)
  std::vector<i64> narrow, wide;
  i64 wmax = 1, mmax = 1, atot = 0;
  for (i64 b = 0; b < batch; ++b) {
    require(m[b] > 0 && n[b] > 0, "column_id: empty matrix");
    require(n[b] < (i64{1} << 30) && m[b] < (i64{1} << 40), "column_id: matrix too large");
    atot = std::max<i64>(atot, a_off[b] + m[b] * n[b]);
    if (n[b] <= kMaxW) {
      narrow.push_back(b);
      wmax = std::max<i64>(wmax, n[b]);
      mmax = std::max<i64>(mmax, m[b]);
    } else {
      wide.push_back(b);
    }
  }
  cudaStream_t st;
  TBF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  {
    DevBuf<double2> dA(static_cast<size_t>(atot));
    dA.upload(reinterpret_cast<const double2*>(A), static_cast<size_t>(atot), st);
    if (!narrow.empty()) {
      const i64 nb = static_cast<i64>(narrow.size());
      LevelDesc L{};
      L.d = 1;
      L.nslots = nb;
      L.wmax = wmax;
      L.m = mmax;
      L.pr = wmax <= 16 ? 256 : wmax <= 64 ? 128 : 64;  // R packed: (w(w+1)/2 + pr w) x 16 B fits the 220 KB budget
      if (const char* e = std::getenv("OIOBF_ID_PR")) L.pr = std::atoi(e);  // debug override
      i64 parts = std::max<i64>(1, (148 * 8 + nb - 1) / nb);
      parts = std::min(parts, std::max<i64>(1, (mmax + 4 * L.pr - 1) / (4 * L.pr)));
      if (const char* e = std::getenv("OIOBF_ID_NPARTS")) parts = std::atoi(e);  // debug override
      L.nparts = parts;
      L.rpp = (mmax + parts - 1) / parts;
      std::vector<int> hw(static_cast<size_t>(nb)), ht(static_cast<size_t>(nb * wmax));
      std::vector<i64> hm(static_cast<size_t>(nb)), hoff(static_cast<size_t>(nb)), hmr(static_cast<size_t>(nb));
      std::vector<int> hn(static_cast<size_t>(nb));
      for (i64 q = 0; q < nb; ++q) {
        const i64 b = narrow[static_cast<size_t>(q)];
        hm[static_cast<size_t>(q)] = m[b];
        hoff[static_cast<size_t>(q)] = a_off[b];
        hw[static_cast<size_t>(q)] = static_cast<int>(n[b]);
        hn[static_cast<size_t>(q)] = static_cast<int>(n[b]);
        hmr[static_cast<size_t>(q)] = max_rank ? max_rank[b] : -1;
        for (i64 c = 0; c < n[b]; ++c) ht[static_cast<size_t>(q * wmax + c)] = static_cast<int>(c + 1);
      }
      DevBuf<int> dw = to_device(hw, st), dt = to_device(ht, st), dn = to_device(hn, st);
      DevBuf<i64> dm = to_device(hm, st), doff = to_device(hoff, st), dmr = to_device(hmr, st);
      DevBuf<double2> rpart(static_cast<size_t>(nb * L.nparts * wmax * wmax));
      launch_matrix_ids(nb, doff.p, dm.p, dn.p, dA.p, L.nparts, L.rpp, L.pr, wmax, rpart.p, st);
      DevBuf<int> drank(static_cast<size_t>(nb)), dsat(static_cast<size_t>(nb)),
          dperm(static_cast<size_t>(nb * wmax)), dsk(static_cast<size_t>(nb * wmax));
      DevBuf<double2> dint(static_cast<size_t>(nb * wmax * wmax));
      DevBuf<double> dgap(static_cast<size_t>(nb));
      launch_finish_var(L, dm.p, tol, kTieEps, dmr.p, rpart.p, dt.p, dw.p, drank.p, dsat.p, dperm.p, dsk.p, dint.p,
                        dgap.p, st);
      std::vector<int> hr(static_cast<size_t>(nb)), hs(static_cast<size_t>(nb)),
          hp(static_cast<size_t>(nb * wmax)), hk(static_cast<size_t>(nb * wmax));
      std::vector<double2> hi(static_cast<size_t>(nb * wmax * wmax));
      drank.download(hr.data(), hr.size(), st);
      dsat.download(hs.data(), hs.size(), st);
      dperm.download(hp.data(), hp.size(), st);
      dsk.download(hk.data(), hk.size(), st);
      dint.download(hi.data(), hi.size(), st);
      TBF_CUDA(cudaStreamSynchronize(st));
      for (i64 q = 0; q < nb; ++q) {
        const i64 b = narrow[static_cast<size_t>(q)];
        const int r = hr[static_cast<size_t>(q)];
        const i64 w = n[b];
        rank[b] = r;
        if (saturated) saturated[b] = hs[static_cast<size_t>(q)];
        double mx = 0;
        for (i64 e = 0; e < r * w; ++e) {
          const double2 v = hi[static_cast<size_t>(q * wmax * wmax + e)];
          interp[2 * (i_off[b] + e)] = v.x;
          interp[2 * (i_off[b] + e) + 1] = v.y;
          mx = std::max(mx, std::sqrt(v.x * v.x + v.y * v.y));
        }
        if (interp_max_abs) interp_max_abs[b] = (r > 0) ? mx : 0.0;
        for (int e = 0; e < r; ++e) skel[s_off[b] + e] = hk[static_cast<size_t>(q * wmax + e)];
        if (perm)
          for (i64 e = 0; e < w; ++e) perm[s_off[b] + e] = hp[static_cast<size_t>(q * wmax + e)];
      }
    }
    if (!wide.empty()) {
      const i64 nw = static_cast<i64>(wide.size());
      std::vector<WideIdJob> jobs(static_cast<size_t>(nw));
      i64 ntot = 0, itot = 0;
      for (i64 q = 0; q < nw; ++q) {
        const i64 b = wide[static_cast<size_t>(q)];
        WideIdJob& J = jobs[static_cast<size_t>(q)];
        J.a_off = a_off[b];
        J.m = m[b];
        J.n = static_cast<int>(n[b]);
        J.max_rank = max_rank ? max_rank[b] : -1;
        J.n_off = ntot;
        J.i_off = itot;
        J.pad = 0;
        ntot += n[b];
        itot += std::min(m[b], n[b]) * n[b];
      }
      DevBuf<WideIdJob> djobs = to_device(jobs, st);
      DevBuf<double> dnrm(static_cast<size_t>(ntot));
      DevBuf<int> dperm(static_cast<size_t>(ntot)), dpos(static_cast<size_t>(ntot)), dsk(static_cast<size_t>(ntot)),
          drank(static_cast<size_t>(nw)), dsat(static_cast<size_t>(nw));
      DevBuf<double2> dint(static_cast<size_t>(std::max<i64>(itot, 1)));
      launch_wide_ids(nw, djobs.p, dA.p, dnrm.p, dperm.p, dpos.p, tol, drank.p, dsat.p, dsk.p, dint.p, st);
      std::vector<int> hr(static_cast<size_t>(nw)), hs(static_cast<size_t>(nw)), hp(static_cast<size_t>(ntot)),
          hk(static_cast<size_t>(ntot));
      drank.download(hr.data(), hr.size(), st);
      dsat.download(hs.data(), hs.size(), st);
      dperm.download(hp.data(), hp.size(), st);
      dsk.download(hk.data(), hk.size(), st);
      TBF_CUDA(cudaStreamSynchronize(st));
      for (i64 q = 0; q < nw; ++q) {
        const i64 b = wide[static_cast<size_t>(q)];
        const WideIdJob& J = jobs[static_cast<size_t>(q)];
        const int r = hr[static_cast<size_t>(q)];
        const i64 w = n[b];
        rank[b] = r;
        if (saturated) saturated[b] = hs[static_cast<size_t>(q)];
        std::vector<double2> hi(static_cast<size_t>(std::max<i64>(r * w, 1)));
        if (r > 0) {
          TBF_CUDA(cudaMemcpyAsync(hi.data(), dint.p + J.i_off, sizeof(double2) * static_cast<size_t>(r * w),
                                   cudaMemcpyDeviceToHost, st));
          TBF_CUDA(cudaStreamSynchronize(st));
        }
        double mx = 0;
        for (i64 e = 0; e < r * w; ++e) {
          const double2 v = hi[static_cast<size_t>(e)];
          interp[2 * (i_off[b] + e)] = v.x;
          interp[2 * (i_off[b] + e) + 1] = v.y;
          mx = std::max(mx, std::sqrt(v.x * v.x + v.y * v.y));
        }
        if (interp_max_abs) interp_max_abs[b] = (r > 0) ? mx : 0.0;
        for (int e = 0; e < r; ++e) skel[s_off[b] + e] = hk[static_cast<size_t>(J.n_off + e)];
        if (perm)
          for (i64 e = 0; e < w; ++e) perm[s_off[b] + e] = hp[static_cast<size_t>(J.n_off + e)];
      }
    }
  }
  cudaStreamDestroy(st);
  CAPI_END
}

}  // extern "C"
