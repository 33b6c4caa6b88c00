// Persistent dataflow apply kernel (Alg. 2 as one launch).
//
// The whole contraction -- V/W boxes, core GEMV row chunks, P/U boxes -- is a
// list of CTA-sized work items in a host-computed ticket order (a topological
// order of the item DAG, sorted by a simulated start time, runflow in
// runtime.cu).  One CTA per resident slot loops:
//   ticket = atomicAdd(next)            (the next ticket is claimed while the
//                                        current item runs)
//   prologue of the item                (factor rows: independent of inputs)
//   wait for the item's producers       (per-item completion flags, acquire)
//   run it                              (box_device.cuh / the GEMV rows below)
//   publish done[item] = mark           (CTA barrier, fence, release store)
// Items only wait on items with smaller tickets, and every claimed ticket
// belongs to a running CTA, so the smallest unfinished item can always run:
// no deadlock whatever the residency.  Producer -> consumer overlap across
// levels replaces the kernel boundaries of the per-level engine: the P/U boxes
// of a row multi-set t start as soon as its core rows are done, while the
// GEMV still streams the cores of later t.
//
// Host-buffer contraction: F arrives in slabs by DMA on a copy stream that
// raises a per-slab flag (a 4-byte copy after each slab); items reading F wait
// on those flags, so compute starts on the first slab.  G may be mapped pinned
// host memory: the U level writes the result straight over PCIe.
//
// Completion flags hold an epoch mark (ctl[2] + 1); the last CTA to finish
// advances the epoch and resets the ticket counter and the input flags, so a
// replay needs no memset.  A spinning wait traps after ~4 s instead of hanging.
#include "box_device.cuh"

namespace tbf {

namespace {

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ double2 ld_stream2(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Poll with relaxed loads (an acquire per poll would cost the SM's other CTAs
// their L1 / load pipe), then one acquire load once the value is seen.
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __noinline__ void spin_done(const int* p, int mark) {
  unsigned long long n = 0;
  while (ld_relaxed_gpu(p) != mark) {
    __nanosleep(256);
    if (++n > (1ull << 24)) __trap();  // ~4 s: a broken dependency, not a slow producer
  }
  (void)ld_acquire_gpu(p);
}
__device__ __noinline__ void spin_flag(const int* p) {
  unsigned long long n = 0;
  while (*reinterpret_cast<const volatile int*>(p) == 0) {
    __nanosleep(256);
    if (++n > (1ull << 24)) __trap();
  }
  (void)ld_acquire_sys(p);
}

// One GEMV item: rows [r0, r1) of one pair, y = K x for all nv vectors.
// Same arithmetic and reduction order as k_gemv (apply_kernels.cu): the flow
// and per-level engines agree bit for bit.
template <bool NV1, class Wait>
__device__ __forceinline__ void gemv_item(const GemvDesc& D, int r0, int r1, int nv_rt,
                                          const double2* __restrict__ cores, const double2* x, double2* y,
                                          double2* sx, Wait wait) {
  constexpr int kAcc = NV1 ? 1 : 4;
  const int nv = NV1 ? 1 : nv_rt;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = D.C;
  constexpr int kWarps = kBoxThreads / 32;
  // this warp's first row into L2 before the wait (cores are constant)
  if (r0 + warp < r1) {
    const char* rp = reinterpret_cast<const char*>(cores + D.core_off + static_cast<long long>(r0 + warp) * C);
    for (int o = lane * 128; o < C * 16; o += 32 * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + o));
  }
  wait();
  for (int v0 = 0; v0 < nv; v0 += kAcc) {
    const int nvc = min(kAcc, nv - v0);
    const double2* xs = x + D.x_off + static_cast<long long>(v0) * C;
    for (int i = threadIdx.x; i < C * nvc; i += kBoxThreads * 4) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i + u * kBoxThreads < C * nvc) v[u] = ld_in<true>(xs + i + u * kBoxThreads);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i + u * kBoxThreads < C * nvc) sx[i + u * kBoxThreads] = v[u];
    }
    __syncthreads();
    for (int r = r0 + warp; r < r1; r += kWarps) {
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
      if (c < C) {
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
  }
}

// wait for the producers of item t (all threads; ends with a CTA barrier)
__device__ __forceinline__ void wait_deps(const FlowArgs& a, const FlowItem& it, int t, int mark, bool fence) {
  for (int i = threadIdx.x; i < it.ndep; i += kBoxThreads) {
    const int dep = a.deps[it.dep_begin + i];
    if (dep >= 0) spin_done(a.done + dep, mark);
    else spin_flag(a.in_flags + (-1 - dep));
  }
  __syncthreads();
  if (fence) asm volatile("fence.proxy.async.global;" ::: "memory");
  if (a.trace && threadIdx.x == 0) a.trace[8 * t + 1] = gtimer();
}

// The two item bodies are separate (non-inlined) functions so each gets the
// register allocation of its own code, not of the persistent loop around it.
__device__ __forceinline__ void flow_box(const FlowArgs& a, BoxSmem& S, const FlowOp& op, const FlowItem& it, int t,
                                      int mark, double2* sm, unsigned& phase) {
  const double2* in = op.in_buf == 0 ? a.F : a.scratch;
  double2* out = op.out_buf == 1 ? a.G : a.scratch;
  // bulk (async-proxy) staging of data produced inside this launch (by
  // generic stores of other CTAs, or by the copy engine for F) needs a proxy
  // fence after the acquire; nothing else does
  const bool fence = it.ndep > 0 && op.info.stage;
  box_body<true>(S, op.info, it.crank, op.mats, in, out, sm, phase, [&] { wait_deps(a, it, t, mark, fence); },
                 [&](int k) {
                   if (a.trace && threadIdx.x == 0 && k >= 3) a.trace[8 * t + 1 + k] = gtimer();
                 });
}

template <bool NV1>
__device__ __forceinline__ void flow_gemv(const FlowArgs& a, const FlowOp& op, const FlowItem& it, int t, int mark,
                                       double2* sm) {
  gemv_item<NV1>(op.gdescs[it.desc], it.r0, it.r1, a.nv, a.cores, a.scratch, a.scratch, sm,
                 [&] { wait_deps(a, it, t, mark, false); });
}

template <bool NV1>
__global__ void __launch_bounds__(kBoxThreads, 2) k_flow(FlowArgs a) {
  extern __shared__ __align__(128) double2 sm[];
  __shared__ BoxSmem S;
  __shared__ FlowItem s_it;
  __shared__ FlowOp s_op;
  __shared__ int s_next;
  __shared__ int s_mark;
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&S.bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_mark = static_cast<int>(*reinterpret_cast<volatile unsigned*>(a.ctl + 2)) + 1;
    s_next = static_cast<int>(atomicAdd(a.ctl, 1u));
  }
  unsigned phase = 0;
  for (;;) {
    __syncthreads();  // s_next visible; the previous item fully done
    const int t = s_next;
    if (t >= a.nitems) break;
    copy_desc(&s_it, a.items + t);
    __syncthreads();  // every thread has read s_next; s_it in place
    if (tid == 0) {
      s_next = static_cast<int>(atomicAdd(a.ctl, 1u));  // claimed while this item runs
      if (a.trace) a.trace[8 * t] = gtimer();
    }
    copy_desc(&s_op, a.ops + s_it.op);
    if (s_it.kind == 0) copy_desc(&S.D, a.ops[s_it.op].descs + s_it.desc);
    __syncthreads();
    if (s_it.kind == 0) flow_box(a, S, s_op, s_it, t, s_mark, sm, phase);
    else flow_gemv<NV1>(a, s_op, s_it, t, s_mark, sm);
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release_gpu(a.done + t, s_mark);
      if (a.trace) {
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        a.trace[8 * t + 2] = gtimer();
        a.trace[8 * t + 3] = smid;
      }
    }
  }
  if (tid == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(a.ctl + 1, 1u);
    if (prev == gridDim.x - 1) {  // last CTA out: reset for the next launch
      for (int q = 0; q < a.nflags; ++q) a.in_flags[q] = 0;
      a.ctl[0] = 0;
      a.ctl[1] = 0;
      __threadfence();
      a.ctl[2] = static_cast<unsigned>(s_mark);
    }
  }
}

}  // namespace

int flow_ctas_per_sm(int nv, size_t smem) {
  int n = 0;
  if (nv == 1) {
    TBF_CUDA(cudaFuncSetAttribute(k_flow<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    TBF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_flow<true>, kBoxThreads, smem));
  } else {
    TBF_CUDA(cudaFuncSetAttribute(k_flow<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    TBF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_flow<false>, kBoxThreads, smem));
  }
  return n;
}

int flow_threads() { return kBoxThreads; }

void launch_flow(const FlowArgs& a, int grid, size_t smem, cudaStream_t st) {
  if (a.nitems == 0 || grid <= 0) return;
  if (a.nv == 1) {
    TBF_CUDA(cudaFuncSetAttribute(k_flow<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    k_flow<true><<<grid, kBoxThreads, smem, st>>>(a);
  } else {
    TBF_CUDA(cudaFuncSetAttribute(k_flow<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    k_flow<false><<<grid, kBoxThreads, smem, st>>>(a);
  }
  TBF_CUDA(cudaGetLastError());
}

}  // namespace tbf
