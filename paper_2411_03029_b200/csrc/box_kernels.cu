// Fused level contractions for the apply, one launch per (side, level [, slab
// group]); the per-box device code (staging, the d mode phases, the layout
// choices) is in box_device.cuh.  This file adds the per-level launch: grid =
// boxes x cs, programmatic dependent launch (the factor prologue runs before
// griddepcontrol.wait).
#include "box_device.cuh"

namespace tbf {

namespace {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// MINB: CTAs per SM the register budget targets -- 3 for boxes whose shared
// memory lets three CTAs co-reside (latency-bound small boxes: config 3's
// levels 1.65 -> 1.56 ms), 2 otherwise (the 80-register cap spills on large
// boxes: config 5 was 4% slower with it)
template <int NT, int MINB, int PATH = 0>
__global__ void __launch_bounds__(NT, MINB) k_box(const BoxDesc* __restrict__ descs, BoxLaunchInfo info,
                                                        const double2* __restrict__ mats,
                                                        const double2* __restrict__ in, double2* __restrict__ out) {
  extern __shared__ __align__(128) double2 sm[];
  __shared__ BoxSmem S;
  pdl_trigger();
  const int cs = info.cs;
  const int item = static_cast<int>(blockIdx.x) / cs;
  const int crank = static_cast<int>(blockIdx.x) - item * cs;
  copy_desc(&S.D, descs + item);
  if (threadIdx.x == 0) {
    mbar_init(&S.bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned phase = 0;
  box_body<MINB >= 3 ? 4 : 8, 2, PATH>(S, info, crank, mats, in, out, sm, phase, [] { pdl_wait(); });
}


}  // namespace

bool pdl_enabled() {
  static const bool on = std::getenv("OIOBF_NO_PDL") == nullptr;
  return on;
}

constexpr size_t kBox3Smem = 72 * 1024;  // three CTAs per SM fit in shared memory

using BoxKernel = void (*)(const BoxDesc*, BoxLaunchInfo, const double2*, const double2*, double2*);
// 128-thread CTAs whose shared memory lets five or six co-reside take the
// 80-register instance (OIOBF_BOX6_KB overrides the threshold for A/B runs)
size_t box6_smem() {  // (read once: launch_box runs per launch outside graphs)
  static const size_t kb = std::getenv("OIOBF_BOX6_KB") ? static_cast<size_t>(std::atoi(std::getenv("OIOBF_BOX6_KB"))) : 47;
  return kb * 1024;
}

// kernel instance for a launch: 128 threads at 6 CTAs / SM (80 registers) for
// small boxes, 256 threads at 3 (80 registers) or 2 (128: large boxes, and
// streamed inputs whose 8 loads in flight would spill at 80) CTAs / SM
// 128-thread instance for `path` whose register budget matches the CTAs per SM
// that shared memory allows anyway (6: 80 registers ... 3: 170): a launch held
// to 4-5 CTAs by its shared memory gets 128 / 102 registers instead of spilling
// at 80.  OIOBF_BOX_MINB=0 restores the two-instance rule (80 registers up to
// OIOBF_BOX6_KB of shared memory).
template <int PATH>
BoxKernel box_kernel128(size_t smem) {
  static const bool fixed = std::getenv("OIOBF_BOX_MINB") && std::getenv("OIOBF_BOX_MINB")[0] == '0';
  if (fixed) return smem <= box6_smem() ? k_box<128, 6, PATH> : k_box<128, 3, PATH>;
  const size_t per_cta = smem + sizeof(BoxSmem) + 1024;  // static shared memory and the per-CTA reserve
  const size_t n = (227 * 1024) / per_cta;
  if (n >= 6) return k_box<128, 6, PATH>;
  if (n == 5) return k_box<128, 5, PATH>;
  if (n == 4) return k_box<128, 4, PATH>;
  return k_box<128, 3, PATH>;
}

BoxKernel box_kernel(int nt, int stage, size_t smem, int path) {
  if (nt == 128) return path == 1 ? box_kernel128<1>(smem) : path == 2 ? box_kernel128<2>(smem) : box_kernel128<0>(smem);
  return smem <= kBox3Smem && stage ? k_box<256, 3> : k_box<256, 2>;
}

int box_ctas_per_sm(int nt, int stage, size_t smem) {
  int n = 0;
  const BoxKernel k = box_kernel(nt, stage, smem, 0);
  TBF_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
  TBF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, nt, smem));
  return n;
}

size_t box_smem_bytes(const BoxLaunchInfo& info) {
  return sizeof(double2) * (static_cast<size_t>(info.smem_mat) + static_cast<size_t>(info.smem_in) +
                            static_cast<size_t>(info.smem_t) + static_cast<size_t>(info.smem_t1));
}



void launch_box(i64 nitems, const BoxDesc* descs, const BoxLaunchInfo& info, const double2* mats,
                const double2* in, double2* out, cudaStream_t st) {
  if (nitems == 0) return;
  if (info.d < 2 || info.d > kMaxD) throw std::runtime_error("launch_box: d out of range");
  if (info.amax > 8) throw std::runtime_error("launch_box: more than 8 rows of mode d-1 per CTA");
  const size_t smem = box_smem_bytes(info);
  const int nt = info.nt > 0 ? info.nt : kBoxThreads;
  const BoxKernel kern = box_kernel(nt, info.stage, smem, info.path);
  TBF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(nitems * info.cs));
  cfg.blockDim = dim3(static_cast<unsigned>(nt));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  TBF_CUDA(cudaLaunchKernelEx(&cfg, kern, descs, info, mats, in, out));
  TBF_CUDA(cudaGetLastError());
}

}  // namespace tbf
