// FP64 roofline denominators measured on the device the library runs on
// (MEASURED_PEAKS.json has HBM and bf16 only): DFMA throughput of the CUDA
// cores and DMMA (mma.sync.m8n8k4.f64, the FP64 tensor-core path on sm_100a;
// tcgen05 has no f64 kind) throughput, both with independent accumulator
// chains on every resident warp.  Diagnostic entry point for bench.py.
#include <vector>

#include "kernels.h"

namespace tbf {
namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters, double b, double c) {
  double a[kChains];
#pragma unroll
  for (int q = 0; q < kChains; ++q) a[q] = threadIdx.x * 1e-3 + q;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < kChains; ++q) a[q] = fma(a[q], b, c);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < kChains; ++q) s += a[q];
  if (s == 1234.5678) out[blockIdx.x] = s;  // keeps the chains live
}

__global__ void __launch_bounds__(256) k_dmma_peak(double* out, int iters) {
  const int lane = threadIdx.x & 31;
  const double av = 1.0 + lane * 1e-6, bv = 1.0 - lane * 1e-6;
  double d[4][2];
#pragma unroll
  for (int q = 0; q < 4; ++q) d[q][0] = d[q][1] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[q][0]), "+d"(d[q][1])
                   : "d"(av), "d"(bv));
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) s += d[q][0] + d[q][1];
  if (s == 1234.5678) out[blockIdx.x] = s;
}

}  // namespace

// out[0] = DFMA TFLOP/s, out[1] = DMMA TFLOP/s, out[2] = SM count, out[3] = SM clock (MHz) at launch
void measure_fp64_peak(double* out) {
  int dev = 0, sms = 0, clk = 0;
  TBF_CUDA(cudaGetDevice(&dev));
  TBF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  TBF_CUDA(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* d = nullptr;
  TBF_CUDA(cudaMalloc(&d, sizeof(double) * 65536));
  cudaEvent_t e0, e1;
  TBF_CUDA(cudaEventCreate(&e0));
  TBF_CUDA(cudaEventCreate(&e1));
  const int blocks = sms * 8, threads = 256;
  auto timed = [&](auto&& launch) {
    launch();  // warm
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      TBF_CUDA(cudaEventRecord(e0));
      launch();
      TBF_CUDA(cudaEventRecord(e1));
      TBF_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      TBF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
    }
    return static_cast<double>(best);
  };
  const int it1 = 4096;
  const double ms1 = timed([&] { k_dfma_peak<<<blocks, threads>>>(d, it1, 0.999999, 1e-9); });
  const double fl1 = 2.0 * kChains * static_cast<double>(it1) * blocks * threads;
  const int it2 = 2048;
  const double ms2 = timed([&] { k_dmma_peak<<<blocks, threads>>>(d, it2); });
  const double fl2 = 2.0 * 256.0 * 4 * static_cast<double>(it2) * blocks * (threads / 32);
  TBF_CUDA(cudaGetLastError());
  out[0] = fl1 / (ms1 * 1e-3) / 1e12;
  out[1] = fl2 / (ms2 * 1e-3) / 1e12;
  out[2] = sms;
  out[3] = clk / 1e3;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
}

}  // namespace tbf
