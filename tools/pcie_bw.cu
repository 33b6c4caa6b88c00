// PCIe ceiling probe (diagnostic, not product): 4 MB pinned H2D / D2H by DMA
// (one copy, split over 2 / 4 streams, 8 sequential slabs) and by zero-copy
// kernel loads / stores on mapped pinned memory.  Event timed after a 0.3 s
// link warm-up.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_zc_read(const double2* __restrict__ h, long long n, double2* d) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride) d[i] = h[i];
}
__global__ void k_zc_write(const double2* __restrict__ d, long long n, double2* h) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride) h[i] = d[i];
}

int main() {
  const size_t bytes = 4 << 20;
  const long long n = bytes / 16;
  char *h, *h2, *d, *d2;
  cudaHostAlloc(reinterpret_cast<void**>(&h), bytes, cudaHostAllocDefault);
  cudaHostAlloc(reinterpret_cast<void**>(&h2), bytes, cudaHostAllocDefault);
  cudaMalloc(&d, bytes);
  cudaMalloc(&d2, bytes);
  cudaStream_t s[8];
  for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, ev[8];
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (auto& x : ev) cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
  auto t0 = std::chrono::steady_clock::now();
  while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < 0.3) {
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s[0]);
    cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, s[0]);
    cudaStreamSynchronize(s[0]);
  }
  auto run = [&](const char* name, auto fn) {
    float best = 1e30f, sum = 0;
    const int reps = 50;
    for (int r = 0; r < reps; ++r) {
      cudaEventRecord(e0, s[0]);
      fn();
      cudaEventRecord(e1, s[0]);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
      sum += ms;
    }
    printf("%-34s best %7.1f us (%5.1f GB/s)  mean %7.1f us\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9,
           sum / reps * 1e3);
  };
  for (int dir = 0; dir < 2; ++dir) {
    const cudaMemcpyKind k = dir == 0 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
    char* dst = dir == 0 ? d : h2;
    const char* src = dir == 0 ? h : d2;
    const char* tag = dir == 0 ? "H2D" : "D2H";
    char name[64];
    snprintf(name, sizeof name, "%s one copy", tag);
    run(name, [&] { cudaMemcpyAsync(dst, src, bytes, k, s[0]); });
    for (int ns : {2, 4}) {
      snprintf(name, sizeof name, "%s split over %d streams", tag, ns);
      run(name, [&] {
        cudaEventRecord(ev[0], s[0]);
        const size_t part = bytes / ns;
        for (int i = 0; i < ns; ++i) {
          cudaStreamWaitEvent(s[i], ev[0], 0);
          cudaMemcpyAsync(dst + i * part, src + i * part, part, k, s[i]);
          cudaEventRecord(ev[i + 1 < 8 ? i + 1 : 7], s[i]);
        }
        for (int i = 1; i < ns; ++i) cudaStreamWaitEvent(s[0], ev[i + 1], 0);
      });
    }
    snprintf(name, sizeof name, "%s 8 sequential slabs", tag);
    run(name, [&] {
      for (int i = 0; i < 8; ++i) cudaMemcpyAsync(dst + i * (bytes / 8), src + i * (bytes / 8), bytes / 8, k, s[0]);
    });
  }
  run("H2D || D2H concurrently (4 MB each)", [&] {
    cudaEventRecord(ev[0], s[0]);
    cudaStreamWaitEvent(s[1], ev[0], 0);
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s[0]);
    cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, s[1]);
    cudaEventRecord(ev[1], s[1]);
    cudaStreamWaitEvent(s[0], ev[1], 0);
  });
  for (int grid : {148, 296, 592}) {
    char name[64];
    snprintf(name, sizeof name, "zero-copy kernel read, %d CTAs", grid);
    run(name, [&] { k_zc_read<<<grid, 256, 0, s[0]>>>(reinterpret_cast<double2*>(h), n, reinterpret_cast<double2*>(d)); });
    snprintf(name, sizeof name, "zero-copy kernel write, %d CTAs", grid);
    run(name, [&] { k_zc_write<<<grid, 256, 0, s[0]>>>(reinterpret_cast<double2*>(d2), n, reinterpret_cast<double2*>(h2)); });
  }
  return 0;
}
