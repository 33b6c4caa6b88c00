// Read-stream ceiling on this B200 (diagnostic, not product): a flat
// 16-B-per-lane streaming read of N bytes, reduced to one value per thread,
// for several CTAs-per-SM and loads-in-flight settings; CUDA-event timed,
// L2 flushed before each run.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double2 ldnc(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

template <int U>
__global__ void k_read(const double2* __restrict__ a, long long n, double* out) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  double s = 0;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldnc(a + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u].x + v[u].y;
  }
  for (; i < n; i += stride) s += a[i].x;
  if (s == 12345.678) out[0] = s;
}

// contiguous chunk per CTA (like the GEMV's row ranges)
template <int U>
__global__ void k_read_chunk(const double2* __restrict__ a, long long n, double* out) {
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long b = per * blockIdx.x, e = min(n, b + per);
  double s = 0;
  long long i = b + threadIdx.x;
  for (; i + (U - 1) * blockDim.x < e; i += U * blockDim.x) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldnc(a + i + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u].x + v[u].y;
  }
  for (; i < e; i += blockDim.x) s += a[i].x;
  if (s == 12345.678) out[0] = s;
}

int main() {
  const long long sizes[2] = {232LL << 20, 2048LL << 20};
  double2* a;
  char* flush;
  double* out;
  cudaMalloc(&a, sizes[1]);
  cudaMalloc(&flush, 512 << 20);
  cudaMalloc(&out, 8);
  cudaMemset(a, 0, sizes[1]);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (long long bytes : sizes) {
    const long long n = bytes / 16;
    for (int chunk = 0; chunk < 2; ++chunk)
      for (int per_sm : {2, 4, 8})
        for (int u : {4, 8, 16}) {
          float best = 1e30f;
          for (int rep = 0; rep < 5; ++rep) {
            cudaMemsetAsync(flush, rep, 512 << 20);
            cudaEventRecord(e0);
            const int grid = 148 * per_sm;
            if (chunk == 0) {
              if (u == 4) k_read<4><<<grid, 256>>>(a, n, out);
              if (u == 8) k_read<8><<<grid, 256>>>(a, n, out);
              if (u == 16) k_read<16><<<grid, 256>>>(a, n, out);
            } else {
              if (u == 4) k_read_chunk<4><<<grid, 256>>>(a, n, out);
              if (u == 8) k_read_chunk<8><<<grid, 256>>>(a, n, out);
              if (u == 16) k_read_chunk<16><<<grid, 256>>>(a, n, out);
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
          }
          printf("%5lld MB %s ctas/SM %d loads/lane %2d: %7.1f us  %6.0f GB/s\n", bytes >> 20,
                 chunk ? "chunked" : "strided", per_sm, u, best * 1e3, bytes / (best * 1e-3) / 1e9);
        }
  }
  return 0;
}
