// DFMA latency / throughput and an LDS+DFMA complex-MAC loop (diagnostic).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_lat(double* out, int n) {
  double a = threadIdx.x, b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = a + (double)(t1 - t0) / n;  // cycles per dependent DFMA
}
__global__ void k_tput(double* out, int n) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 1.0000001, c = 1e-9;
  for (int i = 0; i < n; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_cmac(double* out, int n, int ein) {
  extern __shared__ double2 sm[];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = make_double2(i * 1e-3, 1.0 - i * 1e-3);
  __syncthreads();
  long long t0 = clock64();
  double2 acc = make_double2(0, 0), acc1 = make_double2(0, 0);
  for (int r = 0; r < n; ++r) {
    const double2* xs = sm + (threadIdx.x + r) % 64;
    const double2* M = sm + 2048 + (r % 7);
    for (int x = 0; x + 1 < ein; x += 2) {
      double2 u = xs[7 * x], v = M[7 * x], u1 = xs[7 * x + 7], v1 = M[7 * x + 7];
      acc.x = fma(u.x, v.x, fma(-u.y, v.y, acc.x)); acc.y = fma(u.x, v.y, fma(u.y, v.x, acc.y));
      acc1.x = fma(u1.x, v1.x, fma(-u1.y, v1.y, acc1.x)); acc1.y = fma(u1.x, v1.y, fma(u1.y, v1.x, acc1.y));
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc1.x + acc1.y;
  if (threadIdx.x == 0) out[1 << 20] = (double)(t1 - t0) / (n * ein);  // cycles per complex MAC per thread
}
int main() {
  double* out; cudaMalloc(&out, 16 << 20);
  double h;
  k_lat<<<1, 32>>>(out, 100000); cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency ~ %.2f cycles (minus tiny)\n", h);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int blocks : {148, 148 * 4}) {
    k_tput<<<blocks, 256>>>(out, 1000);
    cudaEventRecord(a); int n = 20000; k_tput<<<blocks, 256>>>(out, n); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 8 * n * (double)blocks * 256;
    printf("DFMA throughput blocks=%d: %.2f TFLOP/s\n", blocks, flops / ms / 1e9);
  }
  for (int warps : {1, 8, 32}) {
    k_cmac<<<1, 32 * warps, 65536>>>(out, 200, 16); cudaDeviceSynchronize();
    cudaMemcpy(&h, out + (1 << 20), 8, cudaMemcpyDeviceToHost);
    printf("LDS+cMAC loop (ein=16), %2d warps/SM: %.1f cycles per complex MAC per thread\n", warps, h);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
