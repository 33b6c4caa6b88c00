// Fixed-cost probes for small launches on B200 (diagnostic, not product).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_null(int* p) { if (threadIdx.x == 9999) p[0] = 1; }
__global__ void k_chain(const long long* __restrict__ idx, double* out, int n) {
  // n dependent global loads (pointer chase) by thread 0 of each CTA
  long long j = blockIdx.x;
  for (int i = 0; i < n; ++i) j = idx[j];
  if (threadIdx.x == 0) out[blockIdx.x] = (double)j;
}
__global__ void k_smem(double* out, int iters) {
  extern __shared__ double s[];
  double a = threadIdx.x;
  for (int i = 0; i < iters; ++i) { s[threadIdx.x] = a; __syncthreads(); a += s[(threadIdx.x + 1) % blockDim.x]; __syncthreads(); }
  if (threadIdx.x == 0) out[blockIdx.x] = a;
}
int main() {
  int* p; cudaMalloc(&p, 4096);
  long long* idx; cudaMalloc(&idx, 1 << 20);
  cudaMemset(idx, 0, 1 << 20);
  double* out; cudaMalloc(&out, 1 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaStream_t st; cudaStreamCreate(&st);
  auto timeit = [&](const char* name, auto fn) {
    for (int i = 0; i < 20; ++i) fn();
    cudaStreamSynchronize(st);
    cudaEventRecord(a, st);
    for (int i = 0; i < 200; ++i) fn();
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-40s %8.2f us/launch\n", name, ms * 1000 / 200);
  };
  for (int ctas : {1, 64, 148, 592}) {
    char nm[64];
    snprintf(nm, 64, "null ctas=%d", ctas);
    timeit(nm, [&] { k_null<<<ctas, 256, 0, st>>>(p); });
  }
  for (int n : {1, 4, 16}) {
    char nm[64];
    snprintf(nm, 64, "chain64 n=%d", n);
    timeit(nm, [&] { k_chain<<<64, 256, 0, st>>>(idx, out, n); });
  }
  timeit("smem sync x100 (64 ctas)", [&] { k_smem<<<64, 256, 2048, st>>>(out, 100); });
  // graph of 5 null kernels
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 5; ++i) k_null<<<64, 256, 0, st>>>(p);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  timeit("graph of 5 null (per graph)", [&] { cudaGraphLaunch(ge, st); });
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
