// k_sum_parent-like access pattern in isolation (diagnostic).
#include <cstdio>
#include <cuda_runtime.h>
struct Desc { long long out_off, total, work_off; int nchild, pad; long long child_off[64]; };
__global__ void k_sum(const Desc* ds, const int* map, const double2* in, double2* out, int mode) {
  __shared__ Desc D;
  const int pidx = map[2 * blockIdx.x], chunk = map[2 * blockIdx.x + 1];
  if (mode == 0) { if (threadIdx.x == 0) D = ds[pidx]; }
  else { const long long* s = (const long long*)(ds + pidx); long long* d = (long long*)&D; for (int i = threadIdx.x; i < (int)(sizeof(Desc)/8); i += blockDim.x) d[i] = s[i]; }
  __syncthreads();
  for (int u = 0; u < 4; ++u) {
    long long q = (long long)chunk * 1024 + u * 256 + threadIdx.x;
    if (q >= D.total) break;
    double2 acc = make_double2(0, 0);
    double2 v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) if (c < D.nchild) v[c] = in[D.child_off[c] + q];
#pragma unroll
    for (int c = 0; c < 8; ++c) if (c < D.nchild) { acc.x += v[c].x; acc.y += v[c].y; }
    out[D.out_off + q] = acc;
  }
}
int main() {
  const int P = 8, total = 2744, nchild = 8;
  Desc h[P]; int map[2 * 28]; int nc = 0;
  for (int p = 0; p < P; ++p) {
    h[p].out_off = 4000000 + p * 3000; h[p].total = total; h[p].nchild = nchild;
    for (int c = 0; c < nchild; ++c) h[p].child_off[c] = (long long)(p * nchild + c) * 3000;
    for (int ch = 0; ch * 1024 < total; ++ch) { map[2 * nc] = p; map[2 * nc + 1] = ch; ++nc; }
  }
  Desc* d; int* dm; double2 *in, *out;
  cudaMalloc(&d, sizeof(h)); cudaMalloc(&dm, sizeof(map)); cudaMalloc(&in, 8 << 20 << 4); out = in;
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice); cudaMemcpy(dm, map, sizeof(map), cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode) {
    for (int i = 0; i < 10; ++i) k_sum<<<nc, 256>>>(d, dm, in, out, mode);
    cudaEventRecord(a);
    for (int i = 0; i < 100; ++i) k_sum<<<nc, 256>>>(d, dm, in, out, mode);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("mode %d (%s): %d ctas, %.2f us/launch\n", mode, mode ? "coop desc copy" : "thread0 desc copy", nc, ms * 10);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
