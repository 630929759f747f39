// FP64 dependent-chain latency on the GPU (DADD, DMUL, DFMA) and LDS latency.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  double x = a, y = b, z = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x + y; x = x + y; x = x + y; x = x + y; }
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) { z = z * b; z = z * b; z = z * b; z = z * b; }
  long long t2 = clock64();
  double w = a;
  for (int i = 0; i < n; ++i) { w = fma(w, b, y); w = fma(w, b, y); w = fma(w, b, y); w = fma(w, b, y); }
  long long t3 = clock64();
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x & 1023;
  long long t4 = clock64();
  for (int i = 0; i < 4 * n; ++i) p = s[p];
  long long t5 = clock64();
  out[threadIdx.x] = x + z + w + p;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t5 - t4; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 64);
  int n = 1000;
  k<<<1, 32>>>(o, c, 1.0, 1e-9, n); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 1.0, 1e-9, n); cudaDeviceSynchronize();
  printf("DADD %.2f  DMUL %.2f  DFMA %.2f  LDS %.2f cycles (dependent)\n", c[0] / (4.0 * n), c[1] / (4.0 * n), c[2] / (4.0 * n), c[3] / (4.0 * n));
  return 0;
}
