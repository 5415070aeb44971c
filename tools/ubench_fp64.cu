// Micro-benchmark: fp64 FMA latency / throughput, shared-memory load
// latency, sqrt / div latency and __syncthreads cost on one SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ub tools/ubench_fp64.cu && /tmp/ub
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double *out, long long *cyc, double x0, int iters) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
  __syncthreads();
  double a = x0 + threadIdx.x, b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, c);  // dependent DFMA chain
  long long t1 = clock64();
  int idx = threadIdx.x & 1023;
  double s = 0.0;
  for (int i = 0; i < iters; ++i) {  // dependent shared loads (pointer chase-ish)
    s += sm[idx];
    idx = (idx + (int)(s > 1e300)) & 1023;
  }
  long long t2 = clock64();
  double r = a;
  for (int i = 0; i < iters / 8; ++i) r = sqrt(r + 1.0);
  long long t3 = clock64();
  double q = a;
  for (int i = 0; i < iters / 8; ++i) q = 1.0 / (q + 1.0);
  long long t4 = clock64();
  for (int i = 0; i < iters / 8; ++i) __syncthreads();
  long long t5 = clock64();
  double u = a;
  for (int i = 0; i < iters / 8; ++i) u += __shfl_xor_sync(0xffffffffu, u, 1);
  long long t6 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = t4 - t3;
    cyc[4] = t5 - t4;
    cyc[5] = t6 - t5;
  }
  out[threadIdx.x] = a + s + r + q + u;
}

__global__ void k_tput(double *out, long long *cyc, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
         a6 = a0 + 6, a7 = a0 + 7;
  const double b = 1.0000001, c = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

int main() {
  double *out;
  long long *cyc, h[8];
  cudaMalloc(&out, 8 * 2048);
  cudaMalloc(&cyc, 64);
  const int iters = 4096;
  k_lat<<<1, 32>>>(out, cyc, 1.0, iters);
  k_lat<<<1, 32>>>(out, cyc, 1.0, iters);
  cudaMemcpy(h, cyc, 48, cudaMemcpyDeviceToHost);
  printf("1 warp: DFMA dep latency %.1f cyc, LDS dep latency %.1f cyc, sqrt %.1f, div %.1f, "
         "bar.sync %.1f, shfl+dadd %.1f cyc\n",
         (double)h[0] / iters, (double)h[1] / iters, (double)h[2] / (iters / 8),
         (double)h[3] / (iters / 8), (double)h[4] / (iters / 8), (double)h[5] / (iters / 8));
  for (int nt : {256, 512, 1024}) {
    k_lat<<<1, nt>>>(out, cyc, 1.0, iters);
    cudaMemcpy(h, cyc, 48, cudaMemcpyDeviceToHost);
    printf("%4d thr: bar.sync %.1f cyc\n", nt, (double)h[4] / (iters / 8));
  }
  for (int nt : {32, 128, 256, 512, 1024}) {
    k_tput<<<1, nt>>>(out, cyc, iters);
    k_tput<<<1, nt>>>(out, cyc, iters);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    double fmas = 8.0 * iters * nt;
    printf("%4d thr: DFMA throughput %.2f FMA/clk/SM\n", nt, fmas / h[0]);
  }
  return 0;
}
