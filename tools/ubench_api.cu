// Host-side cost of the CUDA runtime calls the native driver issues per
// launch (debug aid): empty kernel launch, cudaMallocAsync/cudaFreeAsync,
// cudaMemsetAsync, small D2D cudaMemcpyAsync, cudaEventRecord, and a D2H
// round trip (copy + stream sync).  nvcc -O2 -o tools/ubench_api tools/ubench_api.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(int *p) {
  if (p && threadIdx.x == 1234567) *p = 1;
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int *d = nullptr, *d2 = nullptr, *h = nullptr;
  cudaMalloc(&d, 1 << 20);
  cudaMalloc(&d2, 1 << 20);
  cudaMallocHost(&h, 4096);
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  const int N = 2000;
  auto bench = [&](const char *name, auto fn) {
    for (int i = 0; i < 50; ++i) fn();
    cudaStreamSynchronize(s);
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < N; ++i) fn();
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    auto t2 = std::chrono::steady_clock::now();
    printf("%-28s host %6.2f us/call   (incl. drain %6.2f us/call)\n", name,
           std::chrono::duration<double, std::micro>(t1 - t0).count() / N,
           std::chrono::duration<double, std::micro>(t2 - t0).count() / N);
  };
  bench("launch empty kernel", [&] { k_empty<<<1, 32, 0, s>>>(d); });
  bench("launch + cudaGetLastError", [&] {
    k_empty<<<1, 32, 0, s>>>(d);
    cudaGetLastError();
  });
  bench("cudaMallocAsync+FreeAsync", [&] {
    void *p;
    cudaMallocAsync(&p, 4096, s);
    cudaFreeAsync(p, s);
  });
  bench("cudaMemsetAsync 16 B", [&] { cudaMemsetAsync(d, 0, 16, s); });
  bench("cudaMemcpyAsync D2D 8 B", [&] { cudaMemcpyAsync(d2, d, 8, cudaMemcpyDeviceToDevice, s); });
  bench("cudaMemcpyAsync H2D 64 B", [&] { cudaMemcpyAsync(d2, h, 64, cudaMemcpyHostToDevice, s); });
  bench("cudaEventRecord", [&] { cudaEventRecord(ev, s); });
  bench("D2H 8 B + stream sync", [&] {
    cudaMemcpyAsync(h, d, 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
  });
  bench("kernel + D2H + sync", [&] {
    k_empty<<<1, 32, 0, s>>>(d);
    cudaMemcpyAsync(h, d, 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
  });
  return 0;
}
