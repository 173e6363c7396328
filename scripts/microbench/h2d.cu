// Host<->device transfer cost on this box: pinned cudaMemcpyAsync + stream
// sync for the byte counts of one evaluation step, and an empty-kernel
// launch + sync, to size the fixed part of the e2e step.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o h2d h2d.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_kernel() {}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  void *h, *d;
  cudaMallocHost(&h, 8 << 20);
  cudaMalloc(&d, 8 << 20);
  auto bench = [&](const char* what, auto fn) {
    for (int i = 0; i < 20; ++i) fn();
    cudaStreamSynchronize(s);
    const int n = 200;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) {
      fn();
      cudaStreamSynchronize(s);
    }
    auto t1 = std::chrono::steady_clock::now();
    printf("%-44s %8.2f us\n", what, std::chrono::duration<double, std::micro>(t1 - t0).count() / n);
  };
  bench("empty stream sync", [&] {});
  bench("empty kernel launch + sync", [&] { empty_kernel<<<1, 32, 0, s>>>(); });
  for (size_t b : {4096ul, 65536ul, 262144ul, 327100ul, 1048576ul, 4194304ul}) {
    char l1[64], l2[64];
    snprintf(l1, 64, "H2D %8zu B + sync", b);
    snprintf(l2, 64, "D2H %8zu B + sync", b);
    bench(l1, [&] { cudaMemcpyAsync(d, h, b, cudaMemcpyHostToDevice, s); });
    bench(l2, [&] { cudaMemcpyAsync(h, d, b, cudaMemcpyDeviceToHost, s); });
  }
  bench("H2D 262144 + 65536 B (2 copies) + sync", [&] {
    cudaMemcpyAsync(d, h, 262144, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync((char*)d + 262144, (char*)h + 262144, 65536, cudaMemcpyHostToDevice, s);
  });
  bench("H2D 327100 B + empty kernel + sync", [&] {
    cudaMemcpyAsync(d, h, 327100, cudaMemcpyHostToDevice, s);
    empty_kernel<<<1, 32, 0, s>>>();
  });
  return 0;
}
