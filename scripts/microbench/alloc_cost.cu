// Cost of making N GB of device memory usable: cudaMalloc vs cudaMallocAsync
// (default pool, and a private pool that keeps freed memory), each followed
// by a memset, timed on the host around allocation + memset + sync.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

static double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

int main() {
  cudaFree(0);
  cudaStream_t s;
  cudaStreamCreate(&s);
  const size_t GB = 1ull << 30;
  for (size_t g : {1, 4, 16}) {
    const size_t n = g * GB;
    void* p = nullptr;
    auto t0 = std::chrono::steady_clock::now();
    cudaMalloc(&p, n);
    double a = ms_since(t0);
    cudaMemsetAsync(p, 0, n, s);
    cudaStreamSynchronize(s);
    double b = ms_since(t0);
    cudaFree(p);
    t0 = std::chrono::steady_clock::now();
    cudaMallocAsync(&p, n, s);
    double c = ms_since(t0);
    cudaMemsetAsync(p, 0, n, s);
    cudaStreamSynchronize(s);
    double d = ms_since(t0);
    cudaFreeAsync(p, s);
    cudaStreamSynchronize(s);
    // again (default pool: released at the sync above unless a threshold is set)
    t0 = std::chrono::steady_clock::now();
    cudaMallocAsync(&p, n, s);
    cudaMemsetAsync(p, 0, n, s);
    cudaStreamSynchronize(s);
    double e = ms_since(t0);
    cudaFreeAsync(p, s);
    cudaStreamSynchronize(s);
    std::printf("%zu GB: cudaMalloc %.1f ms (+memset %.1f) | cudaMallocAsync %.1f ms (+memset %.1f) | again %.1f\n", g,
                a, b, c, d, e);
  }
  return 0;
}
