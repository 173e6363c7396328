// Host-side costs of caching a 1.6-GB matrix (100k x 2000 doubles): zero-init
// vector, parallel first-touch copy (4 KB pages vs transparent huge pages),
// pageable H2D, pinned allocation / registration, pinned H2D.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <sys/mman.h>
#include <thread>
#include <vector>
#include <cuda_runtime.h>

static double ms(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}
static void par_copy(char* d, const char* s, size_t n, int T) {
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t)
    th.emplace_back([=] {
      const size_t lo = n * t / T, hi = n * (t + 1) / T;
      std::memcpy(d + lo, s + lo, hi - lo);
    });
  for (auto& x : th) x.join();
}
int main() {
  cudaFree(0);
  const size_t n = 100000ull * 2000 * 8;
  const int T = (int)std::thread::hardware_concurrency();
  std::vector<double> src(n / 8, 1.5);
  auto t0 = std::chrono::steady_clock::now();
  std::vector<double> z(n / 8);
  std::printf("vector<double> zero-init %.1f ms\n", ms(t0));
  t0 = std::chrono::steady_clock::now();
  par_copy((char*)z.data(), (const char*)src.data(), n, T);
  std::printf("parallel copy into it (touched) %.1f ms (%d threads)\n", ms(t0), T);
  t0 = std::chrono::steady_clock::now();
  char* a = (char*)mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  par_copy(a, (const char*)src.data(), n, T);
  std::printf("mmap 4K + parallel first-touch copy %.1f ms\n", ms(t0));
  t0 = std::chrono::steady_clock::now();
  char* b = (char*)mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  madvise(b, n, MADV_HUGEPAGE);
  par_copy(b, (const char*)src.data(), n, T);
  std::printf("mmap THP + parallel first-touch copy %.1f ms\n", ms(t0));
  void* d;
  cudaMalloc(&d, n);
  t0 = std::chrono::steady_clock::now();
  cudaMemcpy(d, src.data(), n, cudaMemcpyHostToDevice);
  std::printf("pageable H2D %.1f ms\n", ms(t0));
  void* h;
  t0 = std::chrono::steady_clock::now();
  cudaHostAlloc(&h, n, cudaHostAllocDefault);
  std::printf("cudaHostAlloc %.1f ms\n", ms(t0));
  t0 = std::chrono::steady_clock::now();
  par_copy((char*)h, (const char*)src.data(), n, T);
  std::printf("parallel copy into pinned %.1f ms\n", ms(t0));
  t0 = std::chrono::steady_clock::now();
  cudaMemcpy(d, h, n, cudaMemcpyHostToDevice);
  std::printf("pinned H2D %.1f ms\n", ms(t0));
  t0 = std::chrono::steady_clock::now();
  cudaHostRegister(b, n, cudaHostRegisterDefault);
  std::printf("cudaHostRegister (THP buffer) %.1f ms\n", ms(t0));
  t0 = std::chrono::steady_clock::now();
  cudaMemcpy(d, b, n, cudaMemcpyHostToDevice);
  std::printf("registered H2D %.1f ms\n", ms(t0));
  return 0;
}
