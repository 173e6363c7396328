// upload_paths.cu -- microbenchmark of host->device paths for the one-time
// matrix upload (ebic_matrix_upload_*): pageable cudaMemcpy, cudaHostRegister
// of the caller's buffer, and chunked staging through a small page-locked
// ring filled by host threads while the DMA runs.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  const size_t bytes = (argc > 1 ? atol(argv[1]) : 80) << 20;
  std::vector<char> host(bytes);
  for (size_t i = 0; i < bytes; i += 4096) host[i] = (char)i;
  std::memset(host.data(), 1, bytes);
  void* d = nullptr;
  cudaFree(0);
  double t0 = now_ms();
  cudaMalloc(&d, bytes);
  printf("cudaMalloc %zu MB: %.2f ms\n", bytes >> 20, now_ms() - t0);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int rep = 0; rep < 3; ++rep) {
    t0 = now_ms();
    cudaMemcpyAsync(d, host.data(), bytes, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    double pageable = now_ms() - t0;
    t0 = now_ms();
    cudaHostRegister(host.data(), bytes, cudaHostRegisterDefault);
    double reg = now_ms() - t0;
    t0 = now_ms();
    cudaMemcpyAsync(d, host.data(), bytes, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    double pinned = now_ms() - t0;
    t0 = now_ms();
    cudaHostUnregister(host.data());
    double unreg = now_ms() - t0;
    // staged ring: K slots of C bytes, T host threads fill slot k while the DMA of k-1 runs
    for (size_t chunk : {4ul << 20, 16ul << 20}) {
      for (int threads : {4, 8}) {
        const int K = 4;
        char* ring = nullptr;
        cudaHostAlloc((void**)&ring, K * chunk, cudaHostAllocDefault);
        cudaEvent_t ev[K];
        for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        t0 = now_ms();
        const size_t n = (bytes + chunk - 1) / chunk;
        for (size_t c = 0; c < n; ++c) {
          const int k = c % K;
          if (c >= (size_t)K) cudaEventSynchronize(ev[k]);
          const size_t off = c * chunk, len = std::min(chunk, bytes - off);
          std::vector<std::thread> th;
          for (int t = 0; t < threads; ++t)
            th.emplace_back([&, t] {
              const size_t a = len * t / threads, b = len * (t + 1) / threads;
              std::memcpy(ring + k * chunk + a, host.data() + off + a, b - a);
            });
          for (auto& x : th) x.join();
          cudaMemcpyAsync((char*)d + off, ring + k * chunk, len, cudaMemcpyHostToDevice, s);
          cudaEventRecord(ev[k], s);
        }
        cudaStreamSynchronize(s);
        printf("  staged chunk %zu MB x %d threads: %.2f ms\n", chunk >> 20, threads, now_ms() - t0);
        cudaFreeHost(ring);
      }
    }
    printf("pageable %.2f ms | register %.2f + pinned copy %.2f + unregister %.2f ms\n", pageable, reg, pinned, unreg);
  }
  return 0;
}
