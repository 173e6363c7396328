// How should the host API move a step's population block to the device?
// (a) cudaMemcpyAsync (copy engine) then the count kernel (CE -> SM dependency);
// (b) an SM copy kernel reading the page-locked block through its device alias;
// (c) (a) captured in a CUDA graph.  Each step ends with a stream sync, the
// counts land in page-locked memory (the kernel writes them through the alias).
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <random>
#include <vector>
#include <cuda_runtime.h>
#include "ebic.h"

__global__ void fetch_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int main() {
  const uint64_t R = 20000, C = 1000, P = 16384;
  std::vector<float> m(R * C);
  std::mt19937 rng(1);
  std::normal_distribution<float> nd;
  for (auto& x : m) x = nd(rng);
  ebic_ctx* ctx;
  ebic_ctx_create(0, &ctx);
  ebic_matrix_upload_f32(ctx, m.data(), R, C, 0);
  ebic_matrix_prepare(ctx, 0.03);
  uint32_t *blk, *out;
  cudaHostAlloc(&blk, (P + 1 + P * 5) * 4 + 64, cudaHostAllocMapped);
  cudaHostAlloc(&out, P * 4, cudaHostAllocMapped);
  uint32_t* offs = blk;
  uint32_t* cols = blk + P + 1;
  offs[0] = 0;
  for (uint64_t i = 0; i < P; ++i) {
    const uint32_t L = 3 + rng() % 3;
    for (uint32_t k = 0; k < L; ++k) cols[offs[i] + k] = rng() % C;
    offs[i + 1] = offs[i] + L;
  }
  const size_t bytes = (P + 1 + offs[P]) * 4, n16 = (bytes + 15) / 16;
  printf("block %zu B\n", bytes);
  uint32_t *dblk, *hblk_dev, *dout;
  cudaMalloc(&dblk, n16 * 16);
  cudaHostGetDevicePointer((void**)&hblk_dev, blk, 0);
  cudaHostGetDevicePointer((void**)&dout, out, 0);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const int N = 300;
  auto timeit = [&](const char* name, auto&& step) {
    for (int r = 0; r < 30; ++r) step();
    double best = 1e30;
    for (int round = 0; round < 3; ++round) {
      auto t0 = std::chrono::steady_clock::now();
      for (int r = 0; r < N; ++r) step();
      auto t1 = std::chrono::steady_clock::now();
      best = std::min(best, std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
    }
    printf("%-58s %.1f us   (err %s)\n", name, best, cudaGetErrorString(cudaGetLastError()));
  };
  timeit("ebic_eval_counts (host API, pinned)", [&] { ebic_eval_counts(ctx, cols, offs, P, 0.03, 0, out); });
  {
    setenv("EBIC_HOST_IN", "1", 1);
    ebic_ctx* c2;
    ebic_ctx_create(0, &c2);
    unsetenv("EBIC_HOST_IN");
    ebic_matrix_upload_f32(c2, m.data(), R, C, 0);
    ebic_matrix_prepare(c2, 0.03);
    std::vector<uint32_t> ref(out, out + P);
    timeit("ebic_eval_counts, EBIC_HOST_IN=1 (kernel reads the bus)", [&] { ebic_eval_counts(c2, cols, offs, P, 0.03, 0, out); });
    printf("    same counts: %s\n", std::equal(ref.begin(), ref.end(), out) ? "yes" : "NO");
    ebic_ctx_destroy(c2);
  }
  timeit("device API + sync (inputs resident)", [&] {
    ebic_eval_counts_device(ctx, dblk + P + 1, dblk, P, 0.03, 0, dout, s);
    cudaStreamSynchronize(s);
  });
  timeit("(a) cudaMemcpyAsync + device API + sync", [&] {
    cudaMemcpyAsync(dblk, blk, bytes, cudaMemcpyHostToDevice, s);
    ebic_eval_counts_device(ctx, dblk + P + 1, dblk, P, 0.03, 0, dout, s);
    cudaStreamSynchronize(s);
  });
  for (int grid : {148, 296, 592}) {
    char name[96];
    snprintf(name, sizeof name, "(b) SM fetch kernel <<<%d,256>>> + device API + sync", grid);
    timeit(name, [&] {
      fetch_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const uint4*>(hblk_dev), reinterpret_cast<uint4*>(dblk), n16);
      ebic_eval_counts_device(ctx, dblk + P + 1, dblk, P, 0.03, 0, dout, s);
      cudaStreamSynchronize(s);
    });
    snprintf(name, sizeof name, "    fetch kernel <<<%d,256>>> alone + sync", grid);
    timeit(name, [&] {
      fetch_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const uint4*>(hblk_dev), reinterpret_cast<uint4*>(dblk), n16);
      cudaStreamSynchronize(s);
    });
  }
  timeit("    cudaMemcpyAsync alone + sync", [&] {
    cudaMemcpyAsync(dblk, blk, bytes, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
  });
  {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    cudaMemcpyAsync(dblk, blk, bytes, cudaMemcpyHostToDevice, s);
    ebic_eval_counts_device(ctx, dblk + P + 1, dblk, P, 0.03, 0, dout, s);
    cudaStreamEndCapture(s, &g);
    if (cudaGraphInstantiate(&ge, g, 0) == cudaSuccess)
      timeit("(c) graph[memcpy + count] + sync", [&] {
        cudaGraphLaunch(ge, s);
        cudaStreamSynchronize(s);
      });
    else
      printf("(c) capture failed: %s\n", cudaGetErrorString(cudaGetLastError()));
  }
  {
    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
    float a = 0, b = 0;
    for (int r = 0; r < N; ++r) {
      cudaEventRecord(e0, s);
      cudaMemcpyAsync(dblk, blk, bytes, cudaMemcpyHostToDevice, s);
      cudaEventRecord(e1, s);
      ebic_eval_counts_device(ctx, dblk + P + 1, dblk, P, 0.03, 0, dout, s);
      cudaEventRecord(e2, s);
      cudaStreamSynchronize(s);
      float x, y;
      cudaEventElapsedTime(&x, e0, e1);
      cudaEventElapsedTime(&y, e1, e2);
      a += x; b += y;
    }
    printf("events: H2D %.1f us, count %.1f us\n", a * 1e3 / N, b * 1e3 / N);
  }
  return 0;
}
