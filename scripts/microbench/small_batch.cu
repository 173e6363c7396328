// C++ timing of ebic_eval_counts on pinned inputs (no Python): where the host
// API's microseconds go.  usage: e2e_host_api [R C P]  (default C3: 20000 1000
// 16384; the SPEC shape: 20000 250 392).  Also times the floor: an empty
// kernel launch + stream sync, and a small pinned H2D + sync.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include <cuda_runtime.h>
#include "ebic.h"
__global__ void empty_kernel() {}
int main(int argc, char** argv) {
  const uint64_t R = argc > 3 ? strtoull(argv[1], nullptr, 10) : 20000;
  const uint64_t C = argc > 3 ? strtoull(argv[2], nullptr, 10) : 1000;
  const uint64_t P = argc > 3 ? strtoull(argv[3], nullptr, 10) : 16384;
  printf("R=%llu C=%llu P=%llu\n", (unsigned long long)R, (unsigned long long)C, (unsigned long long)P);
  std::vector<float> m(R * C);
  std::mt19937 rng(1);
  std::normal_distribution<float> nd;
  for (auto& x : m) x = nd(rng);
  ebic_ctx* ctx;
  ebic_ctx_create(0, &ctx);
  ebic_matrix_upload_f32(ctx, m.data(), R, C, 0);
  ebic_matrix_prepare(ctx, 0.03);
  uint32_t* blk;
  uint32_t* out;
  cudaMallocHost(&blk, (P + 1 + P * 5) * 4);
  cudaMallocHost(&out, P * 4);
  uint32_t* offs = blk;
  uint32_t* cols = blk + P + 1;
  offs[0] = 0;
  for (uint64_t i = 0; i < P; ++i) {
    const uint32_t L = 3 + rng() % 3;
    for (uint32_t k = 0; k < L; ++k) cols[offs[i] + k] = rng() % C;  // (duplicates allowed)
    offs[i + 1] = offs[i] + L;
  }
  // pack cols right after offs (one block)
  for (int rep = 0; rep < 20; ++rep) ebic_eval_counts(ctx, cols, offs, P, 0.03, 0, out);
  const int N = 200;
  auto t0 = std::chrono::steady_clock::now();
  for (int rep = 0; rep < N; ++rep) ebic_eval_counts(ctx, cols, offs, P, 0.03, 0, out);
  auto t1 = std::chrono::steady_clock::now();
  printf("ebic_eval_counts pinned block, C++: %.1f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
  for (int round = 0; round < 2; ++round) {
    t0 = std::chrono::steady_clock::now();
    for (int rep = 0; rep < N; ++rep) ebic_eval_counts(ctx, cols, offs, P, 0.03, 0, out);
    t1 = std::chrono::steady_clock::now();
    printf("  again: %.1f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
  }
  {  // the same steps by hand: H2D of the block, device API into the pinned output's alias, sync
    uint32_t *dblk, *dout = nullptr;
    cudaMalloc(&dblk, (P + 1 + offs[P]) * 4);
    cudaHostGetDevicePointer((void**)&dout, out, 0);
    cudaStream_t s2;
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    for (int rep = 0; rep < 20; ++rep) {
      cudaMemcpyAsync(dblk, blk, (P + 1 + offs[P]) * 4, cudaMemcpyHostToDevice, s2);
      ebic_eval_counts_device(ctx, dblk + P + 1, dblk, P, 0.03, 0, dout, s2);
      cudaStreamSynchronize(s2);
    }
    t0 = std::chrono::steady_clock::now();
    for (int rep = 0; rep < N; ++rep) {
      cudaMemcpyAsync(dblk, blk, (P + 1 + offs[P]) * 4, cudaMemcpyHostToDevice, s2);
      ebic_eval_counts_device(ctx, dblk + P + 1, dblk, P, 0.03, 0, dout, s2);
      cudaStreamSynchronize(s2);
    }
    t1 = std::chrono::steady_clock::now();
    printf("by hand (H2D + device API into the pinned alias + sync): %.1f us\n",
           std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
  }
  // device-resident for comparison
  uint32_t *dc, *dof, *dn;
  cudaMalloc(&dc, offs[P] * 4); cudaMalloc(&dof, (P + 1) * 4); cudaMalloc(&dn, P * 4);
  cudaMemcpy(dc, cols, offs[P] * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dof, offs, (P + 1) * 4, cudaMemcpyHostToDevice);
  cudaStream_t s; cudaStreamCreate(&s);
  for (int rep = 0; rep < 20; ++rep) { ebic_eval_counts_device(ctx, dc, dof, P, 0.03, 0, dn, s); cudaStreamSynchronize(s); }
  t0 = std::chrono::steady_clock::now();
  for (int rep = 0; rep < N; ++rep) { ebic_eval_counts_device(ctx, dc, dof, P, 0.03, 0, dn, s); cudaStreamSynchronize(s); }
  t1 = std::chrono::steady_clock::now();
  printf("ebic_eval_counts_device + sync, C++: %.1f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
  {  // floor: an empty kernel launch + sync, and a small pinned H2D + sync
    for (int rep = 0; rep < 20; ++rep) { empty_kernel<<<1, 32, 0, s>>>(); cudaStreamSynchronize(s); }
    t0 = std::chrono::steady_clock::now();
    for (int rep = 0; rep < N; ++rep) { empty_kernel<<<1, 32, 0, s>>>(); cudaStreamSynchronize(s); }
    t1 = std::chrono::steady_clock::now();
    printf("floor: empty kernel + sync: %.1f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
    t0 = std::chrono::steady_clock::now();
    for (int rep = 0; rep < N; ++rep) {
      cudaMemcpyAsync(dc, blk, (P + 1 + offs[P]) * 4 < offs[P] * 4 ? (P + 1 + offs[P]) * 4 : offs[P] * 4,
                      cudaMemcpyHostToDevice, s);
      cudaStreamSynchronize(s);
    }
    t1 = std::chrono::steady_clock::now();
    printf("floor: pinned H2D of the population + sync: %.1f us\n",
           std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int rep = 0; rep < N; ++rep) ebic_eval_counts_device(ctx, dc, dof, P, 0.03, 0, dn, s);
  cudaEventRecord(e1, s); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("back-to-back kernels (events): %.1f us\n", ms * 1e3 / N);
  t0 = std::chrono::steady_clock::now();
  for (int rep = 0; rep < N; ++rep) { cudaMemcpyAsync(dc, blk, (P + 1 + offs[P]) * 4, cudaMemcpyHostToDevice, s); cudaStreamSynchronize(s); }
  t1 = std::chrono::steady_clock::now();
  printf("H2D of the block + sync: %.1f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
  {
    cudaPointerAttributes a;
    for (int rep = 0; rep < 100; ++rep) cudaPointerGetAttributes(&a, blk);
    t0 = std::chrono::steady_clock::now();
    for (int rep = 0; rep < 1000; ++rep) cudaPointerGetAttributes(&a, blk + rep);
    t1 = std::chrono::steady_clock::now();
    printf("cudaPointerGetAttributes: %.2f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / 1000);
    int dev;
    t0 = std::chrono::steady_clock::now();
    for (int rep = 0; rep < 1000; ++rep) cudaSetDevice(0);
    t1 = std::chrono::steady_clock::now();
    printf("cudaSetDevice: %.2f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / 1000);
    (void)dev;
  }
  return 0;
}
