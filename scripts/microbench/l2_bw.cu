// l2_bw.cu -- L2 read bandwidth of this B200 (the L2 roofline of the config-5
// sweep, bench.py --sweep): every SM streams uint4 loads (L1-bypassing,
// ld.global.cg) over a buffer that fits in the 126 MB L2, many passes; the
// first pass warms it.  Also the same kernel over 4 GiB (HBM) for comparison.
// Prints JSON: {"l2_gbs": ..., "hbm_gbs": ..., "buffer_mb": ...}.
#include <cuda_runtime.h>

#include <cstdio>

__global__ void read_kernel(const uint4* __restrict__ p, size_t n, int passes, unsigned* sink) {
  unsigned acc = 0;
  for (int k = 0; k < passes; ++k)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      uint4 v = __ldcg(p + i);
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  if (acc == 0x12345678u) *sink = acc;
}

static float run(const uint4* p, size_t n, int passes, unsigned* sink, int sms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  read_kernel<<<sms * 4, 512>>>(p, n, 1, sink);  // warm
  cudaEventRecord(a);
  read_kernel<<<sms * 4, 512>>>(p, n, passes, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* sink;
  cudaMalloc(&sink, 4);
  const size_t small = 48ull << 20, big = 4ull << 30;
  uint4* p;
  cudaMalloc(&p, big);
  cudaMemset(p, 1, big);
  float best_l2 = 1e30f, best_hbm = 1e30f;
  for (int r = 0; r < 5; ++r) {
    const float t = run(p, small / 16, 50, sink, sms);
    if (t < best_l2) best_l2 = t;
    const float h = run(p, big / 16, 1, sink, sms);
    if (h < best_hbm) best_hbm = h;
  }
  printf("{\"l2_gbs\": %.1f, \"hbm_read_gbs\": %.1f, \"buffer_mb\": %zu, \"how\": \"ld.global.cg uint4 over a %zu-MB buffer, 50 passes after a warm pass, %d CTAs x 512 threads, best of 5 (CUDA events); HBM: one pass over 4 GiB\"}\n",
         (double)small * 50 / (best_l2 * 1e-3) / 1e9, (double)big / (best_hbm * 1e-3) / 1e9, small >> 20, small >> 20,
         sms * 4);
  return 0;
}
