// Random-chunk HBM read ceiling on this GPU: warps read CHUNK-byte chunks at
// random 128-B-aligned offsets of a large buffer (the access pattern of the
// pair-trend index kernel) vs a sequential sweep of the same byte count.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rc random_chunks.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

__global__ void chunk_read(const uint4* __restrict__ buf, const uint32_t* __restrict__ idx, uint32_t n_chunks,
                           uint32_t chunk_v4, unsigned long long* sink) {
  const int lane = threadIdx.x & 31;
  const uint32_t w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= n_chunks) return;
  const uint4* p = buf + (uint64_t)idx[w] * chunk_v4;
  uint32_t acc = 0;
  for (uint32_t v = lane; v < chunk_v4; v += 32) {
    const uint4 x = __ldg(p + v);
    acc ^= x.x ^ x.y ^ x.z ^ x.w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

// the index kernel's shape: a warp ANDs G chunks (one candidate's pairs);
// DEP: the chunks are read one after another (the next load waits for the
// AND), else all G chunks' loads are issued before combining
template <int G, bool DEP>
__global__ void chunk_and(const uint4* __restrict__ buf, const uint32_t* __restrict__ idx, uint32_t n_groups,
                          uint32_t chunk_v4, unsigned long long* sink) {
  const int lane = threadIdx.x & 31;
  const uint32_t w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= n_groups) return;
  uint32_t acc = 0;
  for (uint32_t v = lane; v < chunk_v4; v += 32) {
    uint4 f = make_uint4(~0u, ~0u, ~0u, ~0u);
    if (DEP) {
      for (int g = 0; g < G; ++g) {
        const uint4 x = __ldg(buf + (uint64_t)idx[w * G + g] * chunk_v4 + v);
        f.x &= x.x; f.y &= x.y; f.z &= x.z; f.w &= x.w;
        if (f.x == 0x9u) break;  // data-dependent: the next load waits for this one
      }
    } else {
      uint4 x[G];
#pragma unroll
      for (int g = 0; g < G; ++g) x[g] = __ldg(buf + (uint64_t)idx[w * G + g] * chunk_v4 + v);
#pragma unroll
      for (int g = 0; g < G; ++g) { f.x &= x[g].x; f.y &= x[g].y; f.z &= x[g].z; f.w &= x[g].w; }
    }
    acc += __popc(f.x) + __popc(f.y) + __popc(f.z) + __popc(f.w);
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
  const size_t total = 2560ull << 20;  // 2.5 GiB buffer
  uint4* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t read_bytes = 120ull << 20;
  std::mt19937 rng(1);
  for (uint32_t chunk : {512u, 1024u, 2560u, 4096u, 10240u, 65536u}) {
    const uint32_t n = (uint32_t)(read_bytes / chunk);
    const uint32_t n_slots = (uint32_t)(total / chunk);
    std::vector<uint32_t> h(n);
    for (auto& x : h) x = rng() % n_slots;
    std::vector<uint32_t> hs(n);
    for (uint32_t i = 0; i < n; ++i) hs[i] = i;  // sequential
    uint32_t *d, *ds;
    cudaMalloc(&d, n * 4);
    cudaMalloc(&ds, n * 4);
    cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(ds, hs.data(), n * 4, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 2; ++mode) {
      const uint32_t* ix = mode ? ds : d;
      float best = 1e9f;
      for (int rep = 0; rep < 8; ++rep) {
        cudaMemset(buf, rep, 256ull << 20);  // evict (L2 126 MB)
        cudaEventRecord(e0);
        chunk_read<<<(n + 7) / 8, 256>>>(buf, ix, n, chunk / 16, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("chunk %6u B %-10s %8u chunks: %.4f ms  %.0f GB/s\n", chunk, mode ? "sequential" : "random", n, best,
             n * (double)chunk / (best * 1e-3) / 1e9);
    }
    cudaFree(d);
    cudaFree(ds);
  }
  {  // 2560-B chunks, groups of 3 per warp (a length-4 candidate), dependent vs batched
    const uint32_t chunk = 2560, n = (uint32_t)(read_bytes / chunk) / 3 * 3, n_slots = (uint32_t)(total / chunk);
    std::vector<uint32_t> h(n);
    for (auto& x : h) x = rng() % n_slots;
    uint32_t* d;
    cudaMalloc(&d, n * 4);
    cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 2; ++mode) {
      float best = 1e9f;
      for (int rep = 0; rep < 8; ++rep) {
        cudaMemset(buf, rep, 256ull << 20);
        cudaEventRecord(e0);
        if (mode) chunk_and<3, false><<<(n / 3 + 7) / 8, 256>>>(buf, d, n / 3, chunk / 16, sink);
        else chunk_and<3, true><<<(n / 3 + 7) / 8, 256>>>(buf, d, n / 3, chunk / 16, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("chunk %6u B x3 per warp %-9s %8u chunks: %.4f ms  %.0f GB/s\n", chunk, mode ? "batched" : "dependent", n,
             best, n * (double)chunk / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
