// h2d_probe.cu -- how fast do SM-initiated reads of pinned host memory deliver one decode step's h
// (B x D bf16), and in what order?  Question behind it: can the in-kernel staging of
// fs_sample_staged release h in K-chunks (the first K-slices early) instead of all at once?
//   mode 0: every CTA copies one contiguous 1/G slice (the current staging); per-CTA done stamp
//   mode 1: NCH chunks; every thread issues its loads of ALL chunks first, then stores chunk by
//           chunk, each followed by fence + CTA barrier + stamp (chunk c's time = max over CTAs)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/h2d_probe tools/h2d_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int kMaxCh = 16;

__global__ void probe(const uint4* __restrict__ src, uint4* dst, size_t n16, int mode, int nch, uint64_t* stamps) {
  const int G = gridDim.x, c0 = blockIdx.x;
  if (threadIdx.x == 0) stamps[(size_t)c0 * (kMaxCh + 1)] = gtime();
  if (mode == 0) {
    const size_t per = (n16 + G - 1) / G, lo = per * c0, hi = min(n16, lo + per);
    for (size_t i = lo + threadIdx.x; i < hi; i += blockDim.x) dst[i] = src[i];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) stamps[(size_t)c0 * (kMaxCh + 1) + 1] = gtime();
    return;
  }
  // chunk c = [c*n16/nch, (c+1)*n16/nch); CTA share of each chunk = 1/G of it
  uint4 v[kMaxCh];
  size_t idx[kMaxCh];
#pragma unroll
  for (int c = 0; c < kMaxCh; ++c) {
    idx[c] = ~size_t(0);
    if (c < nch) {
      const size_t a = n16 * c / nch, b = n16 * (c + 1) / nch, per = (b - a + G - 1) / G;
      const size_t i = a + per * c0 + threadIdx.x;
      if (threadIdx.x < per && i < b) { idx[c] = i; v[c] = src[i]; }
    }
  }
#pragma unroll
  for (int c = 0; c < kMaxCh; ++c) {
    if (c < nch) {
      if (idx[c] != ~size_t(0)) dst[idx[c]] = v[c];
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) stamps[(size_t)c0 * (kMaxCh + 1) + 1 + c] = gtime();
    }
  }
}

int main() {
  const int Bs[] = {1, 32, 256};
  const int D = 4096;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int B : Bs) {
    const size_t bytes = (size_t)B * D * 2, n16 = bytes / 16;
    void* hsrc;
    cudaHostAlloc(&hsrc, bytes, cudaHostAllocMapped);
    memset(hsrc, 1, bytes);
    void* hd;
    cudaHostGetDevicePointer(&hd, hsrc, 0);
    void* d;
    cudaMalloc(&d, bytes);
    uint64_t* st;
    const int G = sms;
    cudaMalloc(&st, (size_t)G * (kMaxCh + 1) * 8);
    std::vector<uint64_t> hs((size_t)G * (kMaxCh + 1));
    struct Cfg { int mode, nch, threads; };
    const Cfg cfgs[] = {{0, 1, 512}, {1, 4, 512}, {1, 8, 512}, {1, 16, 512}, {0, 1, 128}};
    for (const Cfg& c : cfgs) {
      std::vector<std::vector<double>> per(c.mode ? c.nch : 1);
      std::vector<double> ktime;
      for (int rep = 0; rep < 30; ++rep) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        probe<<<G, c.threads>>>(static_cast<const uint4*>(hd), static_cast<uint4*>(d), n16, c.mode, c.nch, st);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpy(hs.data(), st, hs.size() * 8, cudaMemcpyDeviceToHost);
        if (rep < 5) continue;
        ktime.push_back(ms * 1e3);
        uint64_t t0 = ~0ull;
        for (int i = 0; i < G; ++i) t0 = std::min(t0, hs[(size_t)i * (kMaxCh + 1)]);
        for (size_t k = 0; k < per.size(); ++k) {
          uint64_t m = 0;
          for (int i = 0; i < G; ++i) m = std::max(m, hs[(size_t)i * (kMaxCh + 1) + 1 + k]);
          per[k].push_back((m - t0) * 1e-3);
        }
      }
      auto med = [](std::vector<double> x) { std::sort(x.begin(), x.end()); return x[x.size() / 2]; };
      printf("B=%3d bytes=%7zu mode=%d nch=%2d thr=%3d kernel %.2f us  chunk done (us after first CTA start):", B, bytes,
             c.mode, c.nch, c.threads, med(ktime));
      for (auto& x : per) printf(" %.2f", med(x));
      printf("\n");
    }
    cudaFree(d);
    cudaFree(st);
    cudaFreeHost(hsrc);
  }
  return 0;
}
