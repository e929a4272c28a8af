// tma_stream_bench.cu -- microbenchmark: how fast can a TMA ring stream a [V, D] bf16 matrix
// (the LM-head W) from HBM on B200, as a function of grid structure and ring geometry?
// Not part of the library; used to pick the stage-1 load design.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_stream_bench tools/tma_stream_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2603_15854_b200/csrc/fs_sm100.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

struct Args {
  int V, D, S, kbps, box_rows, persistent, tiles_per_cta_unit;
  unsigned long long* sink;
};

// One producer lane issues TMA loads of [box_rows x 64] boxes, KBPS boxes per stage (per row block
// of 128 rows: 128/box_rows boxes per k slice); one consumer lane waits and frees stages.
__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = a.S, KBPS = a.kbps;
  const int stage_bytes = 128 * 128 * KBPS;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * stage_bytes);
  uint64_t* empty = full + S;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { fs::sm100::mbar_init(&full[s], 1); fs::sm100::mbar_init(&empty[s], 1); }
    fs::sm100::fence_barrier_init();
  }
  __syncthreads();
  const int ntiles = (a.V + 127) / 128;
  const int num_kb = a.D / 64;
  int t_begin, t_end;
  if (a.persistent) {
    t_begin = (int)((long long)blockIdx.x * ntiles / gridDim.x);
    t_end = (int)((long long)(blockIdx.x + 1) * ntiles / gridDim.x);
  } else {
    t_begin = blockIdx.x;
    t_end = blockIdx.x + 1;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    int stage = 0; uint32_t phase = 0;
    for (int t = t_begin; t < t_end; ++t)
      for (int kb0 = 0; kb0 < num_kb; kb0 += KBPS) {
        fs::sm100::mbar_wait(&empty[stage], phase ^ 1);
        fs::sm100::mbar_arrive_expect_tx(&full[stage], stage_bytes);
        for (int j = 0; j < KBPS; ++j)
          for (int r = 0; r < 128; r += a.box_rows)
            fs::sm100::tma_load_2d(smem + (size_t)stage * stage_bytes + j * 16384 + r * 128, &tm, &full[stage],
                                   (kb0 + j) * 64, t * 128 + r, fs::sm100::policy_evict_first());
        if (++stage == S) { stage = 0; phase ^= 1; }
      }
  } else if (warp == 1 && lane == 0) {
    int stage = 0; uint32_t phase = 0;
    unsigned long long acc = 0;
    for (int t = t_begin; t < t_end; ++t)
      for (int kb0 = 0; kb0 < num_kb; kb0 += KBPS) {
        fs::sm100::mbar_wait(&full[stage], phase);
        acc += *reinterpret_cast<volatile uint32_t*>(smem + (size_t)stage * stage_bytes);
        fs::sm100::mbar_arrive(&empty[stage]);
        if (++stage == S) { stage = 0; phase ^= 1; }
      }
    if (acc == 0x123456789ULL) a.sink[0] = acc;
  }
}

__global__ void fill_random(uint32_t* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 0x9E3779B9u + 0x7F4A7C15u;
    x ^= x >> 16; x *= 0x85EBCA6Bu; x ^= x >> 13; x *= 0xC2B2AE35u; x ^= x >> 16;
    p[i] = x & 0xBFFFBFFFu;   // two bf16 values, |x| < 2 (no inf/nan patterns)
  }
}

int main(int argc, char** argv) {
  const bool rnd = argc > 1 && argv[1][0] == 'r';
  const int V = 128256, D = 4096;
  void* W;
  CK(cudaMalloc(&W, (size_t)V * D * 2));
  CK(cudaMemset(W, 1, (size_t)V * D * 2));
  if (rnd) fill_random<<<1184, 256>>>(static_cast<uint32_t*>(W), (size_t)V * D / 2);
  printf("W data: %s\n", rnd ? "random bits" : "memset(1)");
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  void* fn;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto encode = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                              CUtensorMapFloatOOBfill)>(fn);
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  struct Cfg { int persistent, S, kbps, box_rows, ctas_per_sm; };
  std::vector<Cfg> cfgs = {
      {1, 12, 1, 128, 1}, {1, 6, 2, 128, 1}, {1, 3, 4, 128, 1}, {1, 13, 1, 128, 1},
      {0, 12, 1, 128, 1}, {0, 6, 2, 128, 1}, {0, 3, 4, 128, 1}, {0, 13, 1, 128, 1},
      {1, 6, 1, 128, 2}, {0, 6, 1, 128, 2}, {1, 3, 2, 128, 2}, {0, 3, 2, 128, 2},
      {1, 4, 1, 128, 3}, {0, 4, 1, 128, 3}, {1, 12, 1, 64, 1}, {0, 12, 1, 64, 1},
      {1, 12, 1, 32, 1}, {0, 12, 1, 32, 1}, {0, 24, 1, 128, 1},
  };
  if (getenv("ONLY_BEST")) cfgs = {{1, 3, 4, 128, 1}, {1, 12, 1, 128, 1}};
  for (int promo : {0, 3}) {
    if (getenv("ONLY_BEST") && promo == 0) continue;
    for (const Cfg& c : cfgs) {
      CUtensorMap tm;
      const cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)V};
      const cuuint64_t strides[1] = {(cuuint64_t)D * 2};
      const cuuint32_t box[2] = {64u, (cuuint32_t)c.box_rows};
      const cuuint32_t estr[2] = {1u, 1u};
      if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, W, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_128B, (CUtensorMapL2promotion)promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != 0) {
        printf("encode failed\n");
        continue;
      }
      Args a{V, D, c.S, c.kbps, c.box_rows, c.persistent, 0, sink};
      const size_t smem = 1024 + (size_t)c.S * 128 * 128 * c.kbps + 2 * c.S * 8 + 64;
      if (smem > 227 * 1024 / c.ctas_per_sm) { printf("skip (smem)\n"); continue; }
      const int grid = c.persistent ? sms * c.ctas_per_sm : (V + 127) / 128;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      for (int w = 0; w < 5; ++w) stream_kernel<<<grid, 64, smem>>>(tm, a);
      CK(cudaGetLastError());
      cudaEventRecord(e0);
      const int iters = getenv("ITERS") ? atoi(getenv("ITERS")) : 20;
      for (int i = 0; i < iters; ++i) stream_kernel<<<grid, 64, smem>>>(tm, a);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double us = 1e3 * ms / iters;
      printf("promo=%d persistent=%d S=%2d kbps=%d box_rows=%3d ctas/sm=%d stage=%3d KB inflight=%4d KB/SM : %8.2f us %8.1f GB/s\n",
             promo, c.persistent, c.S, c.kbps, c.box_rows, c.ctas_per_sm, 16 * c.kbps, 16 * c.kbps * c.S * c.ctas_per_sm,
             us, 2.0 * V * D / (us * 1e-6) / 1e9);
    }
  }
  return 0;
}
