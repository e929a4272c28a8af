// fs_probe.cu -- read-only HBM roofline probe ("a measured read-only peak (a 1 GiB
// bf16 read-reduction kernel), because the copy peak counts read+write traffic").
//
// Every CTA of a persistent grid (two per SM) streams one contiguous slice of `src` into a shared-
// memory ring with 1-D bulk copies (cp.async.bulk: the TMA engine the sampling kernels stream W with,
// minus the tensor map), 16 KB per stage, six stages in flight (the fastest geometry of the sweep in
// profiles/r02/read_probe_geometry.log); one consumer thread folds the first 8 bytes of every
// chunk into an XOR (so no load is dead) and frees the stage.  bench.py divides the bytes by the
// launch time: the ceiling a pure W stream can reach on this GPU, next to the copy peak of
// MEASURED_PEAKS.json.
#include <cuda_runtime.h>

#include <cstdint>

#include "fs_kernels.h"
#include "fs_sm100.cuh"

namespace fs {

namespace {
constexpr int kProbeChunk = 16384;
constexpr int kProbeStages = 6;

__device__ __forceinline__ void bulk_load(void* smem_dst, const void* src, uint32_t bytes, uint64_t* bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          sm100::smem_u32(smem_dst)),
      "l"(src), "r"(bytes), "r"(sm100::smem_u32(bar)), "l"(policy)
      : "memory");
}
}  // namespace

// Slice of CTA c: [c * per, min(bytes, (c + 1) * per)), per = ceil(bytes / G) rounded up to 16 bytes;
// chunks of kProbeChunk bytes from the slice start (the last one shorter).
__global__ void __launch_bounds__(64, 2) read_probe_kernel(const uint8_t* __restrict__ src, size_t bytes,
                                                           unsigned long long* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)kProbeStages * kProbeChunk);
  uint64_t* empty = full + kProbeStages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kProbeStages; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    sm100::fence_barrier_init();
  }
  __syncthreads();
  const size_t per = ((bytes + gridDim.x - 1) / gridDim.x + 15) & ~size_t(15);
  const size_t lo = min(bytes, per * blockIdx.x), hi = min(bytes, lo + per);
  if (threadIdx.x == 0) {
    const uint64_t pol = sm100::policy_evict_first();
    int stage = 0;
    uint32_t phase = 0;
    for (size_t off = lo; off < hi; off += kProbeChunk) {
      const uint32_t n = (uint32_t)min((size_t)kProbeChunk, hi - off);
      sm100::mbar_wait(&empty[stage], phase ^ 1);
      sm100::mbar_arrive_expect_tx(&full[stage], n);
      bulk_load(ring + (size_t)stage * kProbeChunk, src + off, n, &full[stage], pol);
      if (++stage == kProbeStages) { stage = 0; phase ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    int stage = 0;
    uint32_t phase = 0;
    unsigned long long acc = 0;
    for (size_t off = lo; off < hi; off += kProbeChunk) {
      sm100::mbar_wait(&full[stage], phase);
      acc ^= *reinterpret_cast<volatile unsigned long long*>(ring + (size_t)stage * kProbeChunk);
      sm100::mbar_arrive(&empty[stage]);
      if (++stage == kProbeStages) { stage = 0; phase ^= 1; }
    }
    if (lo < hi) atomicXor(sink, acc);
  }
}

cudaError_t launch_read_probe(const void* src, size_t bytes, unsigned long long* sink, int grid, cudaStream_t stream) {
  const size_t smem = 1024 + (size_t)kProbeStages * kProbeChunk + 2 * kProbeStages * 8;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(read_probe_kernel), (int)smem);
  if (e != cudaSuccess) return e;
  read_probe_kernel<<<grid, 64, smem, stream>>>(static_cast<const uint8_t*>(src), bytes, sink);
  return cudaGetLastError();
}

}  // namespace fs
