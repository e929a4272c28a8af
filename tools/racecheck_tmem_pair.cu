// Minimal reproducer for the only racecheck report of the library (fs_fused_tc2.cu prologue):
// a cluster of 2 CTAs does nothing but the collective paired TMEM allocation, a cluster barrier,
// a read of the allocated address, and the paired deallocation.  There is no user-code shared
// memory write at all -- if compute-sanitizer --tool racecheck still reports "Write access at
// <unknown PC> vs Read access at tcgen05.alloc.cta_group::2", the report is the tool's model of the
// paired allocator (its hardware write of the result into both CTAs' slot), not a race in the kernel.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o racecheck_tmem_pair tools/racecheck_tmem_pair.cu
//   compute-sanitizer --tool racecheck ./racecheck_tmem_pair
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2603_15854_b200/csrc/fs_sm100.cuh"

template <bool kPair>
__global__ void alloc_only(uint32_t* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    if (kPair) fs::sm100::tmem_alloc_pair(&slot, 64);
    else fs::sm100::tmem_alloc(&slot, 64);
  }
  fs::sm100::tc_fence_before();
  fs::sm100::cluster_sync();
  __syncthreads();
  fs::sm100::tc_fence_after();
  const uint32_t base = slot;
  if (threadIdx.x == 0) out[blockIdx.x] = base;
  fs::sm100::tc_fence_before();
  fs::sm100::cluster_sync();
  if (warp == 0) {
    fs::sm100::tc_fence_after();
    if (kPair) fs::sm100::tmem_dealloc_pair(base, 64);
    else fs::sm100::tmem_dealloc(base, 64);
  }
}

template <bool kPair>
static cudaError_t launch(uint32_t* d) {     // cluster of 2, as the library launches fs_fused_tc2.cu
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(64);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, alloc_only<kPair>, d);
  if (e != cudaSuccess) return e;
  return cudaDeviceSynchronize();
}

int main() {
  uint32_t* d = nullptr;
  cudaError_t e0 = cudaMalloc(&d, 2 * 148 * sizeof(uint32_t));
  printf("malloc %s\n", cudaGetErrorString(e0));
  fflush(stdout);
  cudaError_t e1 = launch<false>(d);        // control: per-CTA allocation (cta_group::1)
  printf("cta_group::1 %s\n", cudaGetErrorString(e1));
  fflush(stdout);
  cudaError_t e2 = launch<true>(d);         // the paired allocation of fs_fused_tc2.cu
  printf("cta_group::2 %s\n", cudaGetErrorString(e2));
  fflush(stdout);
  uint32_t h[4] = {0, 0, 0, 0};
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("tmem base of CTAs 0..3: %u %u %u %u\n", h[0], h[1], h[2], h[3]);
  cudaFree(d);
  return (e1 == cudaSuccess && e2 == cudaSuccess) ? 0 : 1;
}
