// Minimal reproducer for the only racecheck report of the library (fs_fused_tc2.cu prologue):
// a cluster of 2 CTAs does nothing but the collective paired TMEM allocation, a cluster barrier,
// a read of the allocated address, and the paired deallocation.  There is no user-code shared
// memory write at all -- if compute-sanitizer --tool racecheck still reports "Write access at
// <unknown PC> vs Read access at tcgen05.alloc.cta_group::2", the report is the tool's model of the
// paired allocator (its hardware write of the result into both CTAs' slot), not a race in the kernel.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o racecheck_tmem_pair tools/racecheck_tmem_pair.cu
//   compute-sanitizer --tool racecheck ./racecheck_tmem_pair
// or, as the library is loaded (ctypes from Python; the standalone binary crashes racecheck itself):
//   nvcc ... -Xcompiler -fPIC -shared -DREPRO_AS_LIBRARY -o tools/bin/librepro.so tools/racecheck_tmem_pair.cu
//   compute-sanitizer --tool racecheck python -c "import ctypes; ctypes.CDLL('tools/bin/librepro.so').run_repro(3, 0)"
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2603_15854_b200/csrc/fs_sm100.cuh"

// variant bits (argv[2]): 1 = mbarriers initialised next to the slot before the allocation (as the
// library's prologue), 2 = allocation by warp 1 instead of warp 0, 4 = slot in dynamic shared memory,
// 8 = (pair) the leader's tcgen05.commit multicast-arrives on the barrier next to the slot, and every
// warp of both CTAs arrives remotely on the leader's neighbouring barrier (the kernel's tfull / tempty)
template <bool kPair>
__global__ void alloc_only(uint32_t* out, int variant) {
  __shared__ __align__(16) uint64_t bars_static[8];
  __shared__ uint32_t slot_static[4];
  extern __shared__ __align__(1024) uint8_t dyn[];
  uint64_t* bars = (variant & 4) ? reinterpret_cast<uint64_t*>(dyn) : bars_static;
  uint32_t* slot = (variant & 4) ? reinterpret_cast<uint32_t*>(dyn + 64) : slot_static;
  const int warp = threadIdx.x >> 5;
  if ((variant & 1) && threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) fs::sm100::mbar_init(&bars[i], i == 6 ? 8 : 1);
    fs::sm100::fence_barrier_init();
  }
  if (warp == ((variant & 2) ? 1 : 0)) {
    if (kPair) fs::sm100::tmem_alloc_pair(slot, 64);
    else fs::sm100::tmem_alloc(slot, 64);
  }
  fs::sm100::tc_fence_before();
  fs::sm100::cluster_sync();
  __syncthreads();
  fs::sm100::tc_fence_after();
  const uint32_t base = *slot;
  if (threadIdx.x == 0) out[blockIdx.x] = base;
  if (kPair && (variant & 8) && (variant & 1)) {
    const uint32_t rank = fs::sm100::cluster_ctarank();
    if (rank == 0 && threadIdx.x == 32) fs::sm100::mma_commit_pair(&bars[7], 0x3);   // hardware arrive, both CTAs
    fs::sm100::mbar_wait(&bars[7], 0);
    if ((threadIdx.x & 31) == 0) fs::sm100::mbar_arrive_cluster(fs::sm100::mapa(fs::sm100::smem_u32(&bars[6]), 0));
    if (rank == 0) fs::sm100::mbar_wait(&bars[6], 0);
  }
  fs::sm100::tc_fence_before();
  fs::sm100::cluster_sync();
  if (warp == ((variant & 2) ? 1 : 0)) {
    fs::sm100::tc_fence_after();
    if (kPair) fs::sm100::tmem_dealloc_pair(base, 64);
    else fs::sm100::tmem_dealloc(base, 64);
  }
}

template <bool kPair>
static cudaError_t launch(uint32_t* d, int variant) {     // cluster of 2 for the pair (as fs_fused_tc2.cu), none for the control
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = (variant & 4) ? 2048 : 0;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = kPair ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, alloc_only<kPair>, d, variant);
  if (e != cudaSuccess) return e;
  return cudaDeviceSynchronize();
}

extern "C" int run_repro(int which, int variant) {   // which: 1 control only, 2 pair only, 3 both
  uint32_t* d = nullptr;
  cudaError_t e0 = cudaMalloc(&d, 2 * 148 * sizeof(uint32_t));
  printf("malloc %s\n", cudaGetErrorString(e0));
  fflush(stdout);
  cudaError_t e1 = (which & 1) ? launch<false>(d, variant) : cudaSuccess;   // control: per-CTA allocation (cta_group::1)
  printf("cta_group::1 %s\n", cudaGetErrorString(e1));
  fflush(stdout);
  cudaError_t e2 = (which & 2) ? launch<true>(d, variant) : cudaSuccess;    // the paired allocation of fs_fused_tc2.cu
  printf("cta_group::2 %s\n", cudaGetErrorString(e2));
  fflush(stdout);
  uint32_t h[4] = {0, 0, 0, 0};
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("tmem base of CTAs 0..3: %u %u %u %u\n", h[0], h[1], h[2], h[3]);
  cudaFree(d);
  return (e1 == cudaSuccess && e2 == cudaSuccess) ? 0 : 1;
}

#ifndef REPRO_AS_LIBRARY
#include <cstdlib>
int main(int argc, char** argv) { return run_repro(argc > 1 ? atoi(argv[1]) : 3, argc > 2 ? atoi(argv[2]) : 0); }
#endif
