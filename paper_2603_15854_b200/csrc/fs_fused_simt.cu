// fs_fused_simt.cu -- stage 1 of FlashSampling on CUDA cores.
//
// Same contract and epilogue as the tcgen05 kernel (fs_fused_tc.cu) but the projection is a
// plain fp32 FMA dot product per (row, column), in increasing d order.  Used for fp32 inputs
// (the tiny oracle configuration: true fp32, never TF32 -- DESIGN.md reading R13), for bf16
// shapes TMA cannot describe (D % 8 != 0), and as the sanitizer-friendly twin of the tensor-core
// kernel.  One CTA per 128-row aligned vocabulary tile; one candidate slot per tile.
#include <cuda_bf16.h>

#include "fs_epilogue.cuh"
#include "fs_kernels.h"

namespace fs {

constexpr int kSimtChunks = 8;     // up to 256 columns per launch

template <typename T>
__device__ __forceinline__ float ldf(const T* p) {
  if constexpr (sizeof(T) == 2) return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(p));
  else return *p;
}

template <typename T, bool LSE, bool PRQ>
__global__ void __launch_bounds__(128) fused_simt_kernel(const StageOneParams p) {
  __shared__ RowTab tab;
  __shared__ State scratch[4 * 256];
  const T* __restrict__ h = static_cast<const T*>(p.h);
  const T* __restrict__ W = static_cast<const T*>(p.W);
  fill_rowtab<PRQ>(&tab, p.B, p.temperature, p.seeds, p.steps, p.step, threadIdx.x, 128);
  __syncthreads();
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  const int base = blockIdx.x * 128;
  const int row = base + threadIdx.x;
  RowArgs ra;
  ra.valid = row < p.V;
  ra.v_global = (int32_t)(p.vocab_offset + row);
  ra.v_lo = (uint32_t)ra.v_global;
  ra.warp_v0 = (int32_t)(p.vocab_offset + base + 32 * q);
  ra.bias = (ra.valid && p.bias) ? p.bias[row] : 0.0f;
  EpiArgs ea{};
  ea.invtau = tab.invtau;
  ea.tab = &tab;
  ea.mask = p.mask;
  ea.mask_words = p.mask_words;
  ea.B = p.B;
  ea.row_offset = p.row_offset;
  ea.k0 = (uint32_t)p.seed;
  ea.k1 = (uint32_t)(p.seed >> 32);
  ea.c2 = ctr_step_lo(p.step);
  ea.c3 = ctr_step_hi(p.step, 0u);
  const T* wrow = W + (size_t)(ra.valid ? row : 0) * p.D;
  State st[kSimtChunks];
#pragma unroll
  for (int c = 0; c < kSimtChunks; ++c) {
    st[c] = state_empty();
    if (c * 32 >= p.B) continue;
    float acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.0f;
    const int nb = min(32, p.B - c * 32);
    for (int d = 0; d < p.D; ++d) {
      const float w = ldf(wrow + d);
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nb) acc[j] = fmaf(ldf(h + (size_t)(c * 32 + j) * p.D + d), w, acc[j]);
    }
    if (p.mode == 2) {                        // raw logits for the top-k fallback (f1)
      if (ra.valid)
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nb) p.mat_out[(int64_t)(c * 32 + j) * p.mat_ld + row] = acc[j];
      continue;
    }
    epi_columns<32, LSE, PRQ>(acc, c * 32, ra, ea, st[c], lane);
  }
  if (p.mode == 2) return;
  flush_states<kSimtChunks, 32>(st, scratch, 256, q, lane, threadIdx.x, p.B, p.part + (size_t)blockIdx.x * p.B, 1);
  if (threadIdx.x == 0) p.part_group[blockIdx.x] = base / p.group_size;
  sm100::pdl_launch_dependents();
}

cudaError_t launch_fused_simt(const StageOneParams& p, fs_dtype dtype, bool lse, cudaStream_t stream) {
  const int grid = (p.V + 127) / 128;
  const bool prq = p.seeds != nullptr;
#define FS_SIMT(T)                                                                                    \
  if (lse) { if (prq) fused_simt_kernel<T, true, true><<<grid, 128, 0, stream>>>(p);                  \
             else fused_simt_kernel<T, true, false><<<grid, 128, 0, stream>>>(p); }                   \
  else     { if (prq) fused_simt_kernel<T, false, true><<<grid, 128, 0, stream>>>(p);                 \
             else fused_simt_kernel<T, false, false><<<grid, 128, 0, stream>>>(p); }
  if (dtype == FS_BF16) { FS_SIMT(uint16_t) } else { FS_SIMT(float) }
#undef FS_SIMT
  return cudaGetLastError();
}

}  // namespace fs
