// fs_fused_tc.cu -- stage 1 of FlashSampling on sm_100a tensor cores.
//
// Alg. 2 stage 1 as a persistent, warp-specialised, swap-AB tcgen05 GEMM
// whose epilogue samples instead of storing logits:
//   * grid = #SMs persistent CTAs, each owning a balanced contiguous range of vocabulary rows
//     (16-row granularity, fs_epilogue.cuh cta_rows): W is streamed from HBM exactly once.
//   * MMA shape M = 128 vocabulary rows (A = W tile, K-major) x N = BN batch rows (B = h tile,
//     K-major, zero-filled past B by TMA) x K = 16, fp32 accumulation in TMEM.
//   * warp 0: TMA producer (W with L2 evict_first, h with evict_last) into an S-stage ring of
//             64-wide K slices (128-byte swizzle);
//     warp 1: TMEM allocator + single-thread MMA issuer; double-buffered accumulators (2 x BN
//             columns) so the epilogue of tile t overlaps the MMAs of tile t+1;
//     warps 2-5: epilogue, one per TMEM lane quadrant: tcgen05.ld -> registers -> transform +
//             Philox + Gumbel + warp argmax (fs_epilogue.cuh) -> one candidate per (row, CTA,
//             group segment) written to the candidate buffer.  Logits never leave the SM.
#include <cuda.h>
#include <cuda_runtime.h>

#include "fs_epilogue.cuh"
#include "fs_kernels.h"

namespace fs {

constexpr int kThreadsTC = 192;          // 6 warps
constexpr int kBlockM = 128;
constexpr int kBlockK = 64;              // 64 bf16 = 128 B = one swizzle row
constexpr int kWStageBytes = kBlockM * kBlockK * 2;

template <int BN>
struct TcCfg {
  static constexpr int kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                   : (2 * BN <= 256) ? 256 : 512;
  static constexpr int kHStageBytes = BN * kBlockK * 2;
  static constexpr int kStageBytes = kWStageBytes + kHStageBytes;
  static constexpr int kColsPerChunk = BN < 32 ? BN : 32;
  static constexpr int kChunks = BN / kColsPerChunk;
  // bytes after the stage ring: 2S+4 mbarriers, tmem address, invtau[BN], scratch[4][BN]
  static constexpr int extra_bytes(int S) { return (2 * S + 4) * 8 + 16 + BN * 4 + 4 * BN * 16 + 64; }
};

template <int BN, bool LSE>
__global__ void __launch_bounds__(kThreadsTC, 1)
fused_tc_kernel(const __grid_constant__ CUtensorMap tmW128, const __grid_constant__ CUtensorMap tmW16,
                const __grid_constant__ CUtensorMap tmH, const StageOneParams p) {
  using Cfg = TcCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages;
  uint8_t* w_ring = smem;
  uint8_t* h_ring = smem + (size_t)S * kWStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(h_ring + (size_t)S * Cfg::kHStageBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* invtau = reinterpret_cast<float*>(tmem_slot + 4);
  State* scratch = reinterpret_cast<State*>(invtau + BN);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    sm100::prefetch_tmap(&tmW128);
    sm100::prefetch_tmap(&tmW16);
    sm100::prefetch_tmap(&tmH);
    for (int s = 0; s < S; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&tfull[i], 1);
      sm100::mbar_init(&tempty[i], 128);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  for (int b = threadIdx.x; b < BN; b += kThreadsTC) {
    float it = __int_as_float(0x7FC00000);                 // NaN: padding column / invalid tau
    if (b < p.B) {
      const float t = p.temperature ? p.temperature[b] : 1.0f;
      if (t > 0.0f && isfinite(t)) it = 1.0f / t;
    }
    invtau[b] = it;
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  sm100::pdl_launch_dependents();

  int r0, r1;
  cta_rows(blockIdx.x, gridDim.x, p.V, r0, r1);
  const int num_kb = (p.D + kBlockK - 1) / kBlockK;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------ TMA producer ------------------------------------
      const uint64_t pol_w = sm100::policy_evict_first(), pol_h = sm100::policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int t0 = r0; t0 < r1;) {
        const int t1 = tile_end(t0, r1), base = t0 & ~127;
        const bool full_tile = (t0 == base) && (t1 - t0 == kBlockM);
        const int nbox = (t1 - t0 + 15) >> 4;
        const uint32_t bytes = (full_tile ? kWStageBytes : nbox * 16 * kBlockK * 2) + Cfg::kHStageBytes;
        for (int kb = 0; kb < num_kb; ++kb) {
          sm100::mbar_wait(&empty[stage], phase ^ 1);
          sm100::mbar_arrive_expect_tx(&full[stage], bytes);
          uint8_t* wdst = w_ring + (size_t)stage * kWStageBytes;
          if (full_tile) {
            sm100::tma_load_2d(wdst, &tmW128, &full[stage], kb * kBlockK, t0, pol_w);
          } else {
            for (int j = 0; j < nbox; ++j)
              sm100::tma_load_2d(wdst + (t0 - base + 16 * j) * (kBlockK * 2), &tmW16, &full[stage], kb * kBlockK,
                                 t0 + 16 * j, pol_w);
          }
          sm100::tma_load_2d(h_ring + (size_t)stage * Cfg::kHStageBytes, &tmH, &full[stage], kb * kBlockK, 0,
                             pol_h);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        t0 = t1;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------ MMA issuer --------------------------------------
      constexpr uint32_t idesc = sm100::umma_idesc_bf16(kBlockM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int tile_i = 0;
      for (int t0 = r0; t0 < r1; ++tile_i) {
        const int t1 = tile_end(t0, r1);
        const int buf = tile_i & 1;
        const uint32_t use = (uint32_t)(tile_i >> 1);
        sm100::mbar_wait(&tempty[buf], (use & 1) ^ 1);
        sm100::tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(buf * BN);
        for (int kb = 0; kb < num_kb; ++kb) {
          sm100::mbar_wait(&full[stage], phase);
          sm100::tc_fence_after();
          const uint64_t adesc = sm100::umma_desc_sw128(sm100::smem_u32(w_ring + (size_t)stage * kWStageBytes));
          const uint64_t bdesc = sm100::umma_desc_sw128(sm100::smem_u32(h_ring + (size_t)stage * Cfg::kHStageBytes));
#pragma unroll
          for (int k = 0; k < kBlockK / 16; ++k)
            sm100::mma_bf16_ss(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
          sm100::mma_commit(&empty[stage]);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        sm100::mma_commit(&tfull[buf]);
        t0 = t1;
      }
    }
  } else {
    // -------------------------------- epilogue ------------------------------------------
    const int q = warp & 3;                       // TMEM lane quadrant this warp may access
    const int epi_tid = threadIdx.x - 64;
    EpiArgs ea;
    ea.invtau = invtau;
    ea.mask = p.mask;
    ea.mask_words = p.mask_words;
    ea.B = p.B;
    ea.row_offset = p.row_offset;
    ea.k0 = (uint32_t)p.seed;
    ea.k1 = (uint32_t)(p.seed >> 32);
    ea.c2 = ctr_step_lo(p.step);
    ea.c3 = ctr_step_hi(p.step, 0u);
    State st[Cfg::kChunks];
#pragma unroll
    for (int c = 0; c < Cfg::kChunks; ++c) st[c] = state_empty();
    int seg = 0, cur_group = -1, tile_i = 0;
    State* part_cta = p.part + (size_t)blockIdx.x * p.max_seg * p.B;
    for (int t0 = r0; t0 < r1; ++tile_i) {
      const int t1 = tile_end(t0, r1), base = t0 & ~127;
      const int grp = t0 / p.group_size;
      if (cur_group >= 0 && grp != cur_group) {
        flush_states<Cfg::kChunks, Cfg::kColsPerChunk>(st, scratch, BN, q, lane, epi_tid, p.B,
                                                      part_cta + (size_t)seg * p.B, 1);
        if (epi_tid == 0) p.part_group[blockIdx.x * p.max_seg + seg] = cur_group;
        ++seg;
      }
      cur_group = grp;
      const int buf = tile_i & 1;
      const uint32_t use = (uint32_t)(tile_i >> 1);
      sm100::mbar_wait(&tfull[buf], use & 1);
      sm100::tc_fence_after();
      const int row = base + 32 * q + lane;
      RowArgs ra;
      ra.valid = row >= t0 && row < t1;
      ra.v_global = (int32_t)(p.vocab_offset + row);
      ra.v_lo = (uint32_t)ra.v_global;
      ra.warp_v0 = (int32_t)(p.vocab_offset + base + 32 * q);
      ra.bias = (ra.valid && p.bias) ? p.bias[row] : 0.0f;
      const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * BN);
#pragma unroll
      for (int c = 0; c < Cfg::kChunks; ++c) {
        uint32_t r[32];
        if constexpr (Cfg::kColsPerChunk == 32) sm100::tmem_ld_32x32b_x32(taddr + c * 32, r);
        else sm100::tmem_ld_32x32b_x16(taddr, r);
        sm100::tmem_wait_ld();
        if (c == Cfg::kChunks - 1) {
          sm100::tc_fence_before();
          sm100::mbar_arrive(&tempty[buf]);        // accumulator buffer free for tile t+2
        }
        float acc[32];
#pragma unroll
        for (int i = 0; i < Cfg::kColsPerChunk; ++i) acc[i] = __uint_as_float(r[i]);
        epi_columns<Cfg::kColsPerChunk, LSE>(acc, c * Cfg::kColsPerChunk, ra, ea, st[c], lane);
      }
      t0 = t1;
    }
    if (cur_group >= 0) {
      flush_states<Cfg::kChunks, Cfg::kColsPerChunk>(st, scratch, BN, q, lane, epi_tid, p.B,
                                                    part_cta + (size_t)seg * p.B, 1);
      if (epi_tid == 0) p.part_group[blockIdx.x * p.max_seg + seg] = cur_group;
      ++seg;
    }
    if (epi_tid == 0)
      for (int s = seg; s < p.max_seg; ++s) p.part_group[blockIdx.x * p.max_seg + s] = -1;
  }

  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

template <int BN, bool LSE>
static cudaError_t launch_bn(const TcMaps& maps, const StageOneParams& p, int grid, cudaStream_t stream) {
  using Cfg = TcCfg<BN>;
  const int S = p.stages;
  const size_t smem = 1024 + (size_t)S * Cfg::kStageBytes + Cfg::extra_bytes(S);
  auto kern = fused_tc_kernel<BN, LSE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreadsTC, smem, stream>>>(maps.w128, maps.w16, maps.h, p);
  return cudaGetLastError();
}

int tc_block_n(int B) {
  if (B <= 16) return 16;
  if (B <= 32) return 32;
  return ((B + 31) / 32) * 32;
}

int tc_stages(int BN) {
  const int budget = 227 * 1024 - 1024;
  const int stage = kWStageBytes + BN * kBlockK * 2;
  int S = 16;
  while (S > 2 && S * stage + ((2 * S + 4) * 8 + 16 + BN * 4 + 4 * BN * 16 + 64) > budget) --S;
  return S;
}

cudaError_t launch_fused_tc(const TcMaps& maps, const StageOneParams& p, int BN, bool lse, int grid,
                            cudaStream_t stream) {
#define FS_CASE(N)                                                                     \
  case N:                                                                              \
    return lse ? launch_bn<N, true>(maps, p, grid, stream) : launch_bn<N, false>(maps, p, grid, stream);
  switch (BN) {
    FS_CASE(16)
    FS_CASE(32)
    FS_CASE(64)
    FS_CASE(96)
    FS_CASE(128)
    FS_CASE(160)
    FS_CASE(192)
    FS_CASE(224)
    FS_CASE(256)
    default:
      return cudaErrorInvalidValue;
  }
#undef FS_CASE
}

}  // namespace fs
