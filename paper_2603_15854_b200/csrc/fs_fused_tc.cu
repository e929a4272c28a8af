// fs_fused_tc.cu -- stage 1 of FlashSampling on sm_100a tensor cores.
//
// Alg. 2 stage 1 as a persistent, warp-specialised, swap-AB tcgen05 GEMM
// whose epilogue samples instead of storing logits:
//   * grid = #SMs persistent CTAs, each owning a balanced contiguous range of vocabulary rows
//     (16-row granularity, fs_epilogue.cuh cta_rows): W is streamed from HBM exactly once.
//     The range is cut at group boundaries into segments; each segment has its own TMA
//     descriptor whose row extent is the segment itself, so every W load is one full 128-row
//     box and the ragged last tile is clipped by TMA out-of-bounds handling (no DRAM traffic,
//     no small boxes -- small boxes cost ~12% of stream bandwidth on B200).
//   * MMA shape M = 128 vocabulary rows (A = W tile, K-major) x N = BN batch rows (B = h tile,
//     K-major, zero-filled past B by TMA) x K = 16, fp32 accumulation in TMEM.
//   * warp 0: TMA producer (W with L2 evict_first, h with evict_last) into an S-stage ring of
//             KBPS 64-wide K slices per stage (128-byte swizzle);
//     warp 1: TMEM allocator + single-thread MMA issuer; two accumulator buffers (2 x BN TMEM
//             columns), tile t goes to buffer t mod 2;
//     warps 2-9: two epilogue warpgroups; group s drains buffer s (tiles s, s+2, ...), one warp
//             per TMEM lane quadrant: tcgen05.ld -> registers -> transform + Philox + Gumbel +
//             warp argmax (fs_epilogue.cuh) -> candidates.  Logits never leave the SM; the
//             only HBM writes are the candidates.
#include <cuda.h>
#include <cuda_runtime.h>

#include "fs_epilogue.cuh"
#include "fs_kernels.h"
#include "fs_topk_epi.cuh"

namespace fs {

constexpr int kEpiWarps = 8;
constexpr int kThreadsTC = 64 + 32 * kEpiWarps;   // 10 warps
constexpr int kBlockM = 128;
constexpr int kBlockK = 64;                       // 64 bf16 = 128 B = one swizzle row
constexpr int kWStageBytes = kBlockM * kBlockK * 2;
constexpr int kExtraBytes = 64 * 8 + 16 + (int)sizeof(RowTab) + 64;   // barriers, tmem slot, row table

static int tmem_cols_for(int BN) {
  int c = 32;
  while (c < 2 * BN) c <<= 1;
  return c;
}

// Segments of a CTA range: [a, b) = intersection of [r0, r1) with one group; tiles are
// [a + 128k, min(b, a + 128(k+1))).
__device__ __forceinline__ int seg_end(int a, int r1, int gs) { return min(r1, (a / gs + 1) * gs); }

// MODE 0: sampling epilogue; 1: top-k candidate lists (fs_topk_epi.cuh); 2: raw fp32 logits.
template <bool LSE, bool XFORM, bool PRQ, int MODE = 0>
__global__ void __launch_bounds__(kThreadsTC, 1)
fused_tc_kernel(const __grid_constant__ CUtensorMap tmH, const StageOneParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base by pointer arithmetic on the shared array, so that every pointer derived
  // from it stays in the shared address space (LDS/STS/ATOMS, not generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = p.stages, BN = p.bn, KBPS = p.kbps;
  const int h_stage_bytes = BN * kBlockK * 2;                 // per 64-wide K slice
  uint8_t* w_ring = smem;
  uint8_t* h_ring = smem + (size_t)S * KBPS * kWStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(h_ring + (size_t)S * KBPS * h_stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  RowTab* tab = reinterpret_cast<RowTab*>(tmem_slot + 4);
  const CUtensorMap* wmaps = p.wmaps + (size_t)blockIdx.x * p.max_seg;
  TopkSmem ts{};
  if (MODE == 1) {
    uint8_t* tk = reinterpret_cast<uint8_t*>(tab + 1);
    ts.thr = reinterpret_cast<uint32_t*>(tk);
    ts.cnt = reinterpret_cast<int*>(ts.thr + BN);
    ts.hist = reinterpret_cast<uint32_t*>(ts.cnt + BN);
    ts.buf = reinterpret_cast<Cand*>(ts.hist + kEpiWarps * 256);
    ts.cap = p.topk_cap;
    ts.k = p.topk_k;
    for (int i = threadIdx.x; i < BN; i += kThreadsTC) {
      ts.thr[i] = kKeyNegInf;                     // only finite l~ enter (R19)
      ts.cnt[i] = 0;
    }
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    if (p.dbg_times) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      p.dbg_times[blockIdx.x * 8 + 0] = sm100::globaltimer();
      p.dbg_times[blockIdx.x * 8 + 4] = smid;
    }
    sm100::prefetch_tmap(&tmH);
    for (int s = 0; s < p.max_seg; ++s) sm100::prefetch_tmap(&wmaps[s]);
    for (int s = 0; s < S; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&tfull[i], 1);
      sm100::mbar_init(&tempty[i], MODE == 1 ? 256 : 128);   // mode 1: both warp quads drain every tile
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc(tmem_slot, (uint32_t)p.tmem_cols);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  sm100::pdl_launch_dependents();
  if (warp != 0) {
    // every input but W is read past the dependency wait (the producer defers only its h loads)
    if (p.pdl_w) sm100::pdl_wait();
    if (XFORM) {
      fill_rowtab<PRQ>(tab, p.B, p.temperature, p.seeds, p.steps, p.step, threadIdx.x - 32, kThreadsTC - 32);
      sm100::named_bar_sync(4, kThreadsTC - 32);
    }
    if (p.h_host)
      stage_h_slice(p.h_host, p.h, (size_t)p.B * p.D * 2, threadIdx.x - 32, kThreadsTC - 32, 4, p.h_bar);
  }

  int r0, r1;
  cta_rows(blockIdx.x, gridDim.x, p.V, p.unit_rows, r0, r1);
  const int num_kb = (p.D + kBlockK - 1) / kBlockK;
  const int gs = p.group_size;
  // tile rows a multiple of 8 (the swizzle atom); 16 in the top-k modes, whose span maxima are
  // indexed by 16-row unit (fs_topk.cu)
  constexpr int kTileGran = MODE == 0 ? 8 : 16;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------ TMA producer ------------------------------------
      const uint64_t pol_w = p.w_policy ? sm100::policy_evict_first() : sm100::policy_evict_normal();
      const uint64_t pol_h = sm100::policy_evict_last();
      // full boxes (OOB-clipped rows still counted): T_seg rows of W + the h tile per K slice
      // PDL: the first S stages' W loads are issued before the dependency wait; their h loads
      // (the stage barrier still expects those bytes) are deferred until it returns.
      auto load_h = [&](int stg, int kb0, int nk) {
        for (int j = 0; j < nk; ++j)
          sm100::tma_load_2d(h_ring + ((size_t)stg * KBPS + j) * h_stage_bytes, &tmH, &full[stg],
                             (kb0 + j) * kBlockK, 0, pol_h);
      };
      int pend[16];
      int npend = 0;
      bool waited = !p.pdl_w && !p.h_host;      // h loads wait for the dependency / the staged h
      auto flush_pending = [&]() {
        sm100::pdl_wait();
        if (p.h_host) wait_h_staged(p.h_bar);
        if (p.dbg_times) p.dbg_times[blockIdx.x * 8 + 1] = sm100::globaltimer();
        waited = true;
        for (int i = 0; i < npend; ++i) load_h(pend[i] & 31, pend[i] >> 8, (pend[i] >> 5) & 7);
        npend = 0;
      };
      int stage = 0;
      uint32_t phase = 0;
      int seg = 0;
      for (int a = r0; a < r1; ++seg) {
        const int b = seg_end(a, r1, gs);
        const CUtensorMap* wm = &wmaps[seg];
        const int T = seg_tile_rows(b - a, kBlockM, kTileGran);
        const uint32_t stage_tx = (uint32_t)(T * kBlockK * 2 + h_stage_bytes);
        for (int t0 = a; t0 < b; t0 += T) {
          for (int kb0 = 0; kb0 < num_kb; kb0 += KBPS) {
            const int nk = min(KBPS, num_kb - kb0);
            sm100::mbar_wait(&empty[stage], phase ^ 1);
            if (p.dbg_no_mma == 2) {            // debug: MMAs on stale tiles, no loads
              sm100::mbar_arrive(&full[stage]);
              if (++stage == S) { stage = 0; phase ^= 1; }
              continue;
            }
            sm100::mbar_arrive_expect_tx(&full[stage], stage_tx * nk);
            for (int j = 0; j < nk; ++j)
              sm100::tma_load_2d(w_ring + ((size_t)stage * KBPS + j) * kWStageBytes, wm, &full[stage],
                                 (kb0 + j) * kBlockK, t0 - a, pol_w);
            if (waited) {
              load_h(stage, kb0, nk);
            } else {
              pend[npend++] = stage | (nk << 5) | (kb0 << 8);
              if (npend == S) flush_pending();
            }
            if (++stage == S) { stage = 0; phase ^= 1; }
          }
        }
        a = b;
      }
      if (!waited) flush_pending();
      if (p.dbg_times) p.dbg_times[blockIdx.x * 8 + 2] = sm100::globaltimer();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------ MMA issuer --------------------------------------
      const uint32_t idesc = sm100::umma_idesc_bf16(kBlockM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int tile_i = 0;
      uint64_t wait_acc = 0, wait_data = 0;   // debug (dbg_times): ns the MMA issuer waited
      for (int a = r0; a < r1;) {
        const int b = seg_end(a, r1, gs);
        const int T = seg_tile_rows(b - a, kBlockM, kTileGran);
        for (int t0 = a; t0 < b; t0 += T, ++tile_i) {
          const int buf = tile_i & 1;
          const uint32_t use = (uint32_t)(tile_i >> 1);
          const uint64_t tw0 = p.dbg_times ? sm100::globaltimer() : 0;
          sm100::mbar_wait(&tempty[buf], (use & 1) ^ 1);
          if (p.dbg_times) wait_acc += sm100::globaltimer() - tw0;   // MMA idle: accumulator not drained
          sm100::tc_fence_after();
          const uint32_t d_tmem = tmem_base + (uint32_t)(buf * BN);
          for (int kb0 = 0; kb0 < num_kb; kb0 += KBPS) {
            const int nk = p.dbg_no_mma == 1 ? 0 : min(KBPS, num_kb - kb0);
            const uint64_t fw0 = p.dbg_times ? sm100::globaltimer() : 0;
            sm100::mbar_wait(&full[stage], phase);
            if (p.dbg_times) wait_data += sm100::globaltimer() - fw0;   // MMA idle: operands not landed
            sm100::tc_fence_after();
            for (int j = 0; j < nk; ++j) {
              const uint64_t adesc =
                  sm100::umma_desc_sw128(sm100::smem_u32(w_ring + ((size_t)stage * KBPS + j) * kWStageBytes));
              const uint64_t bdesc =
                  sm100::umma_desc_sw128(sm100::smem_u32(h_ring + ((size_t)stage * KBPS + j) * h_stage_bytes));
#pragma unroll
              for (int k = 0; k < kBlockK / 16; ++k)
                sm100::mma_bf16_ss(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, ((kb0 + j) | k) != 0 ? 1u : 0u);
            }
            sm100::mma_commit(&empty[stage]);
            if (++stage == S) { stage = 0; phase ^= 1; }
          }
          sm100::mma_commit(&tfull[buf]);
        }
        a = b;
      }
      if (p.dbg_times) {
        p.dbg_times[blockIdx.x * 8 + 6] = wait_acc;
        p.dbg_times[blockIdx.x * 8 + 7] = wait_data;
      }
    }
  } else if constexpr (MODE == 1) {
    // ------------------------- top-k candidate epilogue (f1) ----------------------------
    const int e = warp - 2;
    const int qd = e >> 2, wq = e & 3, q = warp & 3;
    EpiArgs ea{};
    ea.invtau = tab->invtau;
    ea.tab = tab;
    ea.mask = p.mask;
    ea.mask_words = p.mask_words;
    ea.B = p.B;
    uint32_t* hist = ts.hist + e * 256;
    int tile_i = 0;
    for (int a = r0; a < r1;) {
      const int b = seg_end(a, r1, gs);
      const int T = seg_tile_rows(b - a, kBlockM, kTileGran);
      for (int t0 = a; t0 < b; t0 += T, ++tile_i) {
        const int buf = tile_i & 1;
        const uint32_t use = (uint32_t)(tile_i >> 1);
        sm100::mbar_wait(&tfull[buf], use & 1);
        sm100::tc_fence_after();
        const int t1 = min(b, t0 + T);
        const int row = t0 + 32 * q + lane;
        RowArgs ra;
        ra.valid = row < t1;
        ra.v_global = (int32_t)(p.vocab_offset + row);
        ra.v_lo = (uint32_t)ra.v_global;
        ra.warp_v0 = (int32_t)(p.vocab_offset + t0 + 32 * q);
        ra.bias = (XFORM && ra.valid && p.bias) ? p.bias[row] : 0.0f;
        const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * BN);
        if (p.dbg_no_epi == 0) epi_tile_topk<XFORM>(taddr, ra, ea, ts, lane, qd);
        release_tmem(&tempty[buf], 0, lane);
        if (p.dbg_no_epi < 2) {
          sm100::named_bar_sync(2 + qd, 128);
          topk_compact_cols(ts, p.B, qd, wq, ts.cap - kBlockM, hist, lane);   // room for one more tile
          sm100::named_bar_sync(2 + qd, 128);
        }
      }
      a = b;
    }
    topk_write_cols(ts, p.B, qd, wq, lane, p.topk_cand, p.topk_stride, p.topk_rowcnt, p.topk_lb, gridDim.x,
                    blockIdx.x, p.topk_m, hist);
  } else if constexpr (MODE == 2) {
    // ------------------------------ raw logits (fallback) -------------------------------
    const int e = warp - 2;
    const int set = e >> 2;
    const int q = warp & 3;
    int tile_i = 0;
    for (int a = r0; a < r1;) {
      const int b = seg_end(a, r1, gs);
      const int T = seg_tile_rows(b - a, kBlockM, kTileGran);
      for (int t0 = a; t0 < b; t0 += T, ++tile_i) {
        if ((tile_i & 1) != set) continue;
        const uint32_t use = (uint32_t)(tile_i >> 1);
        sm100::mbar_wait(&tfull[set], use & 1);
        sm100::tc_fence_after();
        const int row = t0 + 32 * q + lane;
        const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(set * BN);
        const int span0 = t0 + 32 * q, t1 = min(b, t0 + T);
        epi_tile_store(taddr, row < t1, row, p.B, p.mat_out, p.mat_ld, p.topk_gmax, p.topk_gld, span0 >> 4,
                       max(0, min(32, t1 - span0)), lane);
        release_tmem(&tempty[set], 0, lane);
      }
      a = b;
    }
  } else {
    // -------------------------------- epilogue ------------------------------------------
    const int e = warp - 2;                       // 0..7
    const int set = e >> 2;                       // drains TMEM buffer `set`
    const int q = warp & 3;                       // TMEM lane quadrant this warp may access
    EpiArgs ea;
    ea.invtau = tab->invtau;
    ea.tab = tab;
    ea.mask = p.mask;
    ea.mask_words = p.mask_words;
    ea.B = p.B;
    ea.row_offset = p.row_offset;
    ea.k0 = (uint32_t)p.seed;
    ea.k1 = (uint32_t)(p.seed >> 32);
    ea.c2 = ctr_step_lo(p.step);
    ea.c3 = ctr_step_hi(p.step, 0u);
    ea.dbg_skip = p.dbg_no_epi;
    ea.need_lt = p.need_lt;
    State st[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) st[c] = state_empty();
    const int slot0 = blockIdx.x * p.max_seg;
    int tile_i = 0, seg = 0;
    for (int a = r0; a < r1; ++seg) {
      const int b = seg_end(a, r1, gs);
      const int T = seg_tile_rows(b - a, kBlockM, kTileGran);
      for (int t0 = a; t0 < b; t0 += T, ++tile_i) {
        if ((tile_i & 1) != set) continue;
        const int t1 = min(b, t0 + T);
        const uint32_t use = (uint32_t)(tile_i >> 1);
        if (p.epi_sleep) sm100::mbar_wait_sleep(&tfull[set], use & 1, (uint32_t)p.epi_sleep);
        else if (p.spin_wait) sm100::mbar_wait_spin(&tfull[set], use & 1);   // A/B only
        else sm100::mbar_wait(&tfull[set], use & 1);
        sm100::tc_fence_after();
        const int row = t0 + 32 * q + lane;     // TMEM lane l of this tile = row t0 + l
        RowArgs ra;
        ra.valid = row < t1;
        ra.v_global = (int32_t)(p.vocab_offset + row);
        ra.v_lo = (uint32_t)ra.v_global;
        ra.warp_v0 = (int32_t)(p.vocab_offset + t0 + 32 * q);
        ra.bias = (XFORM && ra.valid && p.bias) ? p.bias[row] : 0.0f;
        const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(set * BN);
        if (p.B <= 8) epi_tile_tc<LSE, XFORM, 1, PRQ>(taddr, ra, ea, st, lane, &tempty[set]);
        else epi_tile_tc<LSE, XFORM, 2, PRQ>(taddr, ra, ea, st, lane, &tempty[set]);
      }
      if (gs < p.V) {                           // grouped: one candidate slot per (segment, warp)
        const int slot = (slot0 + seg) * kEpiWarps + e;
        flush_warp(st, lane, p.B, p.part + (size_t)slot * p.B);
        if (lane == 0) p.part_group[slot] = a / gs;
      }
      a = b;
    }
    if (gs < p.V) {
      // unused segment slots: empty candidates tagged with the last group, so that group ids are
      // non-decreasing over ALL slots (stage 2 finds a group's slots by binary search)
      const int last_group = (r1 > r0 ? r1 - 1 : r0) / gs;
      for (int s = seg; s < p.max_seg; ++s) {
        const int slot = (slot0 + s) * kEpiWarps + e;
        flush_warp(st, lane, p.B, p.part + (size_t)slot * p.B);
        if (lane == 0) p.part_group[slot] = last_group;
      }
    } else {
      // Single group: all tiles are drained, so every MMA has consumed its stage and the TMA
      // ring is free; use it as scratch to merge the 8 warps' candidates into ONE slot per CTA
      // (stage 2 then reads #CTA candidates per row instead of 8 x #CTA).
      sm100::named_bar_sync(1, 32 * kEpiWarps);
      if (p.dbg_times && threadIdx.x == 64) p.dbg_times[blockIdx.x * 8 + 3] = sm100::globaltimer();
      State* scratch = reinterpret_cast<State*>(w_ring);        // [8][BN] <= 32 KB
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int bb = c * 32 + lane;
        if (bb < BN) scratch[e * BN + bb] = st[c];
      }
      sm100::named_bar_sync(1, 32 * kEpiWarps);
      const int et = threadIdx.x - 64;                          // 0..255
      for (int bb = et; bb < p.B; bb += 32 * kEpiWarps) {
        State m = scratch[bb];
#pragma unroll
        for (int w = 1; w < kEpiWarps; ++w) m = state_merge(m, scratch[w * BN + bb]);
        if (p.fin_best) {
          if (m.key != kKeyNone) atomicMax(&p.fin_best[bb], pack_state(m));
        } else {
          p.part[(size_t)blockIdx.x * p.B + bb] = m;            // compact: slot = CTA
        }
      }
      if (p.fin_best)
        finalize_last_cta(p.fin_best, p.fin_ctr, p.B, p.idx_out, p.score_out, et, 32 * kEpiWarps, 1,
                          reinterpret_cast<volatile int*>(scratch + kEpiWarps * BN), gridDim.x, p.h_bar, p.fin_sum, &p.push,
                          p.done_flag);
      else if (et == 0)
        p.part_group[blockIdx.x] = (r0 < r1) ? 0 : -1;
      if (!p.fin_best && p.fin_lse)
        finalize_lse_last_cta(p.part, p.part_group, p.B, p.fin_ctr, p.idx_out, p.score_out, p.logZ_out,
                              p.groups_out, p.logprob_out, et, 32 * kEpiWarps, 1,
                              reinterpret_cast<volatile int*>(scratch + kEpiWarps * BN), p.push);
      if (p.dbg_times && et == 0) p.dbg_times[blockIdx.x * 8 + 5] = sm100::globaltimer();
    }
  }

  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem_base, (uint32_t)p.tmem_cols);
  }
}

int tc_block_n(int B) {
  if (B <= 16) return 16;
  if (B <= 32) return 32;
  return ((B + 31) / 32) * 32;
}

int tc_stages(int BN, int kbps, int extra) {
  const int budget = 227 * 1024 - 1024;
  const int stage = (kWStageBytes + BN * kBlockK * 2) * kbps;
  int S = 16;
  while (S > 0 && S * stage + kExtraBytes + extra > budget) --S;
  return S;
}

int tc_topk_extra_bytes(int BN, int cap) {
  return 2 * BN * 4 + kEpiWarps * 256 * 4 + BN * cap * (int)sizeof(Cand) + 16;
}

int tc_slots_per_segment() { return kEpiWarps; }

cudaError_t launch_fused_tc_topk(const CUtensorMap& hmap, const StageOneParams& p_in, int BN, int grid,
                                 cudaStream_t stream) {
  StageOneParams p = p_in;
  p.bn = BN;
  p.tmem_cols = tmem_cols_for(BN);
  const int extra = p.mode == 1 ? tc_topk_extra_bytes(BN, p.topk_cap) : 0;
  const size_t smem = 1024 + (size_t)p.stages * p.kbps * (kWStageBytes + BN * kBlockK * 2) + kExtraBytes + extra;
  const bool xform = p.bias || p.temperature || p.mask;
  auto kern = p.mode == 2 ? fused_tc_kernel<false, false, false, 2>
                          : xform ? fused_tc_kernel<false, true, false, 1> : fused_tc_kernel<false, false, false, 1>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), 227 * 1024);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreadsTC, smem, stream>>>(hmap, p);
  return cudaGetLastError();
}

using TcKern = void (*)(const CUtensorMap, const StageOneParams);

static TcKern pick_tc_kernel(const StageOneParams& p, bool lse) {
  const bool xform = p.bias || p.temperature || p.mask || p.seeds;
  const bool prq = p.seeds != nullptr;
  return lse ? (prq ? fused_tc_kernel<true, true, true> : xform ? fused_tc_kernel<true, true, false> : fused_tc_kernel<true, false, false>)
             : (prq ? fused_tc_kernel<false, true, true> : xform ? fused_tc_kernel<false, true, false> : fused_tc_kernel<false, false, false>);
}

static size_t tc_smem_bytes(const StageOneParams& p, int BN) {
  return 1024 + (size_t)p.stages * p.kbps * (kWStageBytes + BN * kBlockK * 2) + kExtraBytes;
}

cudaError_t fused_tc_resident(const StageOneParams& p, int BN, bool lse, int* ctas) {
  TcKern kern = pick_tc_kernel(p, lse);
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), 227 * 1024);
  if (e != cudaSuccess) return e;
  int per_sm = 0, dev = 0, sms = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreadsTC, tc_smem_bytes(p, BN))) != cudaSuccess)
    return e;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  *ctas = per_sm * sms;
  return cudaSuccess;
}

cudaError_t launch_fused_tc(const CUtensorMap& hmap, const StageOneParams& p_in, int BN, bool lse, int grid,
                            cudaStream_t stream) {
  StageOneParams p = p_in;
  p.bn = BN;
  p.tmem_cols = tmem_cols_for(BN);
  TcKern kern = pick_tc_kernel(p, lse);
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), 227 * 1024);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreadsTC);
  cfg.dynamicSmemBytes = tc_smem_bytes(p, BN);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = p.pdl_w ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, hmap, p);
}

}  // namespace fs
