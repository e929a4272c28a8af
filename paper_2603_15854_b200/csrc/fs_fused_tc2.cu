// fs_fused_tc2.cu -- stage 1 of FlashSampling on a CTA PAIR (tcgen05 cta_group::2).
//
// Same contract and epilogue as fs_fused_tc.cu, for larger batches.  Two CTAs of a cluster
// (one TPC) compute an M=256 x N=BN x K=16 MMA per instruction: CTA r holds W rows
// [t0 + 128 r, t0 + 128 r + 128) of each 256-row tile (the A operand, split by M) and batch rows
// [r BN/2, (r+1) BN/2) of h (the B operand, split by N); each CTA's TMEM receives its 128 rows
// x all BN columns.  Per W byte a CTA now moves half as many h bytes through its TMA ring and
// shared memory as the 1-CTA kernel (at B=256: 1x instead of 2x the W bytes), which is what
// limits the 1-CTA kernel at B >= 128.
//
// Synchronisation (leader = even CTA, issues all MMAs):
//   full[s]    leader's barrier; both CTAs' 2-SM TMA loads complete_tx on it (peer bit cleared);
//              the leader's producer arms it with the pair's byte count.
//   empty[s]   one per CTA, arrived by the leader's multicast tcgen05.commit.
//   tfull[b]   one per CTA, arrived by the multicast commit after a tile's last MMA.
//   tempty[b]  leader's barrier, 16 arrivals: lane 0 of the 8 epilogue warps of set b in each CTA.
// Epilogue: 16 warps per CTA; set s = buffer s, and the two warps of a TMEM lane quadrant in a
// set split the tile's 32-column chunks (even / odd) -- twice the warps of the 1-CTA kernel, for
// latency hiding at the large batches this kernel serves.
#include <cuda.h>
#include <cuda_runtime.h>

#include "fs_epilogue.cuh"
#include "fs_kernels.h"
#include "fs_topk_epi.cuh"

namespace fs {

namespace {
constexpr int kEpiWarps = 16;                  // 2 sets (TMEM buffers) x 2 column halves x 4 lane quadrants
constexpr int kSlotWarps = 8;                  // candidate slots per (segment, CTA): one per (set, quadrant)
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kBlockK = 64;
constexpr int kWBytes = 128 * kBlockK * 2;                  // this CTA's 128 W rows per K slice
constexpr int kExtraBytes = 64 * 8 + 16 + (int)sizeof(RowTab) + 64;

int tmem_cols_for(int BN) {
  int c = 32;
  while (c < 2 * BN) c <<= 1;
  return c;
}
__device__ __forceinline__ int seg_end2(int a, int r1, int gs) { return min(r1, (a / gs + 1) * gs); }
}  // namespace

// MODE 0: sampling epilogue; MODE 2: raw fp32 logits + per-32-row span maxima for the fused top-k
// raw-logit route (fs_topk.cu gathers the spans at or above the k-th largest), as the 1-CTA kernel's
// mode 2 -- pair tiles are then cut in 32-row units so every CTA half starts on a 16-row span unit.
template <bool LSE, bool XFORM, bool PRQ, int MODE = 0>
__global__ void __launch_bounds__(kThreads, 1)   // 18 warps: <= 96 registers (5 warps on a 16K-register SM sub-partition)
fused_tc2_kernel(const __grid_constant__ CUtensorMap tmH, const StageOneParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base by pointer arithmetic on the shared array, so that every pointer derived
  // from it stays in the shared address space (LDS/STS/ATOMS, not generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = p.stages, BN = p.bn, KBPS = p.kbps;
  constexpr int kGran = MODE == 2 ? 32 : 16;                  // pair tile granularity (rows)
  const int h_bytes = (BN / 2) * kBlockK * 2;                 // this CTA's half of h per K slice
  uint8_t* w_ring = smem;
  uint8_t* h_ring = smem + (size_t)S * KBPS * kWBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(h_ring + (size_t)S * KBPS * h_bytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  RowTab* tab = reinterpret_cast<RowTab*>(tmem_slot + 4);

  const uint32_t rank = sm100::cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const CUtensorMap* wmaps = p.wmaps + (size_t)pair * p.max_seg;
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
      sm100::mbar_init(&tempty[i], 16);
    }
    sm100::fence_barrier_init();
  }
  // The paired allocation (and its release below) is issued by warp 0: issued by any other warp,
  // compute-sanitizer racecheck reports the allocator's result write as a race with the alloc itself
  // (tools/racecheck_tmem_pair.cu: the same prologue is clean with warp 0, flagged with warp 1).
  if (warp == 0) sm100::tmem_alloc_pair(tmem_slot, (uint32_t)p.tmem_cols);
  sm100::tc_fence_before();
  sm100::cluster_sync();                    // both CTAs' barriers exist before any remote signal
  __syncthreads();                          // CTA-level order for the allocator's smem write (racecheck)
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  sm100::pdl_launch_dependents();
  if (warp != 0) {
    // every input but W is read past the dependency wait (the producer defers only its h loads)
    if (p.pdl_w) sm100::pdl_wait();
    if (XFORM) {
      fill_rowtab<PRQ>(tab, p.B, p.temperature, p.seeds, p.steps, p.step, threadIdx.x - 32, kThreads - 32);
      sm100::named_bar_sync(4, kThreads - 32);
    }
    if (p.h_host)
      stage_h_slice(p.h_host, p.h, (size_t)p.B * p.D * 2, threadIdx.x - 32, kThreads - 32, 4, p.h_bar);
  }

  int r0, r1;
  cta_rows(pair, npairs, p.V, p.unit_rows, r0, r1);
  const int num_kb = (p.D + kBlockK - 1) / kBlockK;
  const int gs = p.group_size;

  if (warp == 0) {
    if (lane == 0) {
      // -------------------------- TMA producer (both CTAs) ------------------------------
      const uint64_t pol_w = p.w_policy ? sm100::policy_evict_first() : sm100::policy_evict_normal();
      const uint64_t pol_h = sm100::policy_evict_last();
      // per K slice: both CTAs' Th rows of W (full boxes, OOB-clipped rows counted) + both h halves
      // PDL: W loads of the first S stages before the dependency wait, their h loads after it
      auto load_h = [&](int stg, int kb0, int nk) {
        for (int j = 0; j < nk; ++j)
          sm100::tma_load_2d_pair(h_ring + ((size_t)stg * KBPS + j) * h_bytes, &tmH, &full[stg],
                                  (kb0 + j) * kBlockK, (int)rank * (BN / 2), pol_h);
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
        const int b = seg_end2(a, r1, gs);
        const CUtensorMap* wm = &wmaps[seg];
        const int T2 = seg_tile_rows(b - a, 256, kGran), Th = T2 / 2;   // pair tile, this CTA's half
        const uint32_t pair_tx = 2u * (uint32_t)(Th * kBlockK * 2 + h_bytes);
        for (int t0 = a; t0 < b; t0 += T2) {
          for (int kb0 = 0; kb0 < num_kb; kb0 += KBPS) {
            const int nk = min(KBPS, num_kb - kb0);
            sm100::mbar_wait(&empty[stage], phase ^ 1);
            if (p.dbg_no_mma == 2) {            // debug: MMAs on stale tiles, no loads
              if (rank == 0) sm100::mbar_arrive(&full[stage]);
              if (++stage == S) { stage = 0; phase ^= 1; }
              continue;
            }
            if (rank == 0) sm100::mbar_arrive_expect_tx(&full[stage], pair_tx * nk);
            for (int j = 0; j < nk; ++j)
              sm100::tma_load_2d_pair(w_ring + ((size_t)stage * KBPS + j) * kWBytes, wm, &full[stage],
                                      (kb0 + j) * kBlockK, t0 - a + Th * (int)rank, pol_w);
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
    if (lane == 0 && rank == 0) {
      // -------------------------- MMA issuer (leader only) ------------------------------
      const uint32_t idesc = sm100::umma_idesc_bf16(256, BN);
      int stage = 0;
      uint32_t phase = 0;
      int tile_i = 0;
      uint64_t wait_acc = 0, wait_data = 0;   // debug (dbg_times): ns the MMA issuer waited
      for (int a = r0; a < r1;) {
        const int b = seg_end2(a, r1, gs);
        const int T2 = seg_tile_rows(b - a, 256, kGran);
        for (int t0 = a; t0 < b; t0 += T2, ++tile_i) {
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
                  sm100::umma_desc_sw128(sm100::smem_u32(w_ring + ((size_t)stage * KBPS + j) * kWBytes));
              const uint64_t bdesc =
                  sm100::umma_desc_sw128(sm100::smem_u32(h_ring + ((size_t)stage * KBPS + j) * h_bytes));
#pragma unroll
              for (int k = 0; k < kBlockK / 16; ++k)
                sm100::mma_bf16_ss_pair(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, ((kb0 + j) | k) != 0 ? 1u : 0u);
            }
            sm100::mma_commit_pair(&empty[stage], 0x3);
            if (++stage == S) { stage = 0; phase ^= 1; }
          }
          sm100::mma_commit_pair(&tfull[buf], 0x3);
        }
        a = b;
      }
      if (p.dbg_times) {
        p.dbg_times[blockIdx.x * 8 + 6] = wait_acc;
        p.dbg_times[blockIdx.x * 8 + 7] = wait_data;
      }
    }
  } else if constexpr (MODE == 2) {
    // ------------------------ raw logits + span maxima (both CTAs) ----------------------
    const int e = warp - 2;
    const int set = e >> 3;
    const int half = (e >> 2) & 1;                  // columns 8*half, 8*half + 16, ...
    const int q = warp & 3;
    const uint32_t tempty_leader = sm100::mapa(sm100::smem_u32(&tempty[set]), 0);
    int tile_i = 0;
    for (int a = r0; a < r1;) {
      const int b = seg_end2(a, r1, gs);
      const int T2 = seg_tile_rows(b - a, 256, kGran), Th = T2 / 2;
      for (int t0 = a; t0 < b; t0 += T2, ++tile_i) {
        if ((tile_i & 1) != set) continue;
        const uint32_t use = (uint32_t)(tile_i >> 1);
        sm100::mbar_wait(&tfull[set], use & 1);
        sm100::tc_fence_after();
        const int base = t0 + Th * (int)rank;
        const int hi = min(b, base + Th);
        const int row = base + 32 * q + lane, span0 = base + 32 * q;
        const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(set * BN);
        epi_tile_store(taddr, row < hi, row, p.B, p.mat_out, p.mat_ld, p.topk_gmax, p.topk_gld, span0 >> 4,
                       max(0, min(32, hi - span0)), lane, 8 * half, 16);
        release_tmem(&tempty[set], tempty_leader, lane);
      }
      a = b;
    }
  } else {
    // -------------------------------- epilogue (both CTAs) ------------------------------
    const int e = warp - 2;
    const int set = e >> 3;
    const int half = (e >> 2) & 1;                  // chunks half, half + 2, ...
    const int q = warp & 3;
    const int sw = set * 4 + (e & 3);               // candidate slot of (set, quadrant)
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
    const uint32_t tempty_leader = sm100::mapa(sm100::smem_u32(&tempty[set]), 0);
    State st[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) st[c] = state_empty();
    const int slot0 = pair * p.max_seg;   // slot = ((pair*max_seg + seg)*2 + rank)*8 + sw
    int tile_i = 0, seg = 0;
    for (int a = r0; a < r1; ++seg) {
      const int b = seg_end2(a, r1, gs);
      const int T2 = seg_tile_rows(b - a, 256, kGran), Th = T2 / 2;
      for (int t0 = a; t0 < b; t0 += T2, ++tile_i) {
        if ((tile_i & 1) != set) continue;
        const uint32_t use = (uint32_t)(tile_i >> 1);
        if (p.spin_wait) sm100::mbar_wait_spin(&tfull[set], use & 1);   // A/B only
        else sm100::mbar_wait(&tfull[set], use & 1);
        sm100::tc_fence_after();
        const int base = t0 + Th * (int)rank;
        const int row = base + 32 * q + lane;
        RowArgs ra;
        ra.valid = 32 * q + lane < Th && row < b;
        ra.v_global = (int32_t)(p.vocab_offset + row);
        ra.v_lo = (uint32_t)ra.v_global;
        ra.warp_v0 = (int32_t)(p.vocab_offset + base + 32 * q);
        ra.bias = (XFORM && ra.valid && p.bias) ? p.bias[row] : 0.0f;
        const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(set * BN);
        epi_tile_tc<LSE, XFORM, 1, PRQ>(taddr, ra, ea, st, lane, &tempty[set], tempty_leader, half, 2);
      }
      if (gs < p.V) {
        const int slot = ((slot0 + seg) * 2 + (int)rank) * kSlotWarps + sw;
        flush_warp(st, lane, p.B, p.part + (size_t)slot * p.B, half, 2);
        if (lane == 0) p.part_group[slot] = a / gs;
      }
      a = b;
    }
    if (gs < p.V) {
      // unused segment slots: empty candidates tagged with the last group, so that group ids are
      // non-decreasing over ALL slots (stage 2 finds a group's slots by binary search)
      const int last_group = (r1 > r0 ? r1 - 1 : r0) / gs;
      for (int s = seg; s < p.max_seg; ++s) {
        const int slot = ((slot0 + s) * 2 + (int)rank) * kSlotWarps + sw;
        flush_warp(st, lane, p.B, p.part + (size_t)slot * p.B, half, 2);
        if (lane == 0) p.part_group[slot] = last_group;
      }
    } else {
      // all tiles drained -> this CTA's ring is free (the leader's MMAs no longer read it)
      sm100::named_bar_sync(1, 32 * kEpiWarps);
      if (p.dbg_times && threadIdx.x == 64) p.dbg_times[blockIdx.x * 8 + 3] = sm100::globaltimer();
      State* scratch = reinterpret_cast<State*>(w_ring);        // [8 (set, quadrant)][BN]
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int bb = (half + 2 * c) * 32 + lane;
        if (bb < BN) scratch[sw * BN + bb] = st[c];
      }
      sm100::named_bar_sync(1, 32 * kEpiWarps);
      const int et = threadIdx.x - 64;
      for (int bb = et; bb < p.B; bb += 32 * kEpiWarps) {
        State m = scratch[bb];
#pragma unroll
        for (int w = 1; w < kSlotWarps; ++w) m = state_merge(m, scratch[w * BN + bb]);
        if (p.fin_best) {
          if (m.key != kKeyNone) atomicMax(&p.fin_best[bb], pack_state(m));
        } else {
          p.part[(size_t)blockIdx.x * p.B + bb] = m;
        }
      }
      if (p.fin_best)
        finalize_last_cta(p.fin_best, p.fin_ctr, p.B, p.idx_out, p.score_out, et, 32 * kEpiWarps, 1,
                          reinterpret_cast<volatile int*>(scratch + kSlotWarps * BN), gridDim.x, p.h_bar, p.fin_sum, &p.push,
                          p.done_flag);
      else if (et == 0)
        p.part_group[blockIdx.x] = (r0 < r1) ? 0 : -1;
      if (!p.fin_best && p.fin_lse)
        finalize_lse_last_cta(p.part, p.part_group, p.B, p.fin_ctr, p.idx_out, p.score_out, p.logZ_out,
                              p.groups_out, p.logprob_out, et, 32 * kEpiWarps, 1,
                              reinterpret_cast<volatile int*>(scratch + kSlotWarps * BN), p.push);
      if (p.dbg_times && et == 0) p.dbg_times[blockIdx.x * 8 + 5] = sm100::globaltimer();
    }
  }

  sm100::tc_fence_before();
  sm100::cluster_sync();                    // no remote arrivals / MMAs into our TMEM after this
  if (warp == 0) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc_pair(tmem_base, (uint32_t)p.tmem_cols);
  }
}

int tc2_stages(int BN, int kbps) {
  const int budget = 227 * 1024 - 1024;
  const int stage = (kWBytes + (BN / 2) * kBlockK * 2) * kbps;
  int S = 16;
  while (S > 0 && S * stage + kExtraBytes > budget) --S;
  return S;
}

using Tc2Kern = void (*)(const CUtensorMap, const StageOneParams);

static Tc2Kern pick_tc2_kernel(const StageOneParams& p, bool lse) {
  const bool xform = p.bias || p.temperature || p.mask || p.seeds;
  const bool prq = p.seeds != nullptr;
  return lse ? (prq ? fused_tc2_kernel<true, true, true> : xform ? fused_tc2_kernel<true, true, false> : fused_tc2_kernel<true, false, false>)
             : (prq ? fused_tc2_kernel<false, true, true> : xform ? fused_tc2_kernel<false, true, false> : fused_tc2_kernel<false, false, false>);
}

static cudaLaunchConfig_t tc2_config(const StageOneParams& p, int BN, int grid, cudaStream_t stream,
                                     cudaLaunchAttribute (&attr)[2]) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 1024 + (size_t)p.stages * p.kbps * (kWBytes + (BN / 2) * kBlockK * 2) + kExtraBytes;
  cfg.stream = stream;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = p.pdl_w ? 2 : 1;
  return cfg;
}

cudaError_t launch_fused_tc2_raw(const CUtensorMap& hmap, const StageOneParams& p_in, int BN, int grid,
                                 cudaStream_t stream) {
  StageOneParams p = p_in;
  p.bn = BN;
  p.tmem_cols = tmem_cols_for(BN);
  p.pdl_w = 0;
  auto kern = fused_tc2_kernel<false, false, false, 2>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), 227 * 1024);
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute attr[2];
  cudaLaunchConfig_t cfg = tc2_config(p, BN, grid, stream, attr);
  return cudaLaunchKernelEx(&cfg, kern, hmap, p);
}

cudaError_t fused_tc2_resident(const StageOneParams& p, int BN, bool lse, int grid, int* ctas) {
  Tc2Kern kern = pick_tc2_kernel(p, lse);
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), 227 * 1024);
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute attr[2];
  cudaLaunchConfig_t cfg = tc2_config(p, BN, grid, nullptr, attr);
  cfg.numAttrs = 1;
  int clusters = 0;
  if ((e = cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg)) != cudaSuccess) return e;
  *ctas = 2 * clusters;
  return cudaSuccess;
}

cudaError_t launch_fused_tc2(const CUtensorMap& hmap, const StageOneParams& p_in, int BN, bool lse, int grid,
                             cudaStream_t stream) {
  StageOneParams p = p_in;
  p.bn = BN;
  p.tmem_cols = tmem_cols_for(BN);
  Tc2Kern kern = pick_tc2_kernel(p, lse);
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), 227 * 1024);
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute attr[2];
  cudaLaunchConfig_t cfg = tc2_config(p, BN, grid, stream, attr);
  return cudaLaunchKernelEx(&cfg, kern, hmap, p);
}

}  // namespace fs
