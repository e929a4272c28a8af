// fs_kernels.h -- internal launch interface between the C ABI (fs_api.cu) and the kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <mutex>
#include <set>
#include <utility>

#include "../../include/flashsample.h"
#include "fs_peer.cuh"

namespace fs {

// Rows per tile of a segment of `len` rows: the fewest tiles of at most `max_rows`, made equal (a
// multiple of `gran`).  A small remainder tile after full ones streams a whole K loop with few bytes
// in flight (V = 151,936 / 148 CTAs = 8.02 tiles: 0.95 -> 1.0 of the copy peak).
// Host (descriptor box rows) and device (tile loops) use this same function.
__host__ __device__ inline int seg_tile_rows(int len, int max_rows, int gran) {
  const int n = (len + max_rows - 1) / max_rows;
  if (n <= 1) return max_rows;
  int t = (len + n - 1) / n;
  t = (t + gran - 1) / gran * gran;
  return t < max_rows ? t : max_rows;
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-(function, device) setting: set it once for
// every device a kernel is launched on (the current device), under a lock (several host threads
// may launch at once).
inline cudaError_t ensure_smem_attr(const void* kern, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  if (done.count({kern, dev})) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({kern, dev});
  return e;
}

struct State;
struct Cand;

// Parameters of one stage-1 launch (one chunk of <= 256 batch rows).
struct StageOneParams {
  const void* h;              // [B, D] (SIMT kernel reads it directly; the TC kernel via TMA)
  const void* W;              // [V, D]
  const float* bias;          // [V] (shard-local) or nullptr
  const float* temperature;   // [B] for this chunk or nullptr
  const uint64_t* seeds;      // [B] per-request seeds for this chunk (reading R18) or nullptr
  const uint64_t* steps;      // [B] per-request steps or nullptr (-> step)
  const uint32_t* mask;       // [B][mask_words] for this chunk (global ids) or nullptr
  int64_t mask_words;
  int64_t vocab_offset;       // global id of local row 0
  uint64_t seed, step;
  int B, D, V;                // V = local rows
  int row_offset;             // global batch index of this chunk's row 0
  int group_size;             // local rows per group (multiple of 128); >= V for one group
  int max_seg;                // candidate slots per CTA
  int stages;                 // TMA ring depth (TC kernel)
  int unit_rows;              // CTA range granularity in rows (TC kernel): 16, 32, 64 or 128
  int kbps;                   // 64-wide K slices per ring stage (TC kernel)
  int dbg_no_mma;             // debug: 1 = stream operands without issuing MMAs; 2 = MMAs on stale smem, no loads
  int dbg_no_epi;             // debug: epilogue drains TMEM without computing
  int w_policy;               // 1: W TMA loads carry an L2 evict_first hint
  int epi_sleep;              // ns backoff while epilogue warps wait for an accumulator
  int bn;                     // MMA N (batch columns, padded) (TC kernel; set by launch_fused_tc)
  int tmem_cols;              // TMEM columns allocated (TC kernel; set by launch_fused_tc)
  const CUtensorMap* wmaps;   // [grid][max_seg] device TMA descriptors of each CTA segment (TC kernel)
  State* part;                // [grid * max_seg][B] candidate states
  int* part_group;            // [grid * max_seg] group id of each slot, -1 = unused
  int mode;                   // 0 sample; 1 top-k candidates (fs_topk_epi.cuh); 2 store raw logits
  int topk_k;                 // mode 1: k
  int topk_cap;               // mode 1: candidate list capacity per column (>= k rounded to 32, + 128)
  Cand* topk_cand;            // mode 1: [B][topk_stride] candidates, appended at topk_rowcnt[b] (atomic)
  int topk_stride;            // mode 1: candidate capacity per row (grid * topk_cap)
  int* topk_rowcnt;           // mode 1: [B] candidates written per row (zero on entry)
  uint32_t* topk_lb;          // mode 1: [B][grid] each CTA's topk_m-th largest key (0 if fewer)
  int topk_m;                 // mode 1: ceil(k / grid)
  float* mat_out;             // mode 2: [B][mat_ld] fp32 logits of the local rows
  int64_t mat_ld;
  uint32_t* topk_gmax;        // mode 2 (optional): [B][gld] per 32-row warp span starting at row 16u:
                              // max order_key(raw logit) at u, 1 at u+1 when the span has > 16 rows
  int64_t topk_gld;           // ceil(V / 16)
  // One-kernel finalize (mode 0, single group, no log-mass): each CTA folds its merged candidate
  // into fin_best[b] by a 64-bit atomicMax of (key << 32 | ~idx); the last CTA to finish (fin_ctr)
  // writes idx_out / score_out and resets both, so no stage-2 launch follows.
  unsigned long long* fin_best;   // [256], all 0 between calls; nullptr = write `part` for stage 2
  int spin_wait;                  // A/B: epilogue waits spin on try_wait without the suspend hint
  fs_summary* fin_sum;            // with fin_best: write {M, I, L = NaN} records instead of idx / score
  unsigned long long* done_flag;  // with fin_best: pinned host word set to 1 after the outputs (option)
  unsigned int* fin_ctr;          // CTAs finished, 0 between calls
  int32_t* idx_out;               // [B] of this chunk
  float* score_out;               // [B] or nullptr
  int fin_lse;                    // single group with log-mass, small B: the last CTA runs stage 2's
                                  // per-row reduce over `part` (counter fin_ctr); outputs below
  float* logZ_out;                // [B] or nullptr
  fs_summary* groups_out;         // [B] (the single group's summary, e.g. a TP shard's) or nullptr
  float* logprob_out;             // [B] or nullptr
  int need_lt;                    // some output of the call reads the winner's l~ (log-prob)
  unsigned long long* dbg_times;  // debug: [grid][8] globaltimer ns (start, dependency wait done, last load
                                  // issued, last tile drained), %smid, CTA done, and the MMA issuer's total
                                  // ns waiting for a drained accumulator / for operands (MMA CTAs); or nullptr
  const void* h_host;             // in-kernel staging (fs_sample_staged): pinned host h copied into h by
                                  // all CTAs after the dependency wait, then a grid barrier (h_bar)
                                  // before the first h load; nullptr = h is already on the device
  unsigned int* h_bar;            // grid-barrier counter (reset by the finalizing CTA)
  int pdl_w;                      // launched with PDL: W loads may precede griddepcontrol.wait;
                                  // everything else (h, bias, tau, mask, seeds, outputs) follows it
  PushCtx push;                   // f2: the finalizing CTA also pushes the shard summaries to every
                                  // peer window and releases the flags (push.peers == nullptr: off)
};


int tc_block_n(int B);
int tc_stages(int BN, int kbps, int extra = 0);
int tc_topk_extra_bytes(int BN, int cap);   // shared memory of the top-k lists (mode 1)
int tc_slots_per_segment();   // candidate slots one CTA writes per group segment
int tc2_stages(int BN, int kbps);
// CTA-pair (cta_group::2) stage 1: grid = 2 x pairs, cluster (2,1,1); h map box = BN/2 rows.
cudaError_t launch_fused_tc2(const CUtensorMap& hmap, const StageOneParams& p, int BN, bool lse, int grid,
                             cudaStream_t stream);
cudaError_t launch_fused_tc(const CUtensorMap& hmap, const StageOneParams& p, int BN, bool lse, int grid,
                            cudaStream_t stream);
// How many CTAs of the stage-1 kernel that launch_fused_tc / launch_fused_tc2 would pick for `p`
// can be resident on the current device at once (occupancy API; the pair kernel counts clusters).
// In-kernel staging (a grid barrier) is only used when the whole grid fits.
cudaError_t fused_tc_resident(const StageOneParams& p, int BN, bool lse, int* ctas);
cudaError_t fused_tc2_resident(const StageOneParams& p, int BN, bool lse, int grid, int* ctas);
// p.mode 1 / 2 of the 1-CTA kernel (top-k candidates / raw logits); xform applies to mode 1.
cudaError_t launch_fused_tc_topk(const CUtensorMap& hmap, const StageOneParams& p, int BN, int grid,
                                 cudaStream_t stream);
// CUDA-core stage 1: grid = ceil(V/128) aligned tiles, one slot per tile.
cudaError_t launch_fused_simt(const StageOneParams& p, fs_dtype dtype, bool lse, cudaStream_t stream);

// Where stage 1 put the candidates of each group (stage 2 needs it to find a group's slots).
struct SlotLayout {
  int n_slots;       // candidate slots written
  int simt;          // 1: CUDA-core layout, slot = 128-row tile; 0: tcgen05 layout
  int G;             // tcgen05: persistent CTAs (cta_rows partition)
  int V;             // local rows
  int max_seg;       // tcgen05 grouped: segments per CTA (slot = (cta*max_seg + seg)*8 + warp)
  int group_size;
  int unit_rows;     // tcgen05: CTA range granularity
  int pair;          // tcgen05: 1 if the partition is over CTA pairs (cta_group::2 kernel)
};

// Stage 2: reduce the candidate slots of every row into groups and the final sample.
cudaError_t launch_reduce(const State* part, const int* part_group, const SlotLayout& lay, int B, int n_groups,
                          int32_t* idx_out, float* score_out, float* logZ_out, fs_summary* groups_out,
                          cudaStream_t stream, bool pdl, float* logprob_out = nullptr,
                          const int* grp_lo = nullptr,    // [n_groups+1] first slot per group (host-computed)
                          State* gscratch = nullptr,      // [B][n_groups] group states (warp-per-group kernel)
                          int* row_ctr = nullptr,         // [B] zeroed counters (warp-per-group kernel)
                          const PushCtx* push = nullptr,  // single group: also push the records (f2)
                          int grp_kernel = 0);            // grouped: 0 auto, 1 warp per (row, group), 3 block per row
// Standalone sampler over materialised logits [B][ld] (bf16 or fp32): candidates per (V-block, row).
cudaError_t launch_logits_sample(fs_dtype dtype, const void* logits, int64_t ld, const float* bias,
                                 const float* temperature, const uint32_t* mask, int64_t mask_words, int B, int V,
                                 uint64_t seed, uint64_t step, bool lse, int nblk, State* part, int* part_group,
                                 cudaStream_t stream, const uint64_t* seeds = nullptr,
                                 const uint64_t* steps = nullptr, unsigned long long* fin_best = nullptr,
                                 unsigned int* fin_ctr = nullptr, int32_t* idx_out = nullptr,
                                 float* score_out = nullptr);
int logits_sample_blocks(int B, int V);   // V blocks of the standalone sampler grid
// Fused top-k raw-logit route with span maxima: per row, threshold = k-th largest span max (raw
// space), gather the logits of the spans at or above it (transform: temperature only) into
// cand[b][0, n_b), n_b -> row_count[b].  Then launch_topk_final (no slot bounds).
cudaError_t launch_topk_gather(const float* mat, int64_t ld, const uint32_t* gmax, int64_t gld,
                               const float* temperature, int B, int V, int k, Cand* cand, int64_t stride,
                               int* row_count, cudaStream_t stream);
// Top-k / top-p over materialised logits: chunk candidates (workspace B*topk_chunks(V)*k*8 bytes)
// then a per-row merge + top-p + Gumbel-max.
int topk_chunks(int V);
int topk_max_k();
// row_offset: global batch index of row 0 (shared-stream RNG counter); the per-row arrays
// (temperature, mask, seeds, steps, outputs) are already offset by the caller.
cudaError_t launch_topk_sample(fs_dtype dtype, const void* logits, int64_t ld, const float* bias,
                               const float* temperature, const uint32_t* mask, int64_t mask_words, int B, int V,
                               int k, float top_p, uint64_t seed, uint64_t step, const uint64_t* seeds,
                               const uint64_t* steps, void* cand_ws, int32_t* idx_out, float* score_out,
                               float* logZ_out, float* logprob_out, cudaStream_t stream, int row_offset = 0);
// Merge stage only: cand [B][ncand] (key, id), n_b = row_count[b] (reset to 0) or ncand; slot_lb
// [B][nslots] = each slot's m-th largest key (pruning bound) -> top-k -> top-p -> Gumbel-max.
cudaError_t launch_topk_final(const Cand* cand, int ncand, int* row_count, int B, int k, float top_p,
                              const float* temperature, uint64_t seed, uint64_t step, const uint64_t* seeds,
                              const uint64_t* steps, int32_t* idx_out, float* score_out, float* logZ_out,
                              float* logprob_out, cudaStream_t stream, int row_offset, bool pdl,
                              const uint32_t* slot_lb, int nslots, int m);
// f2 exchange, unfused form (B > 256): push `local` [B] into every peer window, wait, combine.
cudaError_t launch_exchange_combine(const fs_summary* local, const PeerTab& peers, int world, int rank, int B,
                                    int B_max, uint64_t epoch, int32_t* idx_out, float* score_out, float* logZ_out,
                                    unsigned* timeouts, cudaStream_t stream, bool pdl);
// f2 exchange, fused form: the records were pushed by the shard sampler itself (PushCtx); this
// one-block kernel (PDL) only acquires the n flags of `epoch`, combines and acknowledges.
cudaError_t launch_exchange_wait(const PeerTab* peers_dev, int world, int rank, int B, int B_max, uint64_t epoch,
                                 int32_t* idx_out, float* score_out, float* logZ_out, unsigned* timeouts,
                                 cudaStream_t stream, bool pdl);
cudaError_t launch_combine(const fs_summary* gathered, int n, int B, int32_t* idx_out, float* score_out,
                           float* logZ_out, cudaStream_t stream);
cudaError_t launch_merge(const fs_summary* a, const fs_summary* b, fs_summary* out, int count,
                         cudaStream_t stream);
cudaError_t launch_fused_tc2_raw(const CUtensorMap& hmap, const StageOneParams& p, int BN, int grid,
                                 cudaStream_t stream);
cudaError_t launch_read_probe(const void* src, size_t bytes, unsigned long long* sink, int grid, cudaStream_t stream);
cudaError_t launch_random_bits(uint64_t seed, uint64_t step, uint32_t tag, const int32_t* b, const int64_t* v,
                               uint32_t* r, int64_t n, cudaStream_t stream);
cudaError_t launch_gumbel(const uint32_t* r, float* g, int64_t n, cudaStream_t stream);
// Input staging copy (fs_copy_async): src loads before, dst stores after the PDL dependency wait.
// src_host: pinned host src (loads may precede the wait); device src is read after it.
cudaError_t launch_copy_in(void* dst, const void* src, size_t bytes, bool pdl, bool src_host, cudaStream_t stream);

}  // namespace fs
