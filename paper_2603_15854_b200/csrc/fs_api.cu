// fs_api.cu -- the C ABI declared in include/flashsample.h: argument validation, workspace,
// TMA descriptors, kernel selection and the stage-1 / stage-2 launch sequence.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/flashsample.h"
#include "fs_device.cuh"
#include "fs_kernels.h"
#include "fs_nccl.h"

#define FS_VERSION_STRING "flashsample-b200 0.1.0 (sm_100a)"

// Appended to allocation failures: the first call for a shape on a context allocates its workspace,
// so under CUDA graph capture that call must have been made once before, on the same stream.
static const char* const kAllocHint = " (first call of this shape on this context inside CUDA graph capture? call it once outside capture on the same stream)";

namespace {

thread_local std::string g_last_error;

fs_status fail(fs_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}
fs_status cuda_fail(cudaError_t e, const char* where) {
  return fail(FS_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace

struct fs_ctx {
  // Host-side state (workspace pointers, descriptor / layout caches, counters) is guarded by this
  // lock, so concurrent calls from several host threads cannot corrupt it.  The device workspace
  // itself is still one per context: calls on one context must be stream-ordered (header).
  std::recursive_mutex mu;
  int device = 0;
  int num_sms = 0;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  int force_simt = 0;
  int max_ctas = 0;
  int pdl = 1;
  int stages_override = 0;
  int kbps = 0;                    // 0 = default
  int dbg_no_mma = 0;
  int dbg_no_epi = 0;
  int l2promo = 3;                 // CUtensorMapL2promotion for W/h maps (3 = 256B)
  int w_policy = 1;                // 1: W loads evict_first, 0: no cache hint
  unsigned long long* done_flag = nullptr;   // pinned host word the one-kernel finalize sets to 1 (option)
  int grp_kernel = 0;              // grouped stage 2: 0 auto, 1 warp per (row, group), 3 block per row (A/B)
  int spin_wait = 0;               // A/B: epilogue barrier waits without the suspend-time hint
  int epi_sleep = 0;               // ns of backoff in epilogue barrier waits (0 = spin)
  int unit_rows = 0;               // CTA range granularity (0 = default)
  int pair = -1;                   // CTA-pair kernel: -1 auto (by batch size), 0 off, 1 on
  int pair_min_bn = 32;            // auto: use the pair kernel from this MMA N upwards (measured)
  int topk_mode = 0;               // fused top-k: 0 auto, 1 candidate lists in the epilogue, 2 via raw logits
  int topk_spans = 1;
  int* grp_rowcnt = nullptr;       // [256] per-row counters of the warp-per-group stage 2 (kept at 0)
  void* gscratch = nullptr;        // [B][n_groups] group states of the warp-per-group stage 2
  size_t gscratch_bytes = 0;
  int grp_ranges = 1;              // grouped stage 2: host-computed group slot ranges (0 = device binary search)              // raw-logit route: span maxima + gather (1) or full chunk selection (0)
  int* topk_rowcnt = nullptr;      // [256] per-row candidate counters of the list route (kept at 0 between calls)
  int fuse_reduce = 1;             // single-group sampling without log-mass: last CTA finalizes (no stage 2)
  int whole_tiles = 1;             // single-group tensor-core calls: whole-tile CTA ranges on the fewest CTAs
                                   // that keep the pass count (0 = 16-row ranges; DESIGN.md §11 entry 29)
  int pdl_w = 0;                   // stage 1 launched with PDL, W streamed before the dependency wait
                                   // (1: for batch chunks <= pdl_w_max_b rows, 2: always)
  int pdl_w_max_b = 128;
  unsigned long long* dbg_times = nullptr;   // debug: per-CTA timeline of the fused kernels (tools/exp_times.py)
  unsigned long long* fin_buf = nullptr;   // [256] row maxima + CTA counter + staging words (ensure_fin)
  uint64_t staged_fallbacks = 0;           // fs_sample_staged calls staged by the copy kernel instead
  int staging_check = 1;                   // testing: 0 skips the co-residency check of in-kernel staging
  struct ResKey { int pair, bn, stages, kbps, xform, grid; };
  std::vector<std::pair<ResKey, int>> res_cache;   // co-resident CTAs of a stage-1 configuration
  // f2 peer-memory exchange (fs_comm_window_*)
  char* comm_win = nullptr;        // this rank's window (cudaMalloc, exported by IPC)
  size_t comm_off_flags = 0, comm_off_acks = 0, comm_off_status = 0;
  int comm_world = 0, comm_rank = 0, comm_bmax = 0;
  char* comm_peer[fs::kMaxWorld] = {};
  bool comm_open = false;
  fs_summary* comm_local = nullptr;   // [B_max] this rank's shard summaries
  uint64_t comm_epoch = 0;
  fs::PeerTab* comm_peertab = nullptr;  // device copy of the peers' window addresses (fused push)
  // NCCL communicator of fs_comm_init / fs_sample_tp
  ncclComm_t nccl = nullptr;
  int nccl_world = 0, nccl_rank = 0;
  fs_summary* tp_buf = nullptr;       // [1 + world][tp_bmax]: local summaries, then the gathered ones
  int tp_bmax = 0;
  // tensor-map cache: encoding costs host microseconds per map; W maps are reused across calls
  struct MapKey { const void* base; int64_t inner, rows; int box, promo; };
  struct MapEnt { MapKey k; CUtensorMap m; };
  std::vector<MapEnt> map_cache;
  // per-(CTA, segment) W descriptors in device memory (fs_fused_tc.cu), cached per layout
  struct SegKey { const void* W; int64_t D; int V, G, unit, gs, promo, pair, gran; };
  struct SegEnt { SegKey k; CUtensorMap* dev; int max_seg; };
  std::vector<SegEnt> seg_cache;
  // grouped stage 2: first candidate slot of every group ([n_groups + 1], device), per slot layout
  struct GrpKey { int n_slots, simt, G, V, max_seg, gs, unit, pair; };
  struct GrpEnt { GrpKey k; int* dev; };
  std::vector<GrpEnt> grp_cache;
  int time_stage1 = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool;   // created lazily
  size_t ev_used = 0;
  PFN_encodeTiled encode = nullptr;
};

namespace {

fs_status ensure_ws(fs_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->ws_bytes) return FS_OK;
  if (ctx->ws) cudaFree(ctx->ws);
  ctx->ws = nullptr;
  ctx->ws_bytes = 0;
  size_t want = std::max(bytes, (size_t)1 << 20);
  cudaError_t e = cudaMalloc(&ctx->ws, want);
  if (e != cudaSuccess) return fail(FS_ERR_OOM, std::string("workspace cudaMalloc: ") + cudaGetErrorString(e));
  ctx->ws_bytes = want;
  return FS_OK;
}

// Group slot ranges of a stage-1 slot layout (grouped stage 2): mirrors the part_group ids the
// kernels write -- tcgen05: slot ((cta*max_seg + seg)*8 + warp) (pair: ((pair*max_seg + seg)*2 +
// rank)*8 + warp) holds group a/gs of its segment, unused segments the CTA's last group; CUDA-core:
// slot = 128-row tile.  Ids are non-decreasing, so lo[k] = first slot with id >= k.
fs_status group_ranges(fs_ctx* ctx, const fs::SlotLayout& L, int n_groups, const int** out) {
  for (const auto& e : ctx->grp_cache)
    if (e.k.n_slots == L.n_slots && e.k.simt == L.simt && e.k.G == L.G && e.k.V == L.V && e.k.max_seg == L.max_seg &&
        e.k.gs == L.group_size && e.k.unit == L.unit_rows && e.k.pair == L.pair) {
      *out = e.dev;
      return FS_OK;
    }
  std::vector<int> grp((size_t)L.n_slots, 0);
  const int gs = L.group_size;
  if (L.simt) {
    for (int t = 0; t < L.n_slots; ++t) grp[t] = (t * 128) / gs;
  } else {
    const int units = L.pair ? L.G / 2 : L.G;
    const int64_t U = (L.V + L.unit_rows - 1) / L.unit_rows;
    for (int c = 0; c < units; ++c) {
      const int r0 = (int)(L.unit_rows * ((int64_t)c * U / units));
      const int r1 = (int)std::min<int64_t>(L.unit_rows * ((int64_t)(c + 1) * U / units), L.V);
      int seg = 0;
      auto put = [&](int sg, int g) {
        for (int rk = 0; rk < (L.pair ? 2 : 1); ++rk)
          for (int w = 0; w < 8; ++w) {
            const int64_t slot = L.pair ? (((int64_t)c * L.max_seg + sg) * 2 + rk) * 8 + w
                                        : ((int64_t)c * L.max_seg + sg) * 8 + w;
            if (slot < L.n_slots) grp[slot] = g;
          }
      };
      for (int a = r0; a < r1; ++seg) {
        const int b = std::min(r1, (a / gs + 1) * gs);
        put(seg, a / gs);
        a = b;
      }
      const int last = (r1 > r0 ? r1 - 1 : r0) / gs;
      for (; seg < L.max_seg; ++seg) put(seg, last);
    }
  }
  std::vector<int> lo((size_t)n_groups + 1);
  for (int k = 0; k <= n_groups; ++k)
    lo[k] = (int)(std::lower_bound(grp.begin(), grp.end(), k) - grp.begin());
  int* dev = nullptr;
  cudaError_t e = cudaMalloc(&dev, lo.size() * sizeof(int));
  if (e != cudaSuccess) return fail(FS_ERR_OOM, std::string("group range cudaMalloc failed: ") + cudaGetErrorString(e) + kAllocHint);
  e = cudaMemcpy(dev, lo.data(), lo.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "group range copy");
  if (ctx->grp_cache.size() >= 16) {
    cudaFree(ctx->grp_cache.front().dev);
    ctx->grp_cache.erase(ctx->grp_cache.begin());
  }
  ctx->grp_cache.push_back({{L.n_slots, L.simt, L.G, L.V, L.max_seg, gs, L.unit_rows, L.pair}, dev});
  *out = dev;
  return FS_OK;
}

// One-kernel finalize buffer: [256] row maxima, [256] CTA counter, [257] staging barrier (u32) +
// staging-timeout flag (u32), [258] staging-timeout count; zeroed once, left zeroed by every call
// (except the count).
constexpr int kFinWords = 260;
fs_status ensure_fin(fs_ctx* ctx) {
  if (ctx->fin_buf) return FS_OK;
  cudaError_t e = cudaMalloc(&ctx->fin_buf, kFinWords * sizeof(unsigned long long));
  if (e != cudaSuccess) return fail(FS_ERR_OOM, std::string("finalize buffer cudaMalloc failed: ") + cudaGetErrorString(e) + kAllocHint);
  e = cudaMemset(ctx->fin_buf, 0, kFinWords * sizeof(unsigned long long));
  if (e != cudaSuccess) return cuda_fail(e, "finalize buffer memset");
  return FS_OK;
}

fs_status make_map(fs_ctx* ctx, CUtensorMap* m, const void* base, int64_t inner, int64_t rows, int box_rows) {
  for (const auto& e : ctx->map_cache)
    if (e.k.base == base && e.k.inner == inner && e.k.rows == rows && e.k.box == box_rows &&
        e.k.promo == ctx->l2promo) {
      *m = e.m;
      return FS_OK;
    }
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)inner * 2};
  const cuuint32_t box[2] = {64u, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1u, 1u};
  CUresult r = ctx->encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           (CUtensorMapL2promotion)ctx->l2promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FS_ERR_INVALID, "cuTensorMapEncodeTiled failed (code " + std::to_string((int)r) + ")");
  if (ctx->map_cache.size() >= 64) ctx->map_cache.erase(ctx->map_cache.begin());
  ctx->map_cache.push_back(fs_ctx::MapEnt{fs_ctx::MapKey{base, inner, rows, box_rows, ctx->l2promo}, *m});
  return FS_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Host copy of the device partition (fs_epilogue.cuh cta_rows) -- must match it exactly.
void host_cta_rows(int cta, int G, int V, int unit, int& r0, int& r1) {
  const int64_t U = (V + unit - 1) / unit;
  r0 = (int)(unit * ((int64_t)cta * U / G));
  const int64_t e = unit * ((int64_t)(cta + 1) * U / G);
  r1 = (int)(e < (int64_t)V ? e : (int64_t)V);
}

// Box rows per segment = the kernel's tile rows (fs::seg_tile_rows): the 1-CTA kernel's tiles, or
// this CTA's half of the CTA-pair tile (pair = 1).
fs_status segment_maps(fs_ctx* ctx, const void* W, int64_t D, int V, int G, int unit, int gs,
                       const CUtensorMap** out, int* max_seg_out, int pair = 0, int gran = 8) {
  for (const auto& e : ctx->seg_cache)
    if (e.k.W == W && e.k.D == D && e.k.V == V && e.k.G == G && e.k.unit == unit && e.k.gs == gs &&
        e.k.promo == ctx->l2promo && e.k.pair == pair && e.k.gran == gran) {
      *out = e.dev;
      *max_seg_out = e.max_seg;
      return FS_OK;
    }
  int max_seg = 1;
  for (int c = 0; c < G; ++c) {
    int r0, r1, n = 0;
    host_cta_rows(c, G, V, unit, r0, r1);
    for (int a = r0; a < r1; a = std::min(r1, (a / gs + 1) * gs)) ++n;
    max_seg = std::max(max_seg, n);
  }
  std::vector<CUtensorMap> maps((size_t)G * max_seg);
  std::memset(maps.data(), 0, maps.size() * sizeof(CUtensorMap));
  for (int c = 0; c < G; ++c) {
    int r0, r1, s = 0;
    host_cta_rows(c, G, V, unit, r0, r1);
    for (int a = r0; a < r1; ++s) {
      const int b = std::min(r1, (a / gs + 1) * gs);
      const cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)(b - a)};
      const cuuint64_t strides[1] = {(cuuint64_t)D * 2};
      const int T = pair ? fs::seg_tile_rows(b - a, 256, std::max(16, gran)) / 2 : fs::seg_tile_rows(b - a, 128, gran);
      const cuuint32_t box[2] = {64u, (cuuint32_t)T};
      const cuuint32_t estr[2] = {1u, 1u};
      CUresult r = ctx->encode(&maps[(size_t)c * max_seg + s], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                               const_cast<char*>(static_cast<const char*>(W)) + (size_t)a * D * 2, dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               (CUtensorMapL2promotion)ctx->l2promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return fail(FS_ERR_INVALID, "cuTensorMapEncodeTiled (segment) failed");
      a = b;
    }
  }
  if (ctx->seg_cache.size() >= 16) {
    cudaFree(ctx->seg_cache.front().dev);
    ctx->seg_cache.erase(ctx->seg_cache.begin());
  }
  CUtensorMap* dev = nullptr;
  cudaError_t e = cudaMalloc(&dev, maps.size() * sizeof(CUtensorMap));
  if (e != cudaSuccess) return fail(FS_ERR_OOM, std::string("descriptor cudaMalloc failed: ") + cudaGetErrorString(e) + kAllocHint);
  e = cudaMemcpy(dev, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "descriptor upload");
  ctx->seg_cache.push_back(fs_ctx::SegEnt{fs_ctx::SegKey{W, D, V, G, unit, gs, ctx->l2promo, pair, gran}, dev, max_seg});
  *out = dev;
  *max_seg_out = max_seg;
  return FS_OK;
}

struct PathArgs {
  fs_dtype dtype;
  const void* h;
  const void* W;
  const float* bias;
  const float* temperature;
  const uint32_t* mask;
  int64_t mask_words;
  uint64_t seed, step;
  int B, D, V;
  int64_t vocab_offset;
  int group_size;     // local rows per group; >= V means one group
  bool lse;
  int32_t* idx_out;
  float* score_out;
  float* logZ_out;
  fs_summary* groups_out;
  int n_groups;
  float* logprob_out;
  const uint64_t* seeds = nullptr;
  const uint64_t* steps = nullptr;
  const void* h_host = nullptr;   // fs_sample_staged: pinned host h, staged into h by the kernel
  const fs::PushCtx* push = nullptr;   // f2: the shard's summaries also go to the peer windows (B <= 256)
  fs_summary* sum_out = nullptr;       // shard without log-mass: one-kernel finalize writes {M, I, NaN}
};

// time_stage1 option: record a start event now and return the end event to record after stage 1.
fs_status stage1_event(fs_ctx* ctx, cudaStream_t stream, cudaEvent_t* ev_end) {
  *ev_end = nullptr;
  if (!ctx->time_stage1) return FS_OK;
  if (ctx->ev_used == ctx->ev_pool.size()) {
    cudaEvent_t e0, e1;
    if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess)
      return fail(FS_ERR_CUDA, "cudaEventCreate");
    ctx->ev_pool.emplace_back(e0, e1);
  }
  cudaEventRecord(ctx->ev_pool[ctx->ev_used].first, stream);
  *ev_end = ctx->ev_pool[ctx->ev_used].second;
  ++ctx->ev_used;
  return FS_OK;
}

fs_status run_path(fs_ctx* ctx, const PathArgs& a, cudaStream_t stream) {
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  const bool tc = !ctx->force_simt && a.dtype == FS_BF16 && (a.D % 8 == 0) && aligned16(a.h) && aligned16(a.W);
  if (a.sum_out && !(tc && ctx->fuse_reduce)) {   // no one-kernel finalize here: the log-mass shard path
    PathArgs b = a;
    b.lse = true;
    b.groups_out = a.sum_out;
    b.sum_out = nullptr;
    return run_path(ctx, b, stream);
  }
  const size_t esz = a.dtype == FS_BF16 ? 2 : 4;
  const int BN_first = fs::tc_block_n(std::min(a.B, 256));
  const bool pair = tc && (ctx->pair == 1 || (ctx->pair < 0 && BN_first >= ctx->pair_min_bn)) &&
                    (ctx->max_ctas > 0 ? ctx->max_ctas : ctx->num_sms) >= 2;
  // CTA range granularity: 16 rows, except grouped calls on the tensor-core kernels, which cut
  // ranges in whole tiles (128 rows, 256 per CTA pair): group sizes are multiples of 128, so every
  // segment is then whole tiles -- with 16-row ranges almost every CTA straddles a group boundary
  // and pays one extra, partial tile pass (Gemma-3-27B: 15 instead of 14 passes, §11 entry 28)
  int unit = ctx->unit_rows > 0 ? ctx->unit_rows
                                : (tc && a.group_size < a.V && a.group_size % 256 == 0) ? (pair ? 256 : 128) : 16;
  const int U = (a.V + unit - 1) / unit;
  // persistent grid: #SMs CTAs (or #SMs/2 pairs), never more work units than rows allow
  int units = std::min(std::max(1, (ctx->max_ctas > 0 ? ctx->max_ctas : ctx->num_sms) / (pair ? 2 : 1)), U);
  if (ctx->whole_tiles && tc && ctx->max_ctas <= 0 && ctx->unit_rows <= 0 && a.group_size >= a.V) {
    // whole-tile ranges: P = ceil(tiles / units) tile passes are unavoidable; the fewest CTAs (pairs)
    // that still need only P passes get P or P-1 full tiles each (V = 152,064: 132 CTAs x 9 tiles
    // instead of 148 CTAs, some with 9 passes of 116 rows)
    const int tile = pair ? 256 : 128;
    const int tiles = (a.V + tile - 1) / tile;
    const int P = (tiles + units - 1) / units;
    units = (tiles + P - 1) / P;
    unit = tile;
  }
  const int G = units * (pair ? 2 : 1);
  int max_seg = 1, n_slots;
  const CUtensorMap* wmaps = nullptr;
  if (tc) {
    fs_status st0 = segment_maps(ctx, a.W, a.D, a.V, units, unit, std::min(a.group_size, a.V), &wmaps, &max_seg,
                                 pair ? 1 : 0);
    if (st0 != FS_OK) return st0;
    n_slots = (a.group_size >= a.V) ? G : G * max_seg * fs::tc_slots_per_segment();
  } else {
    n_slots = (a.V + 127) / 128;
  }
  const fs::SlotLayout lay{n_slots, tc ? 0 : 1, G, a.V, max_seg, a.group_size, unit, pair ? 1 : 0};
  // one-kernel finalize: the last stage-1 CTA reduces the per-CTA candidates (fs_epilogue.cuh
  // finalize_last_cta) -- single group, no log-mass outputs
  const bool fin = tc && ctx->fuse_reduce && !a.lse && a.group_size >= a.V && (a.idx_out != nullptr || a.sum_out);
  // with log-mass outputs: the last CTA runs the per-row reduce itself (one warp per row; for small
  // B, where a second kernel's launch + grid hop cost more than the serial rows)
  const bool fin_lse = tc && ctx->fuse_reduce && a.lse && a.group_size >= a.V && a.B <= 16;   // measured crossover
  if (fin || fin_lse) {
    fs_status s0 = ensure_fin(ctx);
    if (s0 != FS_OK) return s0;
  }
  const int chunk = 256;
  const int Bc_max = std::min(a.B, chunk);
  const size_t part_bytes = (size_t)n_slots * Bc_max * sizeof(fs::State);
  const size_t grp_off = (part_bytes + 255) & ~size_t(255);
  fs_status st = ensure_ws(ctx, grp_off + (size_t)n_slots * sizeof(int));
  if (st != FS_OK) return st;
  fs::State* part = static_cast<fs::State*>(ctx->ws);
  int* part_group = reinterpret_cast<int*>(static_cast<char*>(ctx->ws) + grp_off);

  for (int r0 = 0; r0 < a.B; r0 += chunk) {
    const int Bc = std::min(chunk, a.B - r0);
    fs::StageOneParams p{};
    p.h = static_cast<const char*>(a.h) + (size_t)r0 * a.D * esz;
    p.W = a.W;
    p.bias = a.bias;
    p.temperature = a.temperature ? a.temperature + r0 : nullptr;
    p.seeds = a.seeds ? a.seeds + r0 : nullptr;
    p.steps = a.steps ? a.steps + r0 : nullptr;
    p.mask = a.mask ? a.mask + (size_t)r0 * a.mask_words : nullptr;
    p.mask_words = a.mask_words;
    p.vocab_offset = a.vocab_offset;
    p.seed = a.seed;
    p.step = a.step;
    p.B = Bc;
    p.D = a.D;
    p.V = a.V;
    p.row_offset = r0;
    p.group_size = a.group_size;
    p.max_seg = max_seg;
    p.unit_rows = unit;
    p.part = part;
    p.part_group = part_group;
    if (a.push) p.push = *a.push;
    cudaEvent_t ev_end = nullptr;
    if ((st = stage1_event(ctx, stream, &ev_end)) != FS_OK) return st;
    if (tc) {
      const int BN = fs::tc_block_n(Bc);
      // K slices per TMA stage: as many as keep >= 3 stages in flight (more contiguous bytes per
      // W row per request; measured on B200).
      p.dbg_no_mma = ctx->dbg_no_mma;
      p.dbg_no_epi = ctx->dbg_no_epi;
      p.dbg_times = ctx->dbg_times;
      p.need_lt = a.logprob_out != nullptr;
      p.w_policy = ctx->w_policy;
      p.epi_sleep = ctx->epi_sleep;
      p.spin_wait = ctx->spin_wait;
      auto stages_for = [&](int k) { return pair ? fs::tc2_stages(BN, k) : fs::tc_stages(BN, k); };
      p.kbps = ctx->kbps;
      if (p.kbps <= 0) {
        p.kbps = 1;
        for (int k = 4; k >= 2; --k)
          if (stages_for(k) >= 3) { p.kbps = k; break; }
      }
      p.stages = ctx->stages_override > 0 ? ctx->stages_override : stages_for(p.kbps);
      if (p.stages < 2) return fail(FS_ERR_INVALID, "K slices per stage too large for shared memory");
      CUtensorMap hmap;
      if ((st = make_map(ctx, &hmap, p.h, a.D, Bc, pair ? BN / 2 : BN)) != FS_OK) return st;
      p.wmaps = wmaps;
      // PDL across steps: worth it while the step is bandwidth-bound; once it is tensor/power-bound
      // (B > pdl_w_max_b, measured: B=256 loops ran 3-15% slower than isolated calls) the overlap of
      // two steps' W streams only competes for the power budget
      p.pdl_w = (ctx->pdl_w >= 2 || (ctx->pdl_w == 1 && Bc <= ctx->pdl_w_max_b)) && ctx->pdl && !ctx->time_stage1;
      if (fin) {
        p.fin_best = ctx->fin_buf;
        p.fin_ctr = reinterpret_cast<unsigned int*>(ctx->fin_buf + 256);
        p.idx_out = a.idx_out ? a.idx_out + r0 : nullptr;
        p.fin_sum = a.sum_out ? a.sum_out + r0 : nullptr;
        if (r0 + chunk >= a.B) p.done_flag = ctx->done_flag;   // the call's last launch
        p.score_out = a.score_out ? a.score_out + r0 : nullptr;
        if (a.h_host) {
          const void* hsrc = static_cast<const char*>(a.h_host) + (size_t)r0 * a.D * esz;
          // the staging grid barrier needs every CTA resident at once: check the occupancy of the
          // exact kernel; otherwise stage with the copy kernel (same results, one more launch)
          const int xform = (p.bias || p.temperature || p.mask) ? 1 : 0;
          const fs_ctx::ResKey rk{pair ? 1 : 0, BN, p.stages, p.kbps, xform, G};
          int resident = -1;
          for (const auto& r : ctx->res_cache)
            if (!std::memcmp(&r.first, &rk, sizeof(rk))) resident = r.second;
          if (resident < 0) {
            e = pair ? fs::fused_tc2_resident(p, BN, a.lse, G, &resident) : fs::fused_tc_resident(p, BN, a.lse, &resident);
            if (e != cudaSuccess) return cuda_fail(e, "occupancy query");
            if (ctx->res_cache.size() >= 32) ctx->res_cache.erase(ctx->res_cache.begin());
            ctx->res_cache.emplace_back(rk, resident);
          }
          if (G <= resident || !ctx->staging_check) {
            p.h_host = hsrc;
            p.h_bar = reinterpret_cast<unsigned int*>(ctx->fin_buf + 257);
          } else {
            e = fs::launch_copy_in(const_cast<void*>(p.h), hsrc, (size_t)Bc * a.D * esz, p.pdl_w, true, stream);
            if (e != cudaSuccess) return cuda_fail(e, "staging copy kernel launch");
            ++ctx->staged_fallbacks;
          }
        }
      }
      if (fin_lse) {
        p.fin_lse = 1;
        p.fin_ctr = reinterpret_cast<unsigned int*>(ctx->fin_buf + 256);
        p.idx_out = a.idx_out ? a.idx_out + r0 : nullptr;
        p.score_out = a.score_out ? a.score_out + r0 : nullptr;
        p.logZ_out = a.logZ_out ? a.logZ_out + r0 : nullptr;
        p.groups_out = a.groups_out ? a.groups_out + (size_t)r0 * a.n_groups : nullptr;
        p.logprob_out = a.logprob_out ? a.logprob_out + r0 : nullptr;
      }
      if (pair) {
        e = fs::launch_fused_tc2(hmap, p, BN, a.lse, G, stream);
        if (e != cudaSuccess) return cuda_fail(e, "stage-1 tcgen05 pair kernel launch");
      } else {
        e = fs::launch_fused_tc(hmap, p, BN, a.lse, G, stream);
        if (e != cudaSuccess) return cuda_fail(e, "stage-1 tcgen05 kernel launch");
      }
    } else {
      e = fs::launch_fused_simt(p, a.dtype, a.lse, stream);
      if (e != cudaSuccess) return cuda_fail(e, "stage-1 CUDA-core kernel launch");
    }
    if (ev_end) cudaEventRecord(ev_end, stream);
    if (fin || fin_lse) continue;             // stage 1 wrote the outputs
    const int* grp_lo = nullptr;
    if (a.n_groups > 1 && ctx->grp_ranges && (st = group_ranges(ctx, lay, a.n_groups, &grp_lo)) != FS_OK)
      return st;
    fs::State* gscratch = nullptr;
    if (grp_lo) {                             // warp-per-(row, group) stage 2: scratch + row counters
      if (!ctx->grp_rowcnt) {
        e = cudaMalloc(&ctx->grp_rowcnt, 256 * sizeof(int));
        if (e != cudaSuccess) return fail(FS_ERR_OOM, std::string("group row counter cudaMalloc failed: ") + cudaGetErrorString(e) + kAllocHint);
        e = cudaMemset(ctx->grp_rowcnt, 0, 256 * sizeof(int));
        if (e != cudaSuccess) return cuda_fail(e, "group row counter memset");
      }
      const size_t need = (size_t)Bc * a.n_groups * sizeof(fs::State);
      if (need > ctx->gscratch_bytes) {
        if (ctx->gscratch) cudaFree(ctx->gscratch);
        ctx->gscratch = nullptr;
        ctx->gscratch_bytes = 0;
        e = cudaMalloc(&ctx->gscratch, need);
        if (e != cudaSuccess) return fail(FS_ERR_OOM, std::string("group scratch cudaMalloc failed: ") + cudaGetErrorString(e) + kAllocHint);
        ctx->gscratch_bytes = need;
      }
      gscratch = static_cast<fs::State*>(ctx->gscratch);
    }
    e = fs::launch_reduce(part, part_group, lay, Bc, a.n_groups, a.idx_out ? a.idx_out + r0 : nullptr,
                          a.score_out ? a.score_out + r0 : nullptr, a.logZ_out ? a.logZ_out + r0 : nullptr,
                          a.groups_out ? a.groups_out + (size_t)r0 * a.n_groups : nullptr, stream,
                          ctx->pdl != 0 && !ctx->time_stage1, a.logprob_out ? a.logprob_out + r0 : nullptr,
                          grp_lo, gscratch, grp_lo ? ctx->grp_rowcnt : nullptr, a.push, ctx->grp_kernel);
    if (e != cudaSuccess) return cuda_fail(e, "stage-2 reduce launch");
  }
  return FS_OK;
}

// Top-k / top-p through the LM head (reading R19).  Stage 1 either keeps the
// k best (key(l~), id) per (row, CTA) in the epilogue (mode 1: logits never leave the SM) or,
// when those lists do not fit in shared memory, stores the raw fp32 logits (mode 2) for the
// chunked top-k kernels.  Both routes see the same fp32 accumulator and transform, so they pick
// the same token.  Stage 2 = topk_final_kernel (merge, top-p, Gumbel-max over the kept set).
fs_status run_topk_path(fs_ctx* ctx, const PathArgs& a, int k, float top_p, cudaStream_t stream) {
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  const bool tc = !ctx->force_simt && a.dtype == FS_BF16 && (a.D % 8 == 0) && aligned16(a.h) && aligned16(a.W);
  const size_t esz = a.dtype == FS_BF16 ? 2 : 4;
  const int unit = ctx->unit_rows > 0 ? ctx->unit_rows : 16;
  const int U = (a.V + unit - 1) / unit;
  const int G = std::min(std::max(1, ctx->max_ctas > 0 ? ctx->max_ctas : ctx->num_sms), U);
  const int chunk = 256;
  const int Bc_max = std::min(a.B, chunk);
  const int BN_max = fs::tc_block_n(Bc_max);
  const int cap = ((k + 31) / 32) * 32 + 128;
  const int extra = fs::tc_topk_extra_bytes(BN_max, cap);
  // lists only when the TMA ring keeps >= 8 K-slices (128 KB of W) in flight next to them
  // (fewer starve the HBM stream; measured: B=64, k=50 -> 4 slices, 356 vs 166 us stage 1)
  auto ring_slices = [&](int BN, int ex) {
    int best = 0;
    for (int kk = 1; kk <= 4; ++kk) {
      const int S = fs::tc_stages(BN, kk, ex);
      if (S >= 2) best = std::max(best, kk * S);
    }
    return best;
  };
  const int slices = tc ? ring_slices(BN_max, extra) : 0;
  if (ctx->topk_mode == 1 && slices < 2)
    return fail(FS_ERR_UNSUPPORTED, "top-k candidate lists do not fit in shared memory for this B and k (topk_mode=1)");
  // raw-logit route with span maxima (stage 1 also writes per-32-row maxima; only the spans at or
  // above the k-th largest are read back): needs the tcgen05 kernel and no bias / mask (the bound is
  // taken on raw logits, valid under the monotone temperature transform)
  const bool spans_ok = tc && ctx->topk_spans && !a.bias && !a.mask && (a.V + 15) / 16 <= 32768;
  // auto: lists for k <= 128 when the ring keeps >= 8 slices (measured: at k = 200 the
  // per-tile compactions cost more than the raw-logit round trip), and -- where the span route is
  // available -- only up to B = 16: from B = 32 the span route is faster (§11 entry 36)
  const bool lists = ctx->topk_mode == 1 ||
                     (ctx->topk_mode == 0 && slices >= 8 && k <= 128 && (BN_max <= 16 || !spans_ok));
  const bool spans = !lists && spans_ok;
  if ((lists || spans) && !ctx->topk_rowcnt) {
    e = cudaMalloc(&ctx->topk_rowcnt, 256 * sizeof(int));
    if (e != cudaSuccess) return fail(FS_ERR_OOM, std::string("row counter cudaMalloc failed: ") + cudaGetErrorString(e) + kAllocHint);
    e = cudaMemset(ctx->topk_rowcnt, 0, 256 * sizeof(int));
    if (e != cudaSuccess) return cuda_fail(e, "row counter memset");
  }
  const CUtensorMap* wmaps = nullptr;
  int max_seg = 1;
  // raw-logit route on the CTA-pair kernel (M = 256, each CTA loads half of h; pair tiles in 32-row
  // units so that every CTA half starts on a 16-row span unit) above B = 128, where halving the h
  // traffic pays (measured per call, k = 50: B = 256 360 -> 329 us; B = 64 / 128 no gain);
  // option pair = 1 forces it from the pair batch size on
  const bool pair2 = tc && !lists && a.B <= chunk && ctx->pair != 0 && G >= 2 &&
                     (ctx->pair == 1 ? BN_max >= ctx->pair_min_bn : BN_max > 128);
  const int G2 = pair2 ? (G / 2) * 2 : G;
  if (tc) {
    fs_status st0 = pair2 ? segment_maps(ctx, a.W, a.D, a.V, G2 / 2, unit, a.V, &wmaps, &max_seg, 1, 32)
                          : segment_maps(ctx, a.W, a.D, a.V, G, unit, a.V, &wmaps, &max_seg, 0, 16);   // top-k modes
    if (st0 != FS_OK) return st0;
  }
  // workspace: candidates [Bc][G*k] (lists) or logits [Bc][V] fp32 + chunk candidates
  const int nslot = lists ? G : fs::topk_chunks(a.V);
  const int stride = lists ? G * cap : spans ? a.V : nslot * k;   // candidates per row
  const size_t cand_bytes = (size_t)Bc_max * (stride * sizeof(fs::Cand) + nslot * sizeof(uint32_t));
  const size_t mat_off = (cand_bytes + 255) & ~size_t(255);
  const size_t mat_bytes = lists ? 0 : (size_t)Bc_max * a.V * sizeof(float);
  const int64_t gld = ((int64_t)a.V + 15) / 16;
  const size_t gmax_off = (mat_off + mat_bytes + 255) & ~size_t(255);
  const size_t gmax_bytes = spans ? (size_t)Bc_max * gld * sizeof(uint32_t) : 0;
  fs_status st = ensure_ws(ctx, gmax_off + gmax_bytes);
  if (st != FS_OK) return st;
  fs::Cand* cand = static_cast<fs::Cand*>(ctx->ws);
  float* mat = reinterpret_cast<float*>(static_cast<char*>(ctx->ws) + mat_off);
  uint32_t* gmax = spans ? reinterpret_cast<uint32_t*>(static_cast<char*>(ctx->ws) + gmax_off) : nullptr;
  for (int r0 = 0; r0 < a.B; r0 += chunk) {
    const int Bc = std::min(chunk, a.B - r0);
    fs::StageOneParams p{};
    p.h = static_cast<const char*>(a.h) + (size_t)r0 * a.D * esz;
    p.W = a.W;
    p.bias = a.bias;
    p.temperature = a.temperature ? a.temperature + r0 : nullptr;
    p.mask = a.mask ? a.mask + (size_t)r0 * a.mask_words : nullptr;
    p.mask_words = a.mask_words;
    p.vocab_offset = a.vocab_offset;
    p.seed = a.seed;
    p.step = a.step;
    p.B = Bc;
    p.D = a.D;
    p.V = a.V;
    p.row_offset = r0;
    p.group_size = ((a.V + 127) / 128) * 128;
    p.max_seg = max_seg;
    p.unit_rows = unit;
    p.mode = lists ? 1 : 2;
    p.topk_k = k;
    p.topk_cap = cap;
    p.topk_cand = cand;
    p.topk_stride = stride;
    p.topk_rowcnt = ctx->topk_rowcnt;
    p.topk_lb = reinterpret_cast<uint32_t*>(cand + (size_t)Bc * stride);
    p.topk_m = (k + G - 1) / G;
    p.mat_out = mat;
    p.mat_ld = a.V;
    p.topk_gmax = gmax;
    p.topk_gld = gld;
    cudaEvent_t ev_end = nullptr;
    if ((st = stage1_event(ctx, stream, &ev_end)) != FS_OK) return st;
    if (tc) {
      const int BN = fs::tc_block_n(Bc);
      p.w_policy = ctx->w_policy;
      p.dbg_no_epi = ctx->dbg_no_epi;
      p.dbg_no_mma = ctx->dbg_no_mma;
      if (pair2) {
        p.kbps = 1;
        for (int kk = 4; kk >= 2; --kk)
          if (fs::tc2_stages(BN, kk) >= 3) { p.kbps = kk; break; }
        p.stages = fs::tc2_stages(BN, p.kbps);
        CUtensorMap hmap;
        if ((st = make_map(ctx, &hmap, p.h, a.D, Bc, BN / 2)) != FS_OK) return st;
        p.wmaps = wmaps;
        e = fs::launch_fused_tc2_raw(hmap, p, BN, G2, stream);
        if (e != cudaSuccess) return cuda_fail(e, "stage-1 tcgen05 pair raw-logit kernel launch");
      } else {
      const int ex = lists ? fs::tc_topk_extra_bytes(BN, cap) : 0;
      p.kbps = 0;
      for (int kk = 4; kk >= 2; --kk)
        if (fs::tc_stages(BN, kk, ex) >= 3) { p.kbps = kk; break; }
      if (p.kbps == 0) {                      // no depth-3 ring: the most slices with >= 2 stages
        int best = 0;
        for (int kk = 1; kk <= 4; ++kk) {
          const int S = fs::tc_stages(BN, kk, ex);
          if (S >= 2 && kk * S > best) { best = kk * S; p.kbps = kk; }
        }
      }
      if (p.kbps == 0) p.kbps = 1;
      p.stages = fs::tc_stages(BN, p.kbps, ex);
      if (p.stages < 2) return fail(FS_ERR_INVALID, "shared memory too small for the top-k epilogue");
      CUtensorMap hmap;
      if ((st = make_map(ctx, &hmap, p.h, a.D, Bc, BN)) != FS_OK) return st;
      p.wmaps = wmaps;
      e = fs::launch_fused_tc_topk(hmap, p, BN, G, stream);
      if (e != cudaSuccess) return cuda_fail(e, "stage-1 top-k kernel launch");
      }
    } else {
      e = fs::launch_fused_simt(p, a.dtype, false, stream);
      if (e != cudaSuccess) return cuda_fail(e, "stage-1 CUDA-core logits kernel launch");
    }
    if (ev_end) cudaEventRecord(ev_end, stream);
    int32_t* idx = a.idx_out + r0;
    float* sc = a.score_out ? a.score_out + r0 : nullptr;
    float* lz = a.logZ_out ? a.logZ_out + r0 : nullptr;
    float* lp = a.logprob_out ? a.logprob_out + r0 : nullptr;
    const uint64_t* sd = a.seeds ? a.seeds + r0 : nullptr;
    const uint64_t* stp = a.steps ? a.steps + r0 : nullptr;
    if (lists)
      e = fs::launch_topk_final(cand, stride, ctx->topk_rowcnt, Bc, k, top_p, p.temperature, a.seed, a.step, sd, stp,
                                idx, sc, lz, lp, stream, r0, ctx->pdl != 0 && !ctx->time_stage1, p.topk_lb, G,
                                p.topk_m);
    else if (spans) {
      e = fs::launch_topk_gather(mat, a.V, gmax, gld, p.temperature, Bc, a.V, k, cand, stride, ctx->topk_rowcnt,
                                 stream);
      if (e == cudaSuccess)
        e = fs::launch_topk_final(cand, stride, ctx->topk_rowcnt, Bc, k, top_p, p.temperature, a.seed, a.step, sd,
                                  stp, idx, sc, lz, lp, stream, r0, false, nullptr, 0, 1);
    } else
      e = fs::launch_topk_sample(FS_F32, mat, a.V, a.bias, p.temperature, p.mask, a.mask_words, Bc, a.V, k, top_p,
                                 a.seed, a.step, sd, stp, cand, idx, sc, lz, lp, stream, r0);
    if (e != cudaSuccess) {
      if (lists || spans) cudaMemsetAsync(ctx->topk_rowcnt, 0, 256 * sizeof(int), stream);   // keep the counters valid
      return cuda_fail(e, "top-k stage-2 launch");
    }
  }
  return FS_OK;
}

#define FS_LOCK(ctx) std::lock_guard<std::recursive_mutex> fs_guard_((ctx)->mu)

fs_status check_common(fs_ctx* ctx, fs_dtype dtype, const void* h, const void* W, int B, int D, int V) {
  if (!ctx) return fail(FS_ERR_INVALID, "ctx is NULL");
  if (dtype != FS_BF16 && dtype != FS_F32) return fail(FS_ERR_INVALID, "unknown dtype");
  if (!h || !W) return fail(FS_ERR_INVALID, "h and W are required");
  if (B < 1 || D < 1 || V < 1) return fail(FS_ERR_INVALID, "B, D and V must be >= 1");
  const size_t esz = dtype == FS_BF16 ? 2 : 4;
  if ((reinterpret_cast<uintptr_t>(h) | reinterpret_cast<uintptr_t>(W)) % esz)
    return fail(FS_ERR_INVALID, "h and W must be aligned to their element size");
  return FS_OK;
}

}  // namespace

extern "C" {

const char* fs_version(void) { return FS_VERSION_STRING; }

const char* fs_status_str(fs_status s) {
  switch (s) {
    case FS_OK: return "FS_OK";
    case FS_ERR_INVALID: return "FS_ERR_INVALID";
    case FS_ERR_UNSUPPORTED: return "FS_ERR_UNSUPPORTED";
    case FS_ERR_CUDA: return "FS_ERR_CUDA";
    case FS_ERR_OOM: return "FS_ERR_OOM";
    case FS_ERR_NCCL: return "FS_ERR_NCCL";
  }
  return "FS_ERR_UNKNOWN";
}

const char* fs_last_error(void) { return g_last_error.c_str(); }

fs_status fs_ctx_create(int device, fs_ctx** out) {
  if (!out) return fail(FS_ERR_INVALID, "out is NULL");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return fail(FS_ERR_UNSUPPORTED, "no CUDA device available");
  if (device < 0 || device >= n) return fail(FS_ERR_INVALID, "device ordinal out of range");
  int major = 0, minor = 0, sms = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (major != 10 || minor != 0)
    return fail(FS_ERR_UNSUPPORTED, "this build targets sm_100a (B200); device is sm_" + std::to_string(major) +
                                        std::to_string(minor));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || fn == nullptr) return fail(FS_ERR_CUDA, "cuTensorMapEncodeTiled entry point not found");
  fs_ctx* c = new fs_ctx();
  c->device = device;
  c->num_sms = sms;
  c->encode = reinterpret_cast<PFN_encodeTiled>(fn);
  *out = c;
  return FS_OK;
}

void fs_ctx_destroy(fs_ctx* ctx) {
  if (!ctx) return;
  for (auto& e : ctx->seg_cache) cudaFree(e.dev);
  for (auto& e : ctx->grp_cache) cudaFree(e.dev);
  for (auto& pr : ctx->ev_pool) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->topk_rowcnt) cudaFree(ctx->topk_rowcnt);
  if (ctx->fin_buf) cudaFree(ctx->fin_buf);
  if (ctx->grp_rowcnt) cudaFree(ctx->grp_rowcnt);
  if (ctx->gscratch) cudaFree(ctx->gscratch);
  fs_comm_window_destroy(ctx);
  fs_comm_destroy(ctx);
  delete ctx;
}

fs_status fs_ctx_set_option(fs_ctx* ctx, const char* name, int64_t value) {
  if (!ctx || !name) return fail(FS_ERR_INVALID, "ctx and name are required");
  FS_LOCK(ctx);
  if (!strcmp(name, "force_simt")) ctx->force_simt = (int)value;
  else if (!strcmp(name, "max_ctas")) ctx->max_ctas = (int)value;
  else if (!strcmp(name, "pdl")) ctx->pdl = (int)value;
  else if (!strcmp(name, "stages")) ctx->stages_override = (int)value;
  else if (!strcmp(name, "kbps")) ctx->kbps = (int)value;
  else if (!strcmp(name, "dbg_no_mma")) ctx->dbg_no_mma = (int)value;
  else if (!strcmp(name, "dbg_no_epi")) ctx->dbg_no_epi = (int)value;
  else if (!strcmp(name, "l2promo")) ctx->l2promo = (int)value;
  else if (!strcmp(name, "w_policy")) ctx->w_policy = (int)value;
  else if (!strcmp(name, "epi_sleep")) ctx->epi_sleep = (int)value;
  else if (!strcmp(name, "pair")) ctx->pair = (int)value;
  else if (!strcmp(name, "fuse_reduce")) ctx->fuse_reduce = (int)value;
  else if (!strcmp(name, "whole_tiles")) ctx->whole_tiles = (int)value;
  else if (!strcmp(name, "topk_spans")) ctx->topk_spans = (int)value;
  else if (!strcmp(name, "grp_ranges")) ctx->grp_ranges = (int)value;
  else if (!strcmp(name, "pdl_w")) ctx->pdl_w = (int)value;
  else if (!strcmp(name, "spin_wait")) ctx->spin_wait = (int)value;
  else if (!strcmp(name, "grp_kernel")) ctx->grp_kernel = (int)value;
  else if (!strcmp(name, "done_flag")) ctx->done_flag = reinterpret_cast<unsigned long long*>(value);
  else if (!strcmp(name, "pdl_w_max_b")) ctx->pdl_w_max_b = (int)value;
  else if (!strcmp(name, "staging_check")) ctx->staging_check = (int)value;
  else if (!strcmp(name, "dbg_times")) ctx->dbg_times = reinterpret_cast<unsigned long long*>(value);
  else if (!strcmp(name, "pair_min_bn")) ctx->pair_min_bn = (int)value;
  else if (!strcmp(name, "topk_mode")) {
    if (value < 0 || value > 2) return fail(FS_ERR_INVALID, "topk_mode must be 0 (auto), 1 (epilogue lists) or 2 (raw logits)");
    ctx->topk_mode = (int)value;
  }
  else if (!strcmp(name, "unit_rows")) {
    if (value != 0 && value != 16 && value != 32 && value != 64 && value != 128)
      return fail(FS_ERR_INVALID, "unit_rows must be 0, 16, 32, 64 or 128");
    ctx->unit_rows = (int)value;
  }
  else if (!strcmp(name, "time_stage1")) { ctx->time_stage1 = (int)value; ctx->ev_used = 0; }
  else return fail(FS_ERR_INVALID, std::string("unknown option ") + name);
  return FS_OK;
}

fs_status fs_ctx_query(fs_ctx* ctx, const char* name, double* out) {
  if (!ctx || !name || !out) return fail(FS_ERR_INVALID, "ctx, name and out are required");
  FS_LOCK(ctx);
  if (!strcmp(name, "stage1_launches")) {
    *out = (double)ctx->ev_used;
    return FS_OK;
  }
  if (!strcmp(name, "stage1_ms")) {
    double total = 0.0;
    for (size_t i = 0; i < ctx->ev_used; ++i) {
      cudaError_t e = cudaEventSynchronize(ctx->ev_pool[i].second);
      if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize");
      float ms = 0.f;
      e = cudaEventElapsedTime(&ms, ctx->ev_pool[i].first, ctx->ev_pool[i].second);
      if (e != cudaSuccess) return cuda_fail(e, "cudaEventElapsedTime");
      total += ms;
    }
    ctx->ev_used = 0;
    *out = total;
    return FS_OK;
  }
  if (!strcmp(name, "comm_timeouts")) {
    unsigned t = 0;
    if (ctx->comm_win) {
      cudaError_t e = cudaMemcpy(&t, ctx->comm_win + ctx->comm_off_status, sizeof(t), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return cuda_fail(e, "comm status read");
    }
    *out = (double)t;
    return FS_OK;
  }
  if (!strcmp(name, "staging_timeouts")) {
    unsigned t = 0;
    if (ctx->fin_buf) {
      cudaError_t e = cudaMemcpy(&t, reinterpret_cast<unsigned*>(ctx->fin_buf + 258), sizeof(t), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return cuda_fail(e, "staging status read");
    }
    *out = (double)t;
    return FS_OK;
  }
  if (!strcmp(name, "nccl_world")) {
    *out = ctx->nccl ? (double)ctx->nccl_world : 0.0;
    return FS_OK;
  }
  if (!strcmp(name, "staged_fallbacks")) {
    *out = (double)ctx->staged_fallbacks;
    return FS_OK;
  }
  if (!strcmp(name, "num_sms")) {
    *out = (double)ctx->num_sms;
    return FS_OK;
  }
  return fail(FS_ERR_INVALID, std::string("unknown query ") + name);
}

fs_status fs_sample(fs_ctx* ctx, fs_dtype dtype, const void* h, const void* W, const float* bias,
                    const float* temperature, const uint32_t* mask, uint64_t seed, uint64_t step, int B, int D, int V,
                    int32_t* idx_out, float* score_out, void* stream) {
  fs_status s = check_common(ctx, dtype, h, W, B, D, V);
  if (s != FS_OK) return s;
  FS_LOCK(ctx);
  if (!idx_out) return fail(FS_ERR_INVALID, "idx_out is required");
  PathArgs a{dtype, h, W, bias, temperature, mask, ((int64_t)V + 31) / 32, seed, step, B, D, V, 0,
             ((V + 127) / 128) * 128, false, idx_out, score_out, nullptr, nullptr, 1, nullptr};
  return run_path(ctx, a, static_cast<cudaStream_t>(stream));
}

fs_status fs_sample_staged(fs_ctx* ctx, fs_dtype dtype, const void* h_host, void* h_dev, const void* W,
                           const float* bias, const float* temperature, const uint32_t* mask, uint64_t seed,
                           uint64_t step, int B, int D, int V, int32_t* idx_out, float* score_out, void* stream) {
  fs_status s = check_common(ctx, dtype, h_dev, W, B, D, V);
  if (s != FS_OK) return s;
  FS_LOCK(ctx);
  if (!idx_out || !h_host) return fail(FS_ERR_INVALID, "h_host and idx_out are required");
  const size_t esz = dtype == FS_BF16 ? 2 : 4;
  cudaPointerAttributes at{};
  cudaError_t e = cudaPointerGetAttributes(&at, h_host);
  if (e != cudaSuccess || at.type != cudaMemoryTypeHost)
    return fail(FS_ERR_INVALID, "h_host must be pinned (page-locked) host memory");
  if (reinterpret_cast<uintptr_t>(h_host) & 15u) return fail(FS_ERR_INVALID, "h_host must be 16-byte aligned");
  // in-kernel staging needs the one-kernel tcgen05 path; otherwise the copy kernel stages h
  const bool tc = !ctx->force_simt && dtype == FS_BF16 && (D % 8 == 0) && aligned16(h_dev) && aligned16(W);
  PathArgs a{dtype, h_dev, W, bias, temperature, mask, ((int64_t)V + 31) / 32, seed, step, B, D, V, 0,
             ((V + 127) / 128) * 128, false, idx_out, score_out, nullptr, nullptr, 1, nullptr};
  if (tc && ctx->fuse_reduce) {
    a.h_host = h_host;
  } else {
    s = fs_copy_async(ctx, h_dev, h_host, (size_t)B * D * esz, stream);
    if (s != FS_OK) return s;
  }
  return run_path(ctx, a, static_cast<cudaStream_t>(stream));
}

fs_status fs_sample_grouped(fs_ctx* ctx, fs_dtype dtype, const void* h, const void* W, const float* bias,
                            const float* temperature, const uint32_t* mask, uint64_t seed, uint64_t step, int B,
                            int D, int V, int group_size, int32_t* idx_out, float* score_out, float* logZ_out,
                            float* logprob_out, fs_summary* groups_out, void* stream) {
  fs_status s = check_common(ctx, dtype, h, W, B, D, V);
  if (s != FS_OK) return s;
  FS_LOCK(ctx);
  if (!idx_out) return fail(FS_ERR_INVALID, "idx_out is required");
  if (group_size < 128 || group_size % 128 != 0) return fail(FS_ERR_INVALID, "group_size must be a positive multiple of 128");
  const int n_groups = (V + group_size - 1) / group_size;
  PathArgs a{dtype, h, W, bias, temperature, mask, ((int64_t)V + 31) / 32, seed, step, B, D, V, 0,
             group_size, true, idx_out, score_out, logZ_out, groups_out, n_groups, logprob_out};
  return run_path(ctx, a, static_cast<cudaStream_t>(stream));
}

// The rank-local half of Alg. A.4.  need_lse = false (fs_sample_tp without logZ / per-rank outputs):
// only (M, I) of the records are consumed, so the shard runs the plain epilogue with the one-kernel
// finalize writing the records directly (L = NaN) -- no log-mass epilogue, no stage-2 kernel.
static fs_status shard_impl(fs_ctx* ctx, fs_dtype dtype, const void* h, const void* W_shard, const float* bias_shard,
                            const float* temperature, const uint32_t* mask, uint64_t seed, uint64_t step, int B,
                            int D, int V_local, int64_t vocab_offset, int64_t V_total, fs_summary* summary_out,
                            bool need_lse, void* stream) {
  fs_status s = check_common(ctx, dtype, h, W_shard, B, D, V_local);
  if (s != FS_OK) return s;
  FS_LOCK(ctx);
  if (!summary_out) return fail(FS_ERR_INVALID, "summary_out is required");
  if (vocab_offset < 0 || V_total < vocab_offset + V_local || V_total >= (1LL << 31))
    return fail(FS_ERR_INVALID, "need 0 <= vocab_offset, vocab_offset + V_local <= V_total < 2^31");
  PathArgs a{dtype, h, W_shard, bias_shard, temperature, mask, (V_total + 31) / 32, seed, step, B, D, V_local,
             vocab_offset, ((V_local + 127) / 128) * 128, true, nullptr, nullptr, nullptr, summary_out, 1, nullptr};
  if (!need_lse) {
    a.lse = false;
    a.groups_out = nullptr;
    a.sum_out = summary_out;
  }
  return run_path(ctx, a, static_cast<cudaStream_t>(stream));
}

fs_status fs_sample_shard(fs_ctx* ctx, fs_dtype dtype, const void* h, const void* W_shard, const float* bias_shard,
                          const float* temperature, const uint32_t* mask, uint64_t seed, uint64_t step, int B, int D,
                          int V_local, int64_t vocab_offset, int64_t V_total, fs_summary* summary_out, void* stream) {
  return shard_impl(ctx, dtype, h, W_shard, bias_shard, temperature, mask, seed, step, B, D, V_local, vocab_offset,
                    V_total, summary_out, true, stream);
}

static fs_status sample_logits_impl(fs_ctx* ctx, fs_dtype dtype, const void* logits, int64_t ld, const float* bias,
                                    const float* temperature, const uint32_t* mask, uint64_t seed, uint64_t step,
                                    const uint64_t* seeds, const uint64_t* steps, int B, int V, int32_t* idx_out,
                                    float* score_out, float* logZ_out, float* logprob_out, void* stream) {
  if (!ctx) return fail(FS_ERR_INVALID, "ctx is NULL");
  FS_LOCK(ctx);
  if (dtype != FS_BF16 && dtype != FS_F32) return fail(FS_ERR_INVALID, "unknown dtype");
  if (!logits || !idx_out) return fail(FS_ERR_INVALID, "logits and idx_out are required");
  if (B < 1 || V < 1 || ld < V) return fail(FS_ERR_INVALID, "need B >= 1, V >= 1, ld >= V");
  if (B > 65535 * 4) return fail(FS_ERR_UNSUPPORTED, "B too large");
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  cudaStream_t stream_ = static_cast<cudaStream_t>(stream);
  const int nblk = fs::logits_sample_blocks(B, V);
  const size_t part_bytes = (size_t)nblk * B * sizeof(fs::State);
  const size_t grp_off = (part_bytes + 255) & ~size_t(255);
  fs_status st = ensure_ws(ctx, grp_off + (size_t)nblk * sizeof(int));
  if (st != FS_OK) return st;
  fs::State* part = static_cast<fs::State*>(ctx->ws);
  int* part_group = reinterpret_cast<int*>(static_cast<char*>(ctx->ws) + grp_off);
  const bool lse = logZ_out || logprob_out;
  const bool fin = ctx->fuse_reduce && !lse && B <= 256;   // last block finalizes (no stage-2 launch)
  if (fin && (st = ensure_fin(ctx)) != FS_OK) return st;
  e = fs::launch_logits_sample(dtype, logits, ld, bias, temperature, mask, ((int64_t)V + 31) / 32, B, V, seed, step,
                               lse, nblk, part, part_group, stream_, seeds, steps, fin ? ctx->fin_buf : nullptr,
                               fin ? reinterpret_cast<unsigned int*>(ctx->fin_buf + 256) : nullptr, idx_out, score_out);
  if (e != cudaSuccess) return cuda_fail(e, "logits sampler launch");
  if (fin) return FS_OK;
  const fs::SlotLayout lay{nblk, 1, nblk, V, 1, V, 128, 0};
  e = fs::launch_reduce(part, part_group, lay, B, 1, idx_out, score_out, logZ_out, nullptr, stream_, ctx->pdl != 0,
                        logprob_out);
  return e == cudaSuccess ? FS_OK : cuda_fail(e, "stage-2 reduce launch");
}

fs_status fs_sample_logits(fs_ctx* ctx, fs_dtype dtype, const void* logits, int64_t ld, const float* bias,
                           const float* temperature, const uint32_t* mask, uint64_t seed, uint64_t step, int B, int V,
                           int32_t* idx_out, float* score_out, float* logZ_out, float* logprob_out, void* stream) {
  return sample_logits_impl(ctx, dtype, logits, ld, bias, temperature, mask, seed, step, nullptr, nullptr, B, V,
                            idx_out, score_out, logZ_out, logprob_out, stream);
}

fs_status fs_sample_logits_ex(fs_ctx* ctx, fs_dtype dtype, const void* logits, int64_t ld, int B, int V,
                              const fs_sample_args* a, void* stream) {
  if (!a) return fail(FS_ERR_INVALID, "args is NULL");
  const bool use_p = a->top_p > 0.0f && a->top_p < 1.0f;
  if (a->top_k > 0 || use_p) {
    if (a->top_k < 1 || a->top_k > fs::topk_max_k())
      return fail(FS_ERR_UNSUPPORTED, "top-k sampling needs 1 <= top_k <= 1024 (also required for top_p)");
    if (!ctx) return fail(FS_ERR_INVALID, "ctx is NULL");
  FS_LOCK(ctx);
    if (dtype != FS_BF16 && dtype != FS_F32) return fail(FS_ERR_INVALID, "unknown dtype");
    if (!logits || !a->idx_out) return fail(FS_ERR_INVALID, "logits and idx_out are required");
    if (B < 1 || V < 1 || ld < V) return fail(FS_ERR_INVALID, "need B >= 1, V >= 1, ld >= V");
    if (a->steps && !a->seeds) return fail(FS_ERR_INVALID, "steps requires seeds");
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    fs_status st = ensure_ws(ctx, (size_t)B * fs::topk_chunks(V) * (a->top_k * 8 + 4));
    if (st != FS_OK) return st;
    e = fs::launch_topk_sample(dtype, logits, ld, a->bias, a->temperature, a->mask, ((int64_t)V + 31) / 32, B, V,
                               a->top_k, use_p ? a->top_p : 1.0f, a->seed, a->step, a->seeds, a->steps, ctx->ws,
                               a->idx_out, a->score_out, a->logZ_out, a->logprob_out,
                               static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? FS_OK : cuda_fail(e, "top-k sampler launch");
  }
  return sample_logits_impl(ctx, dtype, logits, ld, a->bias, a->temperature, a->mask, a->seed, a->step, a->seeds,
                            a->steps, B, V, a->idx_out, a->score_out, a->logZ_out, a->logprob_out, stream);
}

fs_status fs_sample_ex(fs_ctx* ctx, fs_dtype dtype, const void* h, const void* W, int B, int D, int V,
                       const fs_sample_args* args, void* stream) {
  if (!args) return fail(FS_ERR_INVALID, "args is NULL");
  fs_status s = check_common(ctx, dtype, h, W, B, D, V);
  if (s != FS_OK) return s;
  FS_LOCK(ctx);
  if (!args->idx_out) return fail(FS_ERR_INVALID, "idx_out is required");
  if (args->steps && !args->seeds) return fail(FS_ERR_INVALID, "steps requires seeds");
  const bool use_p = args->top_p > 0.0f && args->top_p < 1.0f;
  if (args->top_k > 0 || use_p) {
    if (args->top_k < 1 || args->top_k > fs::topk_max_k())
      return fail(FS_ERR_UNSUPPORTED, "top-k sampling needs 1 <= top_k <= 1024 (also required for top_p)");
    if (args->groups_out || (args->group_size > 0 && args->group_size < V))
      return fail(FS_ERR_UNSUPPORTED, "top-k / top-p has no grouped summaries");
    PathArgs a{dtype, h, W, args->bias, args->temperature, args->mask, ((int64_t)V + 31) / 32, args->seed,
               args->step, B, D, V, 0, V, false, args->idx_out, args->score_out, args->logZ_out, nullptr, 1,
               args->logprob_out, args->seeds, args->steps};
    return run_topk_path(ctx, a, args->top_k, use_p ? args->top_p : 1.0f, static_cast<cudaStream_t>(stream));
  }
  int gs = args->group_size;
  if (gs < 0 || (gs > 0 && gs % 128 != 0)) return fail(FS_ERR_INVALID, "group_size must be 0 or a multiple of 128");
  if (gs == 0 || gs >= V) gs = ((V + 127) / 128) * 128;
  const int n_groups = (V + gs - 1) / gs;
  const bool lse = args->logZ_out || args->logprob_out || args->groups_out || n_groups > 1;
  PathArgs a{dtype, h, W, args->bias, args->temperature, args->mask, ((int64_t)V + 31) / 32, args->seed, args->step,
             B, D, V, 0, gs, lse, args->idx_out, args->score_out, args->logZ_out, args->groups_out, n_groups,
             args->logprob_out, args->seeds, args->steps};
  return run_path(ctx, a, static_cast<cudaStream_t>(stream));
}

fs_status fs_comm_window_create(fs_ctx* ctx, int world, int rank, int B_max, fs_ipc_handle* handle_out) {
  if (!ctx || !handle_out) return fail(FS_ERR_INVALID, "ctx and handle_out are required");
  FS_LOCK(ctx);
  if (world < 1 || world > fs::kMaxWorld || rank < 0 || rank >= world || B_max < 1)
    return fail(FS_ERR_INVALID, "need 1 <= world <= 16, 0 <= rank < world, B_max >= 1");
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  fs_comm_window_destroy(ctx);
  const size_t rec = (size_t)2 * world * B_max * sizeof(fs_summary);
  ctx->comm_off_flags = (rec + 127) & ~size_t(127);
  ctx->comm_off_acks = ctx->comm_off_flags + (((size_t)2 * world * 8 + 127) & ~size_t(127));
  ctx->comm_off_status = ctx->comm_off_acks + (((size_t)world * 8 + 127) & ~size_t(127));
  const size_t bytes = ctx->comm_off_status + 128;   // status: [0] timeouts, [64] push block counter
  if ((e = cudaMalloc(&ctx->comm_win, bytes)) != cudaSuccess) return fail(FS_ERR_OOM, std::string("window cudaMalloc failed: ") + cudaGetErrorString(e) + kAllocHint);
  if ((e = cudaMemset(ctx->comm_win, 0, bytes)) != cudaSuccess) return cuda_fail(e, "window memset");
  if ((e = cudaMalloc(&ctx->comm_local, (size_t)B_max * sizeof(fs_summary))) != cudaSuccess)
    return fail(FS_ERR_OOM, std::string("summary cudaMalloc failed: ") + cudaGetErrorString(e) + kAllocHint);
  cudaIpcMemHandle_t h;
  if ((e = cudaIpcGetMemHandle(&h, ctx->comm_win)) != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  static_assert(sizeof(h) <= sizeof(fs_ipc_handle), "IPC handle size");
  std::memset(handle_out, 0, sizeof(*handle_out));
  std::memcpy(handle_out->bytes, &h, sizeof(h));
  ctx->comm_world = world;
  ctx->comm_rank = rank;
  ctx->comm_bmax = B_max;
  ctx->comm_epoch = 0;
  return FS_OK;
}

fs_status fs_comm_window_open(fs_ctx* ctx, const fs_ipc_handle* handles) {
  if (!ctx || !handles) return fail(FS_ERR_INVALID, "ctx and handles are required");
  FS_LOCK(ctx);
  if (!ctx->comm_win) return fail(FS_ERR_INVALID, "fs_comm_window_create first");
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  for (int p = 0; p < ctx->comm_world; ++p) {
    if (p == ctx->comm_rank) { ctx->comm_peer[p] = ctx->comm_win; continue; }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles[p].bytes, sizeof(h));
    void* ptr = nullptr;
    if ((e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess)) != cudaSuccess)
      return cuda_fail(e, "cudaIpcOpenMemHandle");
    ctx->comm_peer[p] = static_cast<char*>(ptr);
  }
  fs::PeerTab tab{};
  for (int p = 0; p < ctx->comm_world; ++p) {
    tab.rec[p] = reinterpret_cast<fs_summary*>(ctx->comm_peer[p]);
    tab.flags[p] = reinterpret_cast<uint64_t*>(ctx->comm_peer[p] + ctx->comm_off_flags);
    tab.acks[p] = reinterpret_cast<uint64_t*>(ctx->comm_peer[p] + ctx->comm_off_acks);
  }
  if (!ctx->comm_peertab && (e = cudaMalloc(&ctx->comm_peertab, sizeof(tab))) != cudaSuccess)
    return fail(FS_ERR_OOM, std::string("peer table cudaMalloc failed: ") + cudaGetErrorString(e) + kAllocHint);
  if ((e = cudaMemcpy(ctx->comm_peertab, &tab, sizeof(tab), cudaMemcpyHostToDevice)) != cudaSuccess)
    return cuda_fail(e, "peer table upload");
  ctx->comm_open = true;
  return FS_OK;
}

fs_status fs_comm_window_destroy(fs_ctx* ctx) {
  if (!ctx) return fail(FS_ERR_INVALID, "ctx is NULL");
  FS_LOCK(ctx);
  cudaSetDevice(ctx->device);
  if (ctx->comm_open)
    for (int p = 0; p < ctx->comm_world; ++p)
      if (p != ctx->comm_rank && ctx->comm_peer[p]) cudaIpcCloseMemHandle(ctx->comm_peer[p]);
  for (auto& q : ctx->comm_peer) q = nullptr;
  ctx->comm_open = false;
  if (ctx->comm_win) cudaFree(ctx->comm_win);
  if (ctx->comm_local) cudaFree(ctx->comm_local);
  if (ctx->comm_peertab) cudaFree(ctx->comm_peertab);
  ctx->comm_win = nullptr;
  ctx->comm_local = nullptr;
  ctx->comm_peertab = nullptr;
  ctx->comm_world = 0;
  return FS_OK;
}

fs_status fs_sample_tp_push(fs_ctx* ctx, fs_dtype dtype, const void* h, const void* W_shard, const float* bias_shard,
                            const float* temperature, const uint32_t* mask, uint64_t seed, uint64_t step, int B, int D,
                            int V_local, int64_t vocab_offset, int64_t V_total, int32_t* idx_out, float* score_out,
                            float* logZ_out, void* stream) {
  if (!ctx || !ctx->comm_open) return fail(FS_ERR_INVALID, "open the exchange window first (fs_comm_window_open)");
  FS_LOCK(ctx);
  if (!idx_out) return fail(FS_ERR_INVALID, "idx_out is required");
  if (B > ctx->comm_bmax) return fail(FS_ERR_INVALID, "B exceeds the window's B_max");
  fs_status s = check_common(ctx, dtype, h, W_shard, B, D, V_local);
  if (s != FS_OK) return s;
  if (vocab_offset < 0 || V_total < vocab_offset + V_local || V_total >= (1LL << 31))
    return fail(FS_ERR_INVALID, "need 0 <= vocab_offset, vocab_offset + V_local <= V_total < 2^31");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned* status = reinterpret_cast<unsigned*>(ctx->comm_win + ctx->comm_off_status);
  const uint64_t epoch = ++ctx->comm_epoch;
  const fs::PushCtx pc{ctx->comm_peertab, ctx->comm_world, ctx->comm_rank, ctx->comm_bmax, epoch, status + 16,
                       status};
  const bool tc = !ctx->force_simt && dtype == FS_BF16 && (D % 8 == 0) && aligned16(h) && aligned16(W_shard);
  if (B <= 256 && !logZ_out && tc && ctx->fuse_reduce) {
    // fully fused (no log-mass needed): ONE kernel per rank -- the shard's finalizing CTA writes the
    // records into every peer window, releases its flags, waits for the n ranks' records, combines
    // into idx_out / score_out and acknowledges (fs_epilogue.cuh finalize_last_cta)
    PathArgs a{dtype, h, W_shard, bias_shard, temperature, mask, (V_total + 31) / 32, seed, step, B, D, V_local,
               vocab_offset, ((V_local + 127) / 128) * 128, false, idx_out, score_out, nullptr, nullptr, 1,
               nullptr};
    a.sum_out = ctx->comm_local;
    a.push = &pc;
    return run_path(ctx, a, st);
  }
  if (B <= 256) {
    // fused push: the shard sampler's last reduction step (the last stage-1 CTA for B <= 16, else the
    // stage-2 row reduce) stores the records into every peer window and releases the flags; one
    // PDL-chained block then waits for the n flags and combines
    PathArgs a{dtype, h, W_shard, bias_shard, temperature, mask, (V_total + 31) / 32, seed, step, B, D, V_local,
               vocab_offset, ((V_local + 127) / 128) * 128, true, nullptr, nullptr, nullptr, ctx->comm_local, 1,
               nullptr};
    a.push = &pc;
    if ((s = run_path(ctx, a, st)) != FS_OK) return s;
    cudaError_t e = fs::launch_exchange_wait(ctx->comm_peertab, ctx->comm_world, ctx->comm_rank, B, ctx->comm_bmax,
                                             epoch, idx_out, score_out, logZ_out, status, st, ctx->pdl != 0);
    return e == cudaSuccess ? FS_OK : cuda_fail(e, "exchange wait kernel launch");
  }
  s = fs_sample_shard(ctx, dtype, h, W_shard, bias_shard, temperature, mask, seed, step, B, D, V_local, vocab_offset,
                      V_total, ctx->comm_local, stream);
  if (s != FS_OK) return s;
  fs::PeerTab peers{};
  for (int p = 0; p < ctx->comm_world; ++p) {
    peers.rec[p] = reinterpret_cast<fs_summary*>(ctx->comm_peer[p]);
    peers.flags[p] = reinterpret_cast<uint64_t*>(ctx->comm_peer[p] + ctx->comm_off_flags);
    peers.acks[p] = reinterpret_cast<uint64_t*>(ctx->comm_peer[p] + ctx->comm_off_acks);
  }
  cudaError_t e = fs::launch_exchange_combine(ctx->comm_local, peers, ctx->comm_world, ctx->comm_rank, B,
                                              ctx->comm_bmax, epoch, idx_out, score_out, logZ_out, status, st,
                                              ctx->pdl != 0);
  return e == cudaSuccess ? FS_OK : cuda_fail(e, "exchange kernel launch");
}

fs_status fs_comm_unique_id(void* id_out) {
  if (!id_out) return fail(FS_ERR_INVALID, "id_out is required");
  const fs::NcclApi& nc = fs::nccl_api();
  if (!nc.ok) return fail(FS_ERR_UNSUPPORTED, std::string("NCCL unavailable: ") + nc.why);
  ncclUniqueId id;
  const ncclResult_t r = nc.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(FS_ERR_NCCL, std::string("ncclGetUniqueId: ") + nc.GetErrorString(r));
  std::memcpy(id_out, &id, sizeof(id));
  return FS_OK;
}

fs_status fs_comm_init(fs_ctx* ctx, const void* nccl_unique_id, int world, int rank) {
  if (!ctx || !nccl_unique_id) return fail(FS_ERR_INVALID, "ctx and nccl_unique_id are required");
  FS_LOCK(ctx);
  if (world < 1 || rank < 0 || rank >= world) return fail(FS_ERR_INVALID, "need world >= 1, 0 <= rank < world");
  const fs::NcclApi& nc = fs::nccl_api();
  if (!nc.ok) return fail(FS_ERR_UNSUPPORTED, std::string("NCCL unavailable: ") + nc.why);
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  fs_comm_destroy(ctx);
  ncclUniqueId id;
  std::memcpy(&id, nccl_unique_id, sizeof(id));
  const ncclResult_t r = nc.CommInitRank(&ctx->nccl, world, id, rank);
  if (r != ncclSuccess) {
    ctx->nccl = nullptr;
    return fail(FS_ERR_NCCL, std::string("ncclCommInitRank: ") + nc.GetErrorString(r));
  }
  ctx->nccl_world = world;
  ctx->nccl_rank = rank;
  return FS_OK;
}

fs_status fs_comm_destroy(fs_ctx* ctx) {
  if (!ctx) return fail(FS_ERR_INVALID, "ctx is NULL");
  FS_LOCK(ctx);
  if (ctx->nccl) {
    cudaSetDevice(ctx->device);
    fs::nccl_api().CommDestroy(ctx->nccl);
  }
  if (ctx->tp_buf) cudaFree(ctx->tp_buf);
  ctx->nccl = nullptr;
  ctx->tp_buf = nullptr;
  ctx->tp_bmax = 0;
  ctx->nccl_world = 0;
  return FS_OK;
}

fs_status fs_sample_tp(fs_ctx* ctx, fs_dtype dtype, const void* h, const void* W_shard, const float* bias_shard,
                       const float* temperature, const uint32_t* mask, uint64_t seed, uint64_t step, int B, int D,
                       int V_local, int64_t vocab_offset, int64_t V_total, int32_t* idx_out, float* score_out,
                       float* logZ_out, fs_summary* per_rank_out, void* stream) {
  if (!ctx) return fail(FS_ERR_INVALID, "ctx is NULL");
  FS_LOCK(ctx);
  if (!ctx->nccl) return fail(FS_ERR_INVALID, "no communicator: call fs_comm_init first");
  if (!idx_out) return fail(FS_ERR_INVALID, "idx_out is required");
  const fs::NcclApi& nc = fs::nccl_api();
  // an error of an earlier asynchronous collective surfaces here
  ncclResult_t ar = ncclSuccess;
  ncclResult_t r = nc.CommGetAsyncError(ctx->nccl, &ar);
  if (r != ncclSuccess || (ar != ncclSuccess && ar != ncclInProgress))
    return fail(FS_ERR_NCCL, std::string("NCCL communicator error: ") + nc.GetErrorString(r != ncclSuccess ? r : ar));
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  const int world = ctx->nccl_world;
  if (B > ctx->tp_bmax) {
    if (ctx->tp_buf) cudaFree(ctx->tp_buf);
    ctx->tp_buf = nullptr;
    ctx->tp_bmax = 0;
    if ((e = cudaMalloc(&ctx->tp_buf, (size_t)(1 + world) * B * sizeof(fs_summary))) != cudaSuccess)
      return fail(FS_ERR_OOM, std::string("TP summary buffer cudaMalloc failed: ") + cudaGetErrorString(e) + kAllocHint);
    ctx->tp_bmax = B;
  }
  fs_summary* local = ctx->tp_buf;
  fs_summary* gathered = ctx->tp_buf + ctx->tp_bmax;
  // without logZ / per-rank outputs only (M, I) matter: the shard skips the log-mass epilogue
  fs_status s = shard_impl(ctx, dtype, h, W_shard, bias_shard, temperature, mask, seed, step, B, D, V_local,
                           vocab_offset, V_total, local, logZ_out != nullptr || per_rank_out != nullptr, stream);
  if (s != FS_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // Alg. A.4 line 4: every rank contributes its B x 12-byte message; [world][B] arrives
  r = nc.AllGather(local, gathered, (size_t)B * sizeof(fs_summary), ncclUint8, ctx->nccl, st);
  if (r != ncclSuccess) return fail(FS_ERR_NCCL, std::string("ncclAllGather: ") + nc.GetErrorString(r));
  e = fs::launch_combine(gathered, world, B, idx_out, score_out, logZ_out, st);
  if (e != cudaSuccess) return cuda_fail(e, "combine launch");
  if (per_rank_out && (e = cudaMemcpyAsync(per_rank_out, gathered, (size_t)world * B * sizeof(fs_summary),
                                           cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
    return cuda_fail(e, "per-rank summary copy");
  return FS_OK;
}

fs_status fs_combine_summaries(const fs_summary* gathered, int n, int B, int32_t* idx_out, float* score_out,
                               float* logZ_out, void* stream) {
  if (!gathered || !idx_out || n < 1 || B < 1) return fail(FS_ERR_INVALID, "gathered, idx_out, n >= 1, B >= 1 required");
  cudaError_t e = fs::launch_combine(gathered, n, B, idx_out, score_out, logZ_out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FS_OK : cuda_fail(e, "combine launch");
}

fs_status fs_merge_summaries(const fs_summary* a, const fs_summary* b, fs_summary* out, int count, void* stream) {
  if (!a || !b || !out || count < 0) return fail(FS_ERR_INVALID, "a, b, out required");
  if (count == 0) return FS_OK;
  cudaError_t e = fs::launch_merge(a, b, out, count, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FS_OK : cuda_fail(e, "merge launch");
}

fs_status fs_random_bits(uint64_t seed, uint64_t step, uint32_t tag, const int32_t* b, const int64_t* v,
                         uint32_t* r_out, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!b || !v || !r_out))) return fail(FS_ERR_INVALID, "b, v, r_out required");
  cudaError_t e = fs::launch_random_bits(seed, step, tag, b, v, r_out, n, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FS_OK : cuda_fail(e, "random_bits launch");
}

fs_status fs_copy_async(fs_ctx* ctx, void* dst, const void* src, size_t bytes, void* stream) {
  if (!ctx) return fail(FS_ERR_INVALID, "ctx is required");
  FS_LOCK(ctx);
  if (bytes == 0) return FS_OK;
  if (!dst || !src) return fail(FS_ERR_INVALID, "dst and src are required");
  if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15u)
    return fail(FS_ERR_INVALID, "dst and src must be 16-byte aligned");
  cudaPointerAttributes at{};
  cudaError_t e = cudaPointerGetAttributes(&at, src);
  if (e != cudaSuccess || (at.type != cudaMemoryTypeHost && at.type != cudaMemoryTypeDevice &&
                           at.type != cudaMemoryTypeManaged))
    return fail(FS_ERR_INVALID, "src must be pinned host memory or device memory");
  e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  e = fs::launch_copy_in(dst, src, bytes, ctx->pdl_w && ctx->pdl, at.type == cudaMemoryTypeHost,
                         static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FS_OK : cuda_fail(e, "copy kernel launch");
}

fs_status fs_read_probe(const void* src, size_t bytes, unsigned long long* sink, int grid, void* stream) {
  if (bytes == 0) return FS_OK;
  if (!src || !sink) return fail(FS_ERR_INVALID, "src and sink are required");
  if ((reinterpret_cast<uintptr_t>(src) & 15u) || (bytes & 15u))
    return fail(FS_ERR_INVALID, "src and bytes must be 16-byte aligned");
  if (grid <= 0) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&grid, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_fail(e, "SM count");
    grid *= 2;                                  // two CTAs (rings) per SM
  }
  cudaError_t e = fs::launch_read_probe(src, bytes, sink, grid, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FS_OK : cuda_fail(e, "read probe launch");
}

fs_status fs_gumbel_from_bits(const uint32_t* r, float* g_out, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!r || !g_out))) return fail(FS_ERR_INVALID, "r, g_out required");
  cudaError_t e = fs::launch_gumbel(r, g_out, n, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FS_OK : cuda_fail(e, "gumbel launch");
}

}  // extern "C"
