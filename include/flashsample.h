/*
 * flashsample.h -- C ABI of the B200-native FlashSampling hot path
 * (arXiv 2603.15854, "FlashSampling: exact sampling fused into the LM-head matmul").
 *
 * The library computes, for every batch row b, one exact sample of
 *     Cat(softmax(l~_b)),   l~_{b,v} = transform( sum_d h[b,d] * W[v,d] )
 * as  idx_b = argmax_v ( l~_{b,v} + g_{b,v} ),  g ~ Gumbel(0,1)
 * (Gumbel-Max theorem; fused two-stage Alg. 2), with the
 * [B,V] logits never written to HBM.  "P:n" = line n of PAPER.md.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  Layout      h [B,D] row-major, W [V,D] row-major (nn.Linear weight), both K(=D)-major.
 *              bf16 (FS_BF16) or fp32 (FS_F32).  fp32 is computed with true fp32 FMA on
 *              CUDA cores (never TF32); bf16 on tcgen05 tensor cores with fp32 accumulation
 *              (P:199-202).
 *  Transform   l~ = (acc + bias[v]) * (1/temperature[b]); mask bit 0 -> -inf; NaN -> -inf
 *              (Alg. 2 line 9 P:169, masking §4.6; order = DESIGN.md reading R3).
 *              bias      [V] fp32 or NULL (= 0)
 *              temperature [B] fp32 or NULL (= 1); a row with tau <= 0 or non-finite is undefined
 *              mask      [B][mask_words] uint32, bit (v & 31) of word (v >> 5) = 1 -> token v allowed;
 *                        NULL = all allowed.  mask_words = ceil(V_total/32); ids are GLOBAL ids.
 *  RNG         Philox4x32-10, key = (seed lo, seed hi), counter = (v_global, b>>2, step lo,
 *              (step hi & 0xFFFFFF) | tag<<24), r = out[b & 3]; u = (r+1)/(2^32+1);
 *              g = -log(-log u) evaluated tail-accurately in fp32 (App. C P:849-853;
 *              DESIGN.md readings R1, R2).  Results are a deterministic function of
 *              (inputs, seed, step): independent of tiling, grid, shard count or stream.
 *  Ties        equal perturbed scores resolve to the smallest global vocabulary id (reading R5).
 *  Undefined   a row with no finite l~ (all masked, or invalid tau) yields idx = -1,
 *              score = -inf, log-mass = -inf ("undefined"; reading R7).  Never an error.
 *  Indices     0-based global vocabulary ids (int32).
 *  Memory      every pointer argument except ctx is a DEVICE pointer owned by the caller,
 *              16-byte aligned for h and W; the library never frees or retains them after the
 *              call returns.  The library owns only fs_ctx (workspace, tensor-map cache).
 *  Streams     `stream` is a cudaStream_t (NULL = legacy default stream).  All calls are
 *              asynchronous on it, perform no host synchronisation and, once the workspace has
 *              grown for a shape, no allocation: they are CUDA-graph capturable.
 *  Errors      synchronous status for anything checkable on the host (fs_status); the
 *              message of the last failure on the calling thread is fs_last_error().
 *  Limits      1 <= B (rows are processed in chunks of at most 256 per launch),
 *              1 <= D, 1 <= V < 2^31, bf16 tensor-core path needs D % 8 == 0 (TMA row stride);
 *              other D fall back to the CUDA-core kernel (same results, slower).
 */
#ifndef FLASHSAMPLE_H
#define FLASHSAMPLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FS_OK = 0,
  FS_ERR_INVALID = 1,      /* bad argument (NULL required pointer, size < 1, misalignment, ...) */
  FS_ERR_UNSUPPORTED = 2,  /* valid but not supported by this build (e.g. no sm_100 device)    */
  FS_ERR_CUDA = 3,         /* a CUDA runtime / driver call failed (message in fs_last_error)   */
  FS_ERR_OOM = 4,          /* workspace allocation failed                                      */
  FS_ERR_NCCL = 5          /* an NCCL call or the communicator failed (fs_comm_init / fs_sample_tp) */
} fs_status;

typedef enum { FS_BF16 = 0, FS_F32 = 1 } fs_dtype;

/* Group / shard summary (Lemma "max-stability"; Alg. A.4 message P:830):
 *   max_score = M_k = max_{v in G_k} (l~_v + g_v)     (-inf if the group has no finite l~)
 *   idx       = I_k = smallest global id attaining M_k (-1 if empty)
 *   log_mass  = L_k = log sum_{v in G_k} exp(l~_v)   (-inf if empty)              12 bytes. */
typedef struct {
  float max_score;
  int32_t idx;
  float log_mass;
} fs_summary;

typedef struct fs_ctx fs_ctx;

/* Version string of the library build. */
const char* fs_version(void);
const char* fs_status_str(fs_status s);
/* Message of the last failing call on this thread ("" if none). */
const char* fs_last_error(void);

/* Create a context bound to CUDA device `device` (workspace, tensor-map cache, SM count).
 * Fails with FS_ERR_UNSUPPORTED if the device is not compute capability 10.0 (B200).
 * A context owns one workspace (candidate buffers, the finalize maxima / counter, top-k lists):
 * calls on one context must be ordered -- one stream at a time, or streams ordered by events.
 * Use one context per concurrently sampling stream (the Python binding keys contexts by
 * (device, stream)).  Host-side context state is guarded by a lock, so concurrent calls from
 * several host threads are safe as long as each uses its own context (or serialises its streams). */
fs_status fs_ctx_create(int device, fs_ctx** out);
void fs_ctx_destroy(fs_ctx* ctx);
/* Options (name, value); unknown names -> FS_ERR_INVALID.
 *   "fuse_reduce" (default 1): plain sampling (single group, no logZ / log-prob outputs) ends in
 *       the stage-1 kernel: every CTA folds its candidate per row into a 64-bit atomicMax of
 *       (order key << 32 | ~idx) in the context's workspace, and the last CTA to finish writes
 *       idx_out / score_out (Alg. 2 stage 2, done in L2 instead of a second kernel).
 *       Also: fs_sample_logits (B <= 256, no log-mass) ends in its last block; single-group calls
 *       with log-mass outputs (logZ / log-prob / a TP shard summary) with B <= 16 run the
 *       stage-2 row reduce in the last stage-1 CTA.  0 = separate stage-2 reduce kernels.  Same
 *       results bit for bit.
 *   "pdl_w" (default 0): launch stage 1 with programmatic dependent launch.  The kernel then starts
 *       while the preceding kernel on the stream finishes and streams its first W tiles BEFORE
 *       waiting for it; every other input (h, bias, temperature, mask, seeds, steps) is read and
 *       every output written only after the wait.  Contract: W must not be written by the kernel
 *       immediately preceding the call on the same stream (LM-head weights are read-only while
 *       decoding).  Saves the launch gap and the pipeline fill of back-to-back decode steps.
 *       1 = only for batch chunks of at most "pdl_w_max_b" rows (default 128: larger batches are
 *       tensor/power-bound and two overlapping steps only share the power budget); 2 = always.
 *   "done_flag" (default 0): address of a pinned host uint64 (cudaHostAlloc / pinned torch tensor).
 *       The one-kernel finalize (fuse_reduce paths, incl. fs_sample_staged) stores 1 into it with a
 *       system-scope release after every output of the call is written, so a serving loop can spin
 *       on host memory (reset it to 0 before the call) instead of synchronising the stream.  Per
 *       context: give the waiting loop a context of its own.  0 = off.
 *   "whole_tiles" (default 1): single-group calls on the tensor-core kernels cut the vocabulary into
 *       whole tiles (128 rows, 256 per CTA pair) and run on the fewest CTAs (pairs) that still need
 *       only P = ceil(tiles / #SMs) tile passes, each CTA taking P or P-1 full tiles (V = 152,064:
 *       132 CTAs x 9 tiles instead of 148 CTAs with partial tiles).  Ignored when "max_ctas" or
 *       "unit_rows" is set.  0 = 16-row CTA ranges on every SM.  Same results bit for bit.
 *   Tuning / testing: "force_simt" (1 = CUDA-core kernel), "max_ctas" (cap the persistent grid,
 *   0 = number of SMs), "pdl" (stage 1 -> stage 2 programmatic launch, default 1), "pair" (CTA-pair
 *   kernel: -1 auto, 0 off, 1 on), "stages", "kbps", "unit_rows", "l2promo", "w_policy",
 *   "topk_mode", "topk_spans" (fused top-k raw-logit route: 1 span maxima + gather, 0 chunk
 *   selection), "grp_ranges" (grouped stage 2: 1 host slot ranges, 0 device search), "grp_kernel"
 *   (grouped stage 2: 0 auto, 1 warp per (row, group), 3 block per row), "spin_wait" (1 = epilogue
 *   barrier waits without the suspend-time hint), "time_stage1" (below); debug: "dbg_no_mma",
 *   "dbg_no_epi" (results are garbage), "dbg_times" (device pointer to [grid][8] u64 per-CTA
 *   timestamps, tools/cta_timeline.py; 0 = off). */
fs_status fs_ctx_set_option(fs_ctx* ctx, const char* name, int64_t value);
/* Measurement hook (used by bench.py for the roofline figure).  With option "time_stage1" = 1
 * every call records a CUDA event pair around each stage-1 (fused kernel) launch on the call's
 * stream (PDL between stage 1 and stage 2 is disabled while timing).  fs_ctx_query(ctx,
 * "stage1_ms", &out) waits for the recorded events, returns the summed stage-1 milliseconds and
 * resets the record; "stage1_launches" returns the number of recorded launches (before a
 * "stage1_ms" query resets it).  Other queries: "num_sms"; "nccl_world" (fs_comm_init's world, 0 = no
 * communicator); "comm_timeouts" (f2 exchange waits that
 * gave up); "staging_timeouts" (fs_sample_staged grid barriers that gave up, see there);
 * "staged_fallbacks" (fs_sample_staged calls staged by the copy kernel because the grid could not
 * be co-resident).  Unknown names -> FS_ERR_INVALID. */
fs_status fs_ctx_query(fs_ctx* ctx, const char* name, double* out);

/* fs_sample -- fused LM-head projection + exact Gumbel-max sampling (Alg. 2).
 *   h [B,D], W [V,D] (dtype), bias/temperature/mask as above (mask_words = ceil(V/32)).
 *   idx_out   [B] int32 (required): sampled global vocabulary id, -1 for undefined rows.
 *   score_out [B] fp32 or NULL: the winning perturbed score max_v (l~_v + g_v).
 * Workload per call: W is streamed from HBM exactly once; besides the outputs only B 64-bit
 * atomics per CTA (one-kernel finalize) or per-CTA candidates (B x #CTA x 16 bytes) are written. */
fs_status fs_sample(fs_ctx* ctx, fs_dtype dtype,
                    const void* h, const void* W,
                    const float* bias, const float* temperature, const uint32_t* mask,
                    uint64_t seed, uint64_t step, int B, int D, int V,
                    int32_t* idx_out, float* score_out, void* stream);

/* fs_sample_staged -- fs_sample for a serving loop whose hidden states arrive in host memory:
 * h_host [B,D] is pinned (page-locked) host memory, 16-byte aligned; h_dev is a device buffer of
 * the same size that the call overwrites.  On the one-kernel tcgen05 path (bf16, D % 8 == 0,
 * option "fuse_reduce" on) the sampling kernel stages h itself: every CTA copies its slice of
 * h_host into h_dev over PCIe after the dependency wait, a grid-wide counter orders the slices
 * before the first h load, and W streaming starts meanwhile -- no copy kernel, no copy engine.
 * Otherwise fs_copy_async stages h before fs_sample.  The grid barrier needs all persistent CTAs
 * co-resident: the call checks the occupancy of the exact kernel configuration (and "max_ctas"
 * against the SM count) and stages with the copy kernel instead when the grid cannot fit
 * (query "staged_fallbacks").  Should the CTAs still not be co-resident at run time (a GPU shared
 * through MPS or green contexts), the barrier gives up after ~5 s: the call completes, every row
 * is reported undefined (idx -1, score -inf) and "staging_timeouts" counts it -- no trap, no
 * sticky CUDA error.  idx_out / score_out may also be pinned host memory (see fs_copy_async).
 * Results equal fs_sample on the same h. */
fs_status fs_sample_staged(fs_ctx* ctx, fs_dtype dtype, const void* h_host, void* h_dev, const void* W,
                           const float* bias, const float* temperature, const uint32_t* mask, uint64_t seed,
                           uint64_t step, int B, int D, int V, int32_t* idx_out, float* score_out, void* stream);

/* fs_sample_grouped -- grouped / online FlashSampling with per-group log-mass summaries
 * (Group-Gumbel-Max §4.1, Alg. A.2/A.3 P:768-815, log-normalizer App. E).
 * Groups are contiguous vocabulary ranges G_k = [k*g, min((k+1)*g, V)), k = 0..ceil(V/g)-1,
 * g = group_size, a multiple of 128 (last group ragged).  The outer selection reuses the
 * group maxima (reading R8), so idx_out equals fs_sample's idx_out exactly.
 *   logZ_out   [B] fp32 or NULL: log sum_v exp(l~_v) = logsumexp_k L_k.
 *   logprob_out [B] fp32 or NULL: log p(idx) = l~_idx - logZ.
 *   groups_out [B][ceil(V/g)] fs_summary or NULL.  group_size >= V gives one group (plain
 *   sampling with logZ / log-probabilities). */
fs_status fs_sample_grouped(fs_ctx* ctx, fs_dtype dtype,
                            const void* h, const void* W,
                            const float* bias, const float* temperature, const uint32_t* mask,
                            uint64_t seed, uint64_t step, int B, int D, int V, int group_size,
                            int32_t* idx_out, float* score_out, float* logZ_out, float* logprob_out,
                            fs_summary* groups_out, void* stream);

/* fs_sample_logits -- standalone FlashSampling over MATERIALISED logits (§5.2; Alg. A.1
 * P:747-763 parallelised as in Alg. 2): same transform, RNG layout, tie rule and outputs as
 * fs_sample, for callers that already hold logits (the rival of FlashInfer's
 * sampling_from_logits).  fs_sample_logits(h W^T) equals fs_sample(h, W) up to the rounding of
 * the logits themselves.
 *   logits [B][ld] (dtype bf16 or fp32, row stride ld >= V elements), bias/temperature/mask as above.
 *   idx_out [B] required; score_out, logZ_out, logprob_out [B] fp32 or NULL, where
 *   logprob = l~_idx - logZ = log p(idx) (App. E). */
fs_status fs_sample_logits(fs_ctx* ctx, fs_dtype dtype, const void* logits, int64_t ld,
                           const float* bias, const float* temperature, const uint32_t* mask,
                           uint64_t seed, uint64_t step, int B, int V,
                           int32_t* idx_out, float* score_out, float* logZ_out, float* logprob_out,
                           void* stream);

/* Extended arguments for fs_sample_ex / fs_sample_logits_ex.
 *   seeds [B] uint64 (device) or NULL: per-request RNG streams, batch-position invariant
 *         (reading R18: key = seeds[b], counter = (v >> 2, 2^31, steps[b]), word v & 3);
 *         NULL -> the shared stream (seed, step) of the convention above.
 *   steps [B] uint64 (device) or NULL: per-request step counters (NULL -> `step` for every row).
 *   Greedy rows: temperature[b] == 0 exactly -> argmax of l + bias without noise (R18).
 *   group_size: fs_sample_ex only; 0 -> one group over V (grouped outputs when > 0). */
typedef struct {
  const float* bias;
  const float* temperature;
  const uint32_t* mask;
  uint64_t seed;
  uint64_t step;
  const uint64_t* seeds;
  const uint64_t* steps;
  int group_size;
  int32_t* idx_out;          /* [B] required */
  float* score_out;          /* [B] or NULL */
  float* logZ_out;           /* [B] or NULL */
  float* logprob_out;        /* [B] or NULL */
  fs_summary* groups_out;    /* [B][ceil(V/group_size)] or NULL (group_size > 0) */
  int top_k;                 /* 1..1024 keeps the k largest l~ (R19); <= 0 off */
  float top_p;               /* nucleus on the top-k survivors, (0,1); outside off */
} fs_sample_args;

/* fs_sample_ex -- fs_sample / fs_sample_grouped with per-request streams, greedy rows and every
 * optional output selected through `args` (same kernels, same conventions).
 * With top_k / top_p ("each tile computes top-k candidates locally,
 * a second stage reduces all per-tile candidates into a global top-k"; reading R19): the same
 * truncated distribution as fs_sample_logits_ex, through the LM head.  Stage 1 keeps the k best
 * (l~, id) per (row, CTA) in the epilogue's shared memory (logits never reach HBM); when those
 * lists do not fit (large B x k) it writes the fp32 logits to the context workspace instead
 * (B x V x 4 bytes) and the chunked selection of fs_sample_logits_ex runs on them -- same
 * accumulator, same transform, same token.  FS_ERR_UNSUPPORTED with grouped outputs
 * (group_size < V or groups_out). */
fs_status fs_sample_ex(fs_ctx* ctx, fs_dtype dtype, const void* h, const void* W, int B, int D, int V,
                       const fs_sample_args* args, void* stream);
/* fs_sample_logits_ex -- fs_sample_logits with `args` (group_size and groups_out ignored).
 * Top-k / top-p (reading R19): with top_k in 1..1024 (required when
 * 0 < top_p < 1) the sample is drawn exactly from softmax(l~) restricted to the k largest l~
 * (ties -> smaller id) and then to the shortest prefix of those whose probability mass reaches
 * top_p; logZ_out / logprob_out then refer to that truncated distribution.  Per-chunk top-k
 * selection (block radix select) + per-row merge, top-p and Gumbel-max over the survivors. */
fs_status fs_sample_logits_ex(fs_ctx* ctx, fs_dtype dtype, const void* logits, int64_t ld, int B, int V,
                              const fs_sample_args* args, void* stream);

/* fs_sample_shard -- the rank-local half of distributed FlashSampling for a vocabulary-
 * sharded (tensor-parallel) LM head (§4.2, Alg. A.4).
 *   W_shard [V_local,D] holds global rows [vocab_offset, vocab_offset+V_local);
 *   bias_shard [V_local] or NULL; mask is the GLOBAL bitmask [B][ceil(V_total/32)] or NULL;
 *   the RNG is keyed by global ids, so the union of shards reproduces fs_sample on the
 *   full matrix bit-for-bit.
 *   summary_out [B] fs_summary (required): this shard's (M, I, L) per row -- the 12-byte
 *   message every rank contributes to the all-gather. */
fs_status fs_sample_shard(fs_ctx* ctx, fs_dtype dtype,
                          const void* h, const void* W_shard,
                          const float* bias_shard, const float* temperature, const uint32_t* mask,
                          uint64_t seed, uint64_t step, int B, int D, int V_local,
                          int64_t vocab_offset, int64_t V_total,
                          fs_summary* summary_out, void* stream);

/* fs_combine_summaries -- outer selection over n gathered shard/group summaries
 * (Alg. A.4 lines 5-7, with max reuse P:286): for each row,
 *   idx = I_{k*}, k* = argmax_k M_k (ties -> smaller global id), score = M_{k*},
 *   logZ = logsumexp_k L_k.
 *   gathered [n][B] fs_summary (device); idx_out [B] required; score_out, logZ_out optional. */
fs_status fs_combine_summaries(const fs_summary* gathered, int n, int B,
                               int32_t* idx_out, float* score_out, float* logZ_out,
                               void* stream);

/* ---- Peer-memory exchange for vocabulary-sharded sampling -------------------
 * P:830 lets the coordinator gather the shard summaries by "an all-gather ... or an equivalent
 * reduction".  Instead of a collective call, every rank PUSHES its B x 12-byte records straight
 * into every peer's exchange window (CUDA IPC mapping; NVLink/NVSwitch stores between GPUs) and
 * raises a per-step flag; each rank then waits for the n flags of the step and runs the outer
 * selection on its local copy -- one kernel after stage 2, no NCCL launch, no host round trip.
 *   Window of a rank (device memory owned by its context): records [2 parities][world][B_max]
 *   fs_summary, flags [2][world] uint64 (the epoch that filled the slot), acks [world] uint64
 *   (the last epoch each reader consumed, so a writer never overwrites a parity slot that is
 *   still unread).  Ordering: records, then fence.sys, then the flag (release); readers
 *   acquire the flags before reading the records.
 * fs_comm_window_create: allocate and zero this rank's window for <= B_max rows (one window per
 *   context; replaces a previous one), return its IPC handle (64 opaque bytes) for the caller to
 *   all-gather by any host transport (torch.distributed, gloo).  world <= 16.
 * fs_comm_window_open: map the peers' windows from the gathered handles [world] (entry `rank`
 *   is ignored).  Peers may be other GPUs (peer access over NVLink) or the same GPU.
 * fs_sample_tp_push: fs_sample_shard + push + wait + fs_combine_summaries in stream order;
 *   every rank gets the identical idx_out (score_out, logZ_out optional).  Without logZ_out (B <= 256,
 *   bf16 tcgen05 path): ONE kernel per rank -- the shard sampler's finalizing CTA stores the records
 *   into every peer window, releases its flags, waits for the n ranks' records, runs the outer
 *   selection and acknowledges the epoch.  With logZ_out (B <= 256) the push is fused into the
 *   shard sampler's log-mass reduction step (the finalizing stage-1 CTA for B <= 16, else the
 *   stage-2 row reduce) and one PDL-chained single-block kernel waits for the n flags and combines.
 *   Larger B push from a separate kernel.  All ranks must call it the same number of times (the
 *   step epoch is a per-context counter).  A peer that does not arrive within ~10 s makes the wait
 *   give up: idx_out = -1 and fs_ctx_query("comm_timeouts") counts it.
 * fs_comm_window_destroy: unmap the peers and free the window. */
typedef struct { unsigned char bytes[64]; } fs_ipc_handle;
fs_status fs_comm_window_create(fs_ctx* ctx, int world, int rank, int B_max, fs_ipc_handle* handle_out);
fs_status fs_comm_window_open(fs_ctx* ctx, const fs_ipc_handle* handles);
fs_status fs_sample_tp_push(fs_ctx* ctx, fs_dtype dtype, const void* h, const void* W_shard,
                            const float* bias_shard, const float* temperature, const uint32_t* mask,
                            uint64_t seed, uint64_t step, int B, int D, int V_local,
                            int64_t vocab_offset, int64_t V_total,
                            int32_t* idx_out, float* score_out, float* logZ_out, void* stream);
fs_status fs_comm_window_destroy(fs_ctx* ctx);

/* ---- NCCL-backed vocabulary-sharded sampling (§4.2; Alg. A.4) ----------------
 * The NCCL form of the exchange: Alg. A.4 line 4 "all-gather the per-shard summaries".
 * The library resolves NCCL at run time from the process (torch.distributed's libnccl.so.2) or
 * $FS_NCCL_LIB; without NCCL these calls return FS_ERR_UNSUPPORTED and nothing else is affected.
 * fs_comm_unique_id: write a fresh ncclUniqueId (128 opaque bytes) to id_out -- on ONE rank; the
 *   caller broadcasts it to the others by any host transport (e.g. torch.distributed).
 * fs_comm_init: create this context's NCCL communicator (collective over the `world` ranks, each
 *   with its own context on its own GPU; blocks until all ranks joined).  Replaces a previous one.
 * fs_sample_tp: one sharded decode step on the caller's stream, all inside the library:
 *   fs_sample_shard(W_shard) -> this rank's [B] summaries (M, I, L)
 *   -> ncclAllGather of the B x 12-byte records into [world][B] (context workspace)
 *   -> outer selection (fs_combine_summaries): idx_out [B] identical on every rank, equal to
 *      fs_sample on the unsharded W (global ids; reading R8 max reuse), score_out / logZ_out
 *      optional, per_rank_out [world][B] fs_summary (device) or NULL: the gathered records.
 *   Without logZ_out and per_rank_out only (M, I) of the records are consumed: the shard then runs
 *   the plain epilogue and its last CTA writes the records directly (L unused), so no log-mass
 *   epilogue and no stage-2 kernel run.
 *   Arguments as fs_sample_shard.  Asynchronous; FS_ERR_NCCL when the collective cannot be
 *   enqueued or the communicator reports an asynchronous error (ncclCommGetAsyncError, checked
 *   at every call).
 * fs_comm_destroy: release the communicator (also done by fs_ctx_destroy). */
fs_status fs_comm_unique_id(void* id_out);
fs_status fs_comm_init(fs_ctx* ctx, const void* nccl_unique_id, int world, int rank);
fs_status fs_sample_tp(fs_ctx* ctx, fs_dtype dtype, const void* h, const void* W_shard, const float* bias_shard,
                       const float* temperature, const uint32_t* mask, uint64_t seed, uint64_t step, int B, int D,
                       int V_local, int64_t vocab_offset, int64_t V_total, int32_t* idx_out, float* score_out,
                       float* logZ_out, fs_summary* per_rank_out, void* stream);
fs_status fs_comm_destroy(fs_ctx* ctx);

/* fs_merge_summaries -- online binary merge of two summaries of disjoint vocabulary sets
 * (Alg. A.3, Lemma "binary merge" P:315-349, realised by max reuse):
 *   out.max_score = max, out.idx = idx of the max (ties -> smaller id),
 *   out.log_mass = logaddexp(a.log_mass, b.log_mass).  Associative and commutative.
 *   a, b, out: [count] device arrays (out may alias a or b). */
fs_status fs_merge_summaries(const fs_summary* a, const fs_summary* b, fs_summary* out,
                             int count, void* stream);

/* fs_copy_async -- stage one step's inputs for the end-to-end path (a serving loop's
 * host -> device copy of h [, temperature, mask]).  A kernel on `stream` copies `bytes` from
 * `src` (pinned host memory, read over PCIe through its unified address, or device memory) to
 * device memory `dst`; both 16-byte aligned.  With option "pdl_w" it is launched with
 * programmatic dependent launch: it stores dst only after the preceding kernel on the stream
 * completes (that kernel may still be reading dst) and loads a pinned-host src before that wait
 * (a device src, which the preceding kernel may have produced, only after it); the next
 * fs_sample may start streaming W while the copy runs.  Asynchronous; the caller keeps src alive and
 * unchanged until the stream passes the copy.  FS_ERR_INVALID: NULL / misaligned pointers or a
 * pageable (unregistered) host src.
 * fs_sample writes idx_out / score_out with plain stores, so they may also point to pinned host
 * memory (a device -> host write of B x 4 bytes from the last CTA, no separate copy). */
fs_status fs_copy_async(fs_ctx* ctx, void* dst, const void* src, size_t bytes, void* stream);

/* Diagnostics (used by the tests to pin the device RNG; not on the hot path).
 * fs_random_bits: r[i] = Philox draw for (b[i], v[i]) under (seed, step, tag) -- the exact
 *                 counter layout of the convention above.  All arrays device, length n.
 * fs_gumbel_from_bits: g[i] = device fp32 G32(r[i]). */
fs_status fs_random_bits(uint64_t seed, uint64_t step, uint32_t tag,
                         const int32_t* b, const int64_t* v, uint32_t* r_out, int64_t n,
                         void* stream);
fs_status fs_gumbel_from_bits(const uint32_t* r, float* g_out, int64_t n, void* stream);

/* Read-only HBM roofline probe (a measured read-only peak next to the copy peak, which
 * counts read + write traffic).  `grid` CTAs (<= 0: two per SM) each stream a contiguous slice of the
 * device buffer src[0, bytes) through a shared-memory ring with 1-D bulk copies (the TMA engine the
 * sampling kernels stream W with); the first 8 bytes of every 16 KB chunk of a slice (chunks counted
 * from the slice start, slice = ceil(bytes / grid) rounded up to 16 bytes) are XOR-folded into *sink
 * (device, atomicXor), so no load is dead.  bench.py times it over 1 GiB.  FS_ERR_INVALID: NULL
 * pointers, src or bytes not 16-byte aligned.  Asynchronous on `stream`. */
fs_status fs_read_probe(const void* src, size_t bytes, unsigned long long* sink, int grid, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FLASHSAMPLE_H */
