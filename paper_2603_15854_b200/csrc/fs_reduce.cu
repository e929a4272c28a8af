// fs_reduce.cu -- stage 2 of FlashSampling and the summary kernels.
//
//  reduce   Alg. 2 stage 2: per row, argmax over the per-CTA candidates
//           (ties -> smaller id); in grouped mode first merges the candidates of each group into
//           (M_k, I_k, L_k) (§4.1, Lemma P:254-270) and selects by max reuse.
//           Launched with programmatic dependent launch so its prologue overlaps stage 1.
//  combine  Alg. A.4 outer selection over gathered shard summaries.
//  merge    Alg. A.3 online binary merge of two summaries, by max reuse.
#include <cuda_runtime.h>

#include <algorithm>

#include "fs_device.cuh"
#include "fs_epilogue.cuh"
#include "fs_kernels.h"
#include "fs_sm100.cuh"

namespace fs {

__device__ __forceinline__ State from_summary(const fs_summary& m) {
  State s = state_empty();
  if (m.idx >= 0 && !(m.max_score == -INFINITY)) {
    s.key = order_key(m.max_score);
    s.idx = m.idx;
    s.S = (m.log_mass > -INFINITY) ? expf(m.log_mass - m.max_score) : 0.0f;
  }
  return s;
}

constexpr int kReduceThreads = 256;

// Single group (Alg. 2 stage 2; or one TP shard's summary): one warp per batch row,
// each lane merges slots lane, lane+32, ... (independent loads in flight), then a fixed
// shuffle tree -- deterministic, so logZ is bit-reproducible.
// With push.peers (f2, a TP shard step) every row's record is also stored into the peers'
// exchange windows; the last block to finish (counter push.ctr) releases this rank's flags.
__global__ void __launch_bounds__(128)
reduce_rows_kernel(const State* __restrict__ part, const int* __restrict__ part_group, int n_slots, int B,
                   int32_t* idx_out, float* score_out, float* logZ_out, fs_summary* groups_out,
                   float* logprob_out, PushCtx push) {
  sm100::pdl_wait();                       // stage-1 results are visible past this point
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * 4 + (threadIdx.x >> 5);
  const bool pushing = push.peers != nullptr;
  if (pushing) {                           // readers are done with this parity slot
    push_wait_readers(push, threadIdx.x);
    __syncthreads();
  }
  if (b < B)
    reduce_row(part, part_group, n_slots, B, b, lane, idx_out, score_out, logZ_out, groups_out, logprob_out,
               pushing ? &push : nullptr);
  if (pushing) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(push.ctr, 1u) == gridDim.x - 1) {
      push_release(push);                  // every block's records are visible (fence + counter)
      atomicExch(push.ctr, 0u);
    }
  }
}

// Grouped variant (§4.1, App. E): one block per batch row, one thread per group.  Slots are
// ordered by (unit, segment, warp), so their group ids are non-decreasing: group k's candidates are
// the contiguous slot range [lower_bound(k), upper_bound(k)), found by binary search over the
// group ids staged in shared memory; its loads are issued in batches of 8 independent loads.
__device__ __forceinline__ int lower_bound_smem(const int* a, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ State shfl_xor_state(const State& a, int o) {
  State r;
  r.key = __shfl_xor_sync(0xFFFFFFFFu, a.key, o);
  r.idx = __shfl_xor_sync(0xFFFFFFFFu, a.idx, o);
  r.S = __shfl_xor_sync(0xFFFFFFFFu, a.S, o);
  r.lt = __shfl_xor_sync(0xFFFFFFFFu, a.lt, o);
  return r;
}

__global__ void __launch_bounds__(kReduceThreads)
reduce_groups_kernel(const State* __restrict__ part, const int* __restrict__ part_group, int n_slots, int B,
                     int n_groups, int32_t* idx_out, float* score_out, float* logZ_out, fs_summary* groups_out,
                     float* logprob_out, const int* __restrict__ grp_lo) {
  extern __shared__ int sg[];
  __shared__ State red[kReduceThreads];
  sm100::pdl_wait();
  const int b = blockIdx.x, tid = threadIdx.x;
  if (!grp_lo) {                               // no precomputed ranges: stage the ids, binary search
    for (int s = tid; s < n_slots; s += kReduceThreads) sg[s] = part_group[s];
    __syncthreads();
  }
  // 8 threads per group: thread `sub` merges slots lo+sub, lo+sub+8, ... (one batch of
  // independent loads), then a fixed xor-shuffle tree combines the 8 partial states.
  const int sub = tid & 7;
  State acc = state_empty();
  for (int k0 = 0; k0 < n_groups; k0 += kReduceThreads / 8) {
    const int k = k0 + (tid >> 3);
    State g = state_empty();
    if (k < n_groups) {
      const int lo = grp_lo ? grp_lo[k] : lower_bound_smem(sg, n_slots, k);
      const int hi = grp_lo ? grp_lo[k + 1] : lower_bound_smem(sg, n_slots, k + 1);
      for (int s0 = lo + sub; s0 < hi; s0 += 64) {
        State v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (s0 + 8 * i < hi) v[i] = part[(size_t)(s0 + 8 * i) * B + b];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (s0 + 8 * i < hi) g = state_merge(g, v[i]);
      }
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const State other = shfl_xor_state(g, o);
      g = (sub & o) ? state_merge(other, g) : state_merge(g, other);
    }
    if (sub == 0 && k < n_groups) {
      if (groups_out) groups_out[(size_t)b * n_groups + k] = to_summary(g);
      acc = state_merge(acc, g);
    }
  }
  red[tid] = acc;
  __syncthreads();
  for (int w = kReduceThreads / 2; w > 0; w >>= 1) {
    if (tid < w) red[tid] = state_merge(red[tid], red[tid + w]);
    __syncthreads();
  }
  if (tid == 0) {
    const fs_summary f = to_summary(red[0]);
    if (idx_out) idx_out[b] = f.idx;
    if (score_out) score_out[b] = f.max_score;
    if (logZ_out) logZ_out[b] = f.log_mass;
    if (logprob_out) logprob_out[b] = logprob_of(red[0]);
  }
}

// Grouped stage 2 with host-computed group slot ranges: one warp per (row, group) -- lane L merges
// the group's slots L, L+32, ... then a fixed xor tree -> (M_k, I_k, L_k); the group state goes to
// scratch and the last warp of the row (per-row counter, threadFence pattern) merges the row's
// n_groups states in group order (deterministic) into idx / score / logZ / log-prob.
__global__ void __launch_bounds__(256)
reduce_groups_warp_kernel(const State* __restrict__ part, int B, int n_groups, const int* __restrict__ grp_lo,
                          State* gstate, int* row_ctr, int32_t* idx_out, float* score_out, float* logZ_out,
                          fs_summary* groups_out, float* logprob_out) {
  sm100::pdl_wait();
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * 8 + (threadIdx.x >> 5), b = blockIdx.y;
  if (k >= n_groups) return;
  const int lo = grp_lo[k], hi = grp_lo[k + 1];
  State g = state_empty();
#pragma unroll 4
  for (int s = lo + lane; s < hi; s += 32) g = state_merge(g, part[(size_t)s * B + b]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const State other = shfl_xor_state(g, o);
    g = (lane & o) ? state_merge(other, g) : state_merge(g, other);
  }
  int last = 0;
  if (lane == 0) {
    if (groups_out) groups_out[(size_t)b * n_groups + k] = to_summary(g);
    gstate[(size_t)b * n_groups + k] = g;
    __threadfence();
    last = atomicAdd(&row_ctr[b], 1) == n_groups - 1;
  }
  last = __shfl_sync(0xFFFFFFFFu, last, 0);
  if (!last) return;
  __threadfence();
  State acc = state_empty();
  for (int kk = lane; kk < n_groups; kk += 32) {
    const uint4 u = __ldcg(reinterpret_cast<const uint4*>(gstate + (size_t)b * n_groups + kk));
    acc = state_merge(acc, State{u.x, (int32_t)u.y, __uint_as_float(u.z), u.w});
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const State other = shfl_xor_state(acc, o);
    acc = (lane & o) ? state_merge(other, acc) : state_merge(acc, other);
  }
  if (lane == 0) {
    const fs_summary f = to_summary(acc);
    if (idx_out) idx_out[b] = f.idx;
    if (score_out) score_out[b] = f.max_score;
    if (logZ_out) logZ_out[b] = f.log_mass;
    if (logprob_out) logprob_out[b] = logprob_of(acc);
    row_ctr[b] = 0;                            // ready for the next call
  }
}

__global__ void combine_kernel(const fs_summary* __restrict__ gathered, int n, int B, int32_t* idx_out,
                               float* score_out, float* logZ_out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  State acc = state_empty();
  for (int k = 0; k < n; ++k) acc = state_merge(acc, from_summary(gathered[(size_t)k * B + b]));
  const fs_summary f = to_summary(acc);
  idx_out[b] = f.idx;
  if (score_out) score_out[b] = f.max_score;
  if (logZ_out) logZ_out[b] = f.log_mass;
}

__global__ void merge_kernel(const fs_summary* a, const fs_summary* b, fs_summary* out, int count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const State s = state_merge(from_summary(a[i]), from_summary(b[i]));
  out[i] = to_summary(s);
}

__global__ void random_bits_kernel(uint64_t seed, uint64_t step, uint32_t tag, const int32_t* b, const int64_t* v,
                                   uint32_t* r, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t bi = (uint32_t)b[i];
  const U4 o = philox4x32_10((uint32_t)v[i], bi >> 2, ctr_step_lo(step), ctr_step_hi(step, tag), (uint32_t)seed,
                             (uint32_t)(seed >> 32));
  const uint32_t w[4] = {o.x, o.y, o.z, o.w};
  r[i] = w[bi & 3];
}

__global__ void gumbel_kernel(const uint32_t* r, float* g, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    g[i] = gumbel32(r[i]);
}

cudaError_t launch_reduce(const State* part, const int* part_group, const SlotLayout& lay, int B, int n_groups,
                          int32_t* idx_out, float* score_out, float* logZ_out, fs_summary* groups_out,
                          cudaStream_t stream, bool pdl, float* logprob_out, const int* grp_lo,
                          State* gscratch, int* row_ctr, const PushCtx* push, int grp_kernel) {
  cudaLaunchConfig_t cfg = {};
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  if (n_groups == 1) {
    cfg.gridDim = dim3((B + 3) / 4);
    cfg.blockDim = dim3(128);
    PushCtx pc{};
    if (push) pc = *push;
    return cudaLaunchKernelEx(&cfg, reduce_rows_kernel, part, part_group, lay.n_slots, B, idx_out, score_out,
                              logZ_out, groups_out, logprob_out, pc);
  }
  // warp per (row, group) up to B = 64, block per row above (ncu, Gemma-3-27B 65 groups: B=1 8.3 vs
  // 10.2 us, B=32 10.8 vs 14.1, B=128 16.5 vs 14.2, B=256 23.5 vs 19.2; profiles/r02/stage2_ncu.csv)
  const bool warp_ok = grp_lo && gscratch && row_ctr && B <= 256;
  if (grp_kernel == 0) grp_kernel = (warp_ok && B <= 64) ? 1 : 3;
  if (grp_kernel == 1 && warp_ok) {
    cfg.gridDim = dim3((n_groups + 7) / 8, B);
    cfg.blockDim = dim3(256);
    return cudaLaunchKernelEx(&cfg, reduce_groups_warp_kernel, part, B, n_groups, grp_lo, gscratch, row_ctr,
                              idx_out, score_out, logZ_out, groups_out, logprob_out);
  }
  cfg.gridDim = dim3(B);
  cfg.blockDim = dim3(kReduceThreads);
  cfg.dynamicSmemBytes = grp_lo ? 0 : (size_t)lay.n_slots * sizeof(int);
  if (cfg.dynamicSmemBytes > 40 * 1024) {      // per call: the size varies with the slot count
    cudaError_t e = cudaFuncSetAttribute(reduce_groups_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)cfg.dynamicSmemBytes);
    if (e != cudaSuccess) return e;
  }
  return cudaLaunchKernelEx(&cfg, reduce_groups_kernel, part, part_group, lay.n_slots, B, n_groups, idx_out,
                            score_out, logZ_out, groups_out, logprob_out, grp_lo);
}

// ---------------------------------------------------------------------------------------------
// Peer-memory exchange ("all-gather ... or an equivalent reduction";
// protocol in fs_peer.cuh).  Fused form: the shard sampler's last reduction step already pushed the
// records and released the flags (PushCtx), so one block only (3) acquires the n flags of this
// epoch in the local window, (4) runs the outer selection over the n local records per row, and
// (5) acknowledges the epoch to every peer.  Unfused form (B > 256): the same block first (1)
// waits for the readers of the parity slot and (2) pushes `local` itself.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void wait_combine_ack(const PeerTab& peers, int world, int rank, int B, int B_max,
                                                 uint64_t epoch, int32_t* idx_out, float* score_out,
                                                 float* logZ_out, unsigned* timeouts, int* ok) {
  const int par = (int)(epoch & 1);
  if (threadIdx.x < world)
    if (!wait_flag(peers.flags[rank] + par * world + threadIdx.x, [&](uint64_t v) { return v == epoch; })) *ok = 0;
  __syncthreads();
  const fs_summary* rec = peers.rec[rank] + (size_t)par * world * B_max;
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    State acc = state_empty();
    for (int k = 0; k < world; ++k) acc = state_merge(acc, from_summary(rec[(size_t)k * B_max + b]));
    const fs_summary f = to_summary(acc);
    idx_out[b] = *ok ? f.idx : -1;
    if (score_out) score_out[b] = f.max_score;
    if (logZ_out) logZ_out[b] = f.log_mass;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (!*ok) atomicAdd(timeouts, 1u);
    for (int p = 0; p < world; ++p) st_release_sys(peers.acks[p] + rank, epoch);
  }
}

__global__ void __launch_bounds__(256)
exchange_combine_kernel(const fs_summary* __restrict__ local, PeerTab peers, int world, int rank, int B, int B_max,
                        uint64_t epoch, int32_t* idx_out, float* score_out, float* logZ_out, unsigned* timeouts) {
  __shared__ int ok;
  sm100::pdl_wait();                                   // the shard summaries are complete
  const int par = (int)(epoch & 1);
  if (threadIdx.x == 0) ok = 1;
  __syncthreads();
  const uint64_t prev = epoch >= 2 ? epoch - 2 : 0;
  if (threadIdx.x < world)                            // reader `tid` finished the last use of slot `par`
    if (!wait_flag(peers.acks[rank] + threadIdx.x, [&](uint64_t v) { return v >= prev; })) ok = 0;
  __syncthreads();
  for (int p = 0; p < world; ++p) {
    fs_summary* dst = peers.rec[p] + ((size_t)par * world + rank) * B_max;
    for (int b = threadIdx.x; b < B; b += blockDim.x) dst[b] = local[b];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < world; ++p) st_release_sys(peers.flags[p] + par * world + rank, epoch);
  }
  wait_combine_ack(peers, world, rank, B, B_max, epoch, idx_out, score_out, logZ_out, timeouts, &ok);
}

// Fused form.  Launched with PDL and never waits on the preceding grid: it synchronises with every
// rank's pusher (including this rank's own shard kernel) through the flags alone, and triggers its
// own dependents at once (the next step's W prefetch may start while it waits).
__global__ void __launch_bounds__(256)
exchange_wait_kernel(const PeerTab* __restrict__ peers_dev, int world, int rank, int B, int B_max, uint64_t epoch,
                     int32_t* idx_out, float* score_out, float* logZ_out, unsigned* timeouts) {
  __shared__ int ok;
  __shared__ PeerTab peers;
  sm100::pdl_launch_dependents();
  if (threadIdx.x == 0) ok = 1;
  for (int i = threadIdx.x; i < (int)(sizeof(PeerTab) / 8); i += blockDim.x)
    reinterpret_cast<uint64_t*>(&peers)[i] = reinterpret_cast<const uint64_t*>(peers_dev)[i];
  __syncthreads();
  wait_combine_ack(peers, world, rank, B, B_max, epoch, idx_out, score_out, logZ_out, timeouts, &ok);
}

cudaError_t launch_exchange_combine(const fs_summary* local, const PeerTab& peers, int world, int rank, int B,
                                    int B_max, uint64_t epoch, int32_t* idx_out, float* score_out, float* logZ_out,
                                    unsigned* timeouts, cudaStream_t stream, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.stream = stream;
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(256);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, exchange_combine_kernel, local, peers, world, rank, B, B_max, epoch, idx_out,
                            score_out, logZ_out, timeouts);
}

cudaError_t launch_exchange_wait(const PeerTab* peers_dev, int world, int rank, int B, int B_max, uint64_t epoch,
                                 int32_t* idx_out, float* score_out, float* logZ_out, unsigned* timeouts,
                                 cudaStream_t stream, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.stream = stream;
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(256);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, exchange_wait_kernel, peers_dev, world, rank, B, B_max, epoch, idx_out, score_out,
                            logZ_out, timeouts);
}

cudaError_t launch_combine(const fs_summary* gathered, int n, int B, int32_t* idx_out, float* score_out,
                           float* logZ_out, cudaStream_t stream) {
  combine_kernel<<<(B + 127) / 128, 128, 0, stream>>>(gathered, n, B, idx_out, score_out, logZ_out);
  return cudaGetLastError();
}

cudaError_t launch_merge(const fs_summary* a, const fs_summary* b, fs_summary* out, int count,
                         cudaStream_t stream) {
  merge_kernel<<<(count + 127) / 128, 128, 0, stream>>>(a, b, out, count);
  return cudaGetLastError();
}

cudaError_t launch_random_bits(uint64_t seed, uint64_t step, uint32_t tag, const int32_t* b, const int64_t* v,
                               uint32_t* r, int64_t n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  random_bits_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(seed, step, tag, b, v, r, n);
  return cudaGetLastError();
}

cudaError_t launch_gumbel(const uint32_t* r, float* g, int64_t n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = (n + 255) / 256;
  gumbel_kernel<<<(unsigned)(blocks < 65535 * 16 ? blocks : 65535 * 16), 256, 0, stream>>>(r, g, n);
  return cudaGetLastError();
}

// Input staging for the end-to-end path (fs_copy_async): 16-byte loads of the source (pinned host
// memory through UVA -- a PCIe read -- or device memory) are issued BEFORE the dependency wait, the
// stores to dst only after it (the preceding kernel may still read dst, e.g. last step's h).
// Launched with PDL: it triggers its dependents at once, so the next fused kernel's W prefetch
// overlaps this copy.
constexpr int kCopyThreads = 256;
constexpr int kCopyPerThread = 4;   // 16-byte words per thread per pass
// A device-memory src may be written by the preceding kernel (PDL gives no visibility before the
// wait), so then every load follows the wait; only a pinned host src is read early.
__global__ void __launch_bounds__(kCopyThreads)
copy_in_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, int64_t n16, uint8_t* dst_tail,
               const uint8_t* src_tail, int tail, int src_host) {
  sm100::pdl_launch_dependents();
  if (!src_host) sm100::pdl_wait();
  const int64_t stride = (int64_t)gridDim.x * kCopyThreads;
  int64_t i0 = (int64_t)blockIdx.x * kCopyThreads + threadIdx.x;
  uint4 v[kCopyPerThread];
#pragma unroll
  for (int j = 0; j < kCopyPerThread; ++j)
    if (i0 + j * stride < n16) v[j] = src[i0 + j * stride];
  uint8_t tb = 0;
  if (i0 < tail) tb = src_tail[i0];
  sm100::pdl_wait();
#pragma unroll
  for (int j = 0; j < kCopyPerThread; ++j)
    if (i0 + j * stride < n16) dst[i0 + j * stride] = v[j];
  if (i0 < tail) dst_tail[i0] = tb;
  for (int64_t i = i0 + kCopyPerThread * stride; i < n16; i += stride) dst[i] = src[i];
}

cudaError_t launch_copy_in(void* dst, const void* src, size_t bytes, bool pdl, bool src_host, cudaStream_t stream) {
  const int64_t n16 = (int64_t)(bytes / 16);
  const int tail = (int)(bytes % 16);
  const int64_t per_block = (int64_t)kCopyThreads * kCopyPerThread;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(1024, (n16 + per_block - 1) / per_block));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kCopyThreads);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, copy_in_kernel, static_cast<uint4*>(dst), static_cast<const uint4*>(src), n16,
                            static_cast<uint8_t*>(dst) + n16 * 16, static_cast<const uint8_t*>(src) + n16 * 16, tail,
                            src_host ? 1 : 0);
}

}  // namespace fs
