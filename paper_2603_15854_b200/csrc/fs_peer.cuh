// fs_peer.cuh -- peer-memory exchange of the vocabulary-sharded sampler.
//
// PAPER.md P:830 (Alg. A.4 line 4): the coordinator gathers the per-shard summaries "via an
// all-gather ... or perform an equivalent reduction".  Instead of a collective call, every rank
// stores its B x 12-byte records (M, I, L) straight into every peer's exchange window (CUDA IPC
// mappings: NVLink / NVSwitch stores between GPUs), then releases one flag per (parity, rank);
// every rank acquires the n flags of the step and runs the outer selection (Alg. A.4 lines 5-7)
// on its local copy.
//
// Window of a rank (include/flashsample.h fs_comm_window_create):
//   rec   [2 parities][world][B_max] fs_summary   slot (par, k) holds rank k's records of an epoch
//   flags [2][world] uint64                         epoch that filled slot (par, k)
//   acks  [world] uint64                            last epoch reader k consumed (written by k)
// Ordering: records -> fence.sys -> flag (st.release.sys); readers ld.acquire.sys the flags, read
// the records, then publish their ack to every peer.  A writer waits until every reader acked
// epoch - 2 before overwriting parity slot epoch & 1.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/flashsample.h"

namespace fs {

constexpr int kMaxWorld = 16;

struct PeerTab {                 // the world windows' addresses as mapped in this process
  fs_summary* rec[kMaxWorld];
  uint64_t* flags[kMaxWorld];
  uint64_t* acks[kMaxWorld];
};

// Per-call arguments of the push fused into the shard sampler's last reduction step.
struct PushCtx {
  const PeerTab* peers;          // device copy of the PeerTab (nullptr: no push)
  int world, rank, B_max;
  uint64_t epoch;                // this step's epoch (>= 1); parity slot = epoch & 1
  unsigned* ctr;                 // blocks of the pushing grid that finished (0 between calls)
  unsigned* timeouts;            // incremented when a wait gives up (~10 s)
};

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t peer_globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spin until pred(ld_acquire(p)) or ~10 s; false on timeout.
template <typename Pred>
__device__ __forceinline__ bool wait_flag(const uint64_t* p, Pred pred) {
  const uint64_t t0 = peer_globaltimer();
  uint32_t ns = 32;
  while (!pred(ld_acquire_sys(p))) {
    if (peer_globaltimer() - t0 > 10000000000ull) return false;
    __nanosleep(ns);
    ns = ns < 1024 ? ns * 2 : ns;
  }
  return true;
}

// Writer side, before overwriting parity slot (epoch & 1): thread t < world waits until reader t
// consumed epoch - 2 (its ack in this rank's own window).  Caller synchronises afterwards.
__device__ __forceinline__ void push_wait_readers(const PushCtx& pc, int tid) {
  if (tid < pc.world) {
    const uint64_t prev = pc.epoch >= 2 ? pc.epoch - 2 : 0;
    if (!wait_flag(pc.peers->acks[pc.rank] + tid, [&](uint64_t v) { return v >= prev; })) atomicAdd(pc.timeouts, 1u);
  }
}

// Store row b's record into slot (epoch & 1, rank) of every peer window (NVLink stores).
__device__ __forceinline__ void push_record(const PushCtx& pc, int b, const fs_summary& f) {
  const size_t off = ((size_t)(pc.epoch & 1) * pc.world + pc.rank) * pc.B_max + b;
  for (int p = 0; p < pc.world; ++p) pc.peers->rec[p][off] = f;
}

// After every record of this rank is stored (by this thread or ordered before it by a fence +
// barrier / counter): make them visible system-wide, then release this rank's flag in every window.
__device__ __forceinline__ void push_release(const PushCtx& pc) {
  __threadfence_system();
  const int par = (int)(pc.epoch & 1);
  for (int p = 0; p < pc.world; ++p) st_release_sys(pc.peers->flags[p] + par * pc.world + pc.rank, pc.epoch);
}

}  // namespace fs
