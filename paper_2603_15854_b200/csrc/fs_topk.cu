// fs_topk.cu -- top-k / top-p sampling over materialised logits (§4.6
// P:397-398 "each tile computes top-k candidates locally, a second stage reduces all per-tile
// candidates into a global top-k", then top-p on the k survivors; reading R19).
//
//  A  topk_chunk_kernel   grid (chunks of 4096 columns) x B rows, 256 threads x 16 contiguous
//                         columns: transform (bias, 1/tau, mask) -> order-preserving keys ->
//                         block radix select (4 x 8-bit digits) of the chunk's k largest; ties at
//                         the boundary go to the smaller column (block scan in index order).
//                         Writes k (key, id) candidates per (row, chunk).
//  B  topk_final_kernel   one block per row: radix select of the global k largest over the
//                         row's candidates (streamed from L2), secondary select on the id for
//                         boundary ties, bitonic sort (l~ desc, id asc), top-p prefix cut on
//                         softmax(l~) in fp32, Gumbel-max over the kept set with the per-token
//                         noise of R1 / R18 (0 on greedy rows).
#include <cuda_bf16.h>

#include <algorithm>

#include "fs_device.cuh"
#include "fs_kernels.h"
#include "fs_sm100.cuh"

namespace fs {

namespace {

constexpr int kChunk = 4096;
constexpr int kPerThread = kChunk / 256;
constexpr int kMaxK = 1024;
constexpr int kMaxSurv = 1024;   // chunk fast path: survivors sorted in shared memory

template <typename T>
__device__ __forceinline__ float ldv(const T* p) {
  if constexpr (sizeof(T) == 2) return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(p));
  else return *p;
}

// Digit search of one radix pass, warp 0 (256 bins, lane L holds bins 8L..8L+7): the largest
// digit d whose suffix count reaches krem (desc) or the smallest whose prefix count does (asc).
// Writes (d, krem - count beyond d) to out[0..1].
template <bool DESC>
__device__ __forceinline__ void warp_digit(const uint32_t* hist, int krem, int lane, uint32_t* out) {
  int h[8], sum = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) { h[i] = (int)hist[lane * 8 + i]; sum += h[i]; }
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = DESC ? __shfl_down_sync(0xFFFFFFFFu, incl, o) : __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (DESC ? lane + o < 32 : lane >= o) incl += v;
  }
  const int before = incl - sum;
  const bool here = before < krem && incl >= krem;
  int d = 0, nk = 0, acc = before;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int i = DESC ? 7 - j : j;
    const bool hit = here && nk == 0 && acc + h[i] >= krem;
    d = hit ? lane * 8 + i : d;
    nk = hit ? krem - acc : nk;
    acc += h[i];
  }
  if (here) { out[0] = (uint32_t)d; out[1] = (uint32_t)nk; }
}

// Block-wide radix select over keys held by the calling threads (valid flags), any multiple of 32 threads.
// Returns (threshold T, number of elements equal to T to take) such that the k largest are
// {key > T} plus `take` elements with key == T.  If fewer than k valid elements exist, T = 0
// and take = #(key == 0) (i.e. everything).
__device__ __forceinline__ void block_radix_select(const uint32_t* keys, const bool* valid, int n, int k,
                                                   uint32_t* hist, uint32_t& T, int& take) {
  uint32_t prefix = 0, pmask = 0;
  int krem = k;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int i = 0; i < n; ++i)
      warp_hist_add(hist, valid[i] && (keys[i] & pmask) == prefix, (keys[i] >> shift) & 255u, threadIdx.x & 31);
    __syncthreads();
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) { hist[256] = 0u; hist[257] = (uint32_t)krem; }   // fewer than krem: digit 0
      __syncwarp();
      warp_digit<true>(hist, krem, threadIdx.x, hist + 256);   // >= krem valid keys
    }
    __syncthreads();
    prefix |= hist[256] << shift;
    pmask |= 255u << shift;
    krem = (int)hist[257];
    __syncthreads();
  }
  T = prefix;
  take = krem;
}

__device__ __forceinline__ void bitonic_sort_desc(Cand* a, int n) {   // n power of two, key desc, idx asc
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const Cand x = a[i], y = a[j];
          const bool x_first = (x.key > y.key) || (x.key == y.key && (uint32_t)x.idx < (uint32_t)y.idx);
          if (x_first != up) { a[i] = y; a[j] = x; }
        }
      }
      __syncthreads();
    }
  }
}

template <typename T, bool XFORM>
__global__ void __launch_bounds__(256)
topk_chunk_kernel(const T* __restrict__ logits, int64_t ld, const float* __restrict__ bias,
                  const float* __restrict__ temperature, const uint32_t* __restrict__ mask, int64_t mask_words, int V,
                  int k, int nchunk, Cand* __restrict__ cand, uint32_t* __restrict__ slot_lb, int m) {
  __shared__ uint32_t hist[258];
  __shared__ int scan[256];
  __shared__ int n_gt;
  __shared__ uint32_t runmax[256];
  __shared__ Cand surv[kMaxSurv];
  const int b = blockIdx.y, c = blockIdx.x;
  const int v0 = c * kChunk + threadIdx.x * kPerThread;
  float it = 1.0f;
  if (XFORM && temperature) {
    const float t = temperature[b];
    it = (t == 0.0f) ? 1.0f : (t > 0.0f && isfinite(t)) ? 1.0f / t : __int_as_float(0x7FC00000);
  }
  uint32_t keys[kPerThread];
  bool valid[kPerThread];
  int nvalid = 0;
  // 16 consecutive columns per thread: one 64-byte (fp32) / 32-byte (bf16) vector load when the
  // row is 16-byte aligned and the run is inside V, else scalar loads
  const T* rowp = logits + (int64_t)b * ld;
  float lv[kPerThread];
  const bool vec = v0 + kPerThread <= V && (reinterpret_cast<uintptr_t>(rowp + v0) & 15u) == 0;
  if (vec) {
    const uint4* q = reinterpret_cast<const uint4*>(rowp + v0);
    if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint4 u = __ldg(q + j);
        lv[4 * j] = __uint_as_float(u.x); lv[4 * j + 1] = __uint_as_float(u.y);
        lv[4 * j + 2] = __uint_as_float(u.z); lv[4 * j + 3] = __uint_as_float(u.w);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const uint4 u = __ldg(q + j);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          lv[8 * j + 2 * t] = __uint_as_float(w[t] << 16);
          lv[8 * j + 2 * t + 1] = __uint_as_float(w[t] & 0xFFFF0000u);
        }
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) lv[i] = v0 + i < V ? ldv(rowp + v0 + i) : -INFINITY;
  }
  const uint32_t mword = (XFORM && mask && v0 < V) ? mask[(int64_t)b * mask_words + (v0 >> 5)] : 0xFFFFFFFFu;
#pragma unroll
  for (int i = 0; i < kPerThread; ++i) {
    const int v = v0 + i;
    valid[i] = v < V;
    float l = valid[i] ? lv[i] : -INFINITY;
    if (XFORM && valid[i]) {
      l = (l + (bias ? bias[v] : 0.0f)) * it;
      if (mask && !((mword >> (v & 31)) & 1u)) l = -INFINITY;
    }
    if (isnan(l)) l = -INFINITY;
    keys[i] = order_key(l);
    nvalid += valid[i];
  }
  const int chunk_n = min(kChunk, V - c * kChunk);
  const int kk = min(k, chunk_n);
  Cand* out = cand + ((size_t)b * nchunk + c) * k;
  if (kk <= 256) {
    // Fast path: a lower bound of the chunk's kk-th key from the 256 run maxima (16 columns per
    // thread): kk runs have a maximum >= T, so >= kk elements are >= T.  The survivors {key >= T}
    // (typically ~kk) are sorted (key desc, id asc); the first kk are the chunk's top kk with the
    // same boundary-tie rule as the radix path (smaller column first).
    uint32_t rmax = 0u;
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) rmax = (valid[i] && keys[i] + 1u > rmax) ? keys[i] + 1u : rmax;
    runmax[threadIdx.x] = rmax;                    // key + 1: 0 marks a run with no valid column
    if (threadIdx.x == 0) n_gt = 0;
    __syncthreads();
    if (threadIdx.x < 32) {
      // warp 0: radix select (4 x 8-bit digits) of the kk-th largest of the 256 run maxima
      const int lane = threadIdx.x;
      uint32_t rv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) rv[i] = runmax[lane * 8 + i];
      uint32_t prefix = 0u, pmask = 0u;
      int krem = kk;
      for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
#pragma unroll
        for (int i = 0; i < 8; ++i) hist[lane * 8 + i] = 0u;
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (rv[i] != 0u && (rv[i] & pmask) == prefix) atomicAdd(&hist[(rv[i] >> shift) & 255u], 1u);
        __syncwarp();
        if (lane == 0) { hist[256] = 0u; hist[257] = (uint32_t)krem; }   // fewer than krem: digit 0
        __syncwarp();
        warp_digit<true>(hist, krem, lane, hist + 256);
        __syncwarp();
        prefix |= hist[256] << shift;
        pmask |= 255u << shift;
        krem = (int)hist[257];
        __syncwarp();
      }
      // prefix = the kk-th largest (key + 1); fewer than kk runs with valid columns: keep all
      int nr = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) nr += rv[i] != 0u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nr += __shfl_xor_sync(0xFFFFFFFFu, nr, o);
      if (lane == 0) hist[256] = nr >= kk ? prefix - 1u : 0u;
    }
    __syncthreads();
    const uint32_t T = hist[256];
    int mine = 0;
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) mine += valid[i] && keys[i] >= T;
    const int base = atomicAdd(&n_gt, mine);     // n_gt = survivor count after the barrier
    __syncthreads();
    const int ns = n_gt;
    if (ns <= 256) {
      // few survivors (the usual case): each finds its rank in (key desc, id asc) order directly
      int at = base;
#pragma unroll
      for (int i = 0; i < kPerThread; ++i)
        if (valid[i] && keys[i] >= T) surv[at++] = Cand{keys[i], v0 + i};
      __syncthreads();
      if ((int)threadIdx.x < ns) {
        const Cand x = surv[threadIdx.x];
        int rank = 0;
        for (int j = 0; j < ns; ++j) {
          const Cand y = surv[j];
          rank += (y.key > x.key) || (y.key == x.key && y.idx < x.idx);
        }
        if (rank < kk) out[rank] = x;
        if (rank == m - 1 && m <= chunk_n) slot_lb[(size_t)b * nchunk + c] = x.key;
      }
      for (int j = kk + (int)threadIdx.x; j < k; j += 256) out[j] = Cand{kKeyNone, -1};
      if (threadIdx.x == 0 && m > chunk_n) slot_lb[(size_t)b * nchunk + c] = 0u;
      return;
    }
    if (ns <= kMaxSurv) {
      int at = base;
#pragma unroll
      for (int i = 0; i < kPerThread; ++i)
        if (valid[i] && keys[i] >= T) surv[at++] = Cand{keys[i], v0 + i};
      int npow = 1;
      while (npow < ns) npow <<= 1;
      for (int i = ns + (int)threadIdx.x; i < npow; i += 256) surv[i] = Cand{0u, 0x7FFFFFFF};
      __syncthreads();
      bitonic_sort_desc(surv, npow);
      for (int j = threadIdx.x; j < k; j += 256) out[j] = j < kk ? surv[j] : Cand{kKeyNone, -1};
      if (threadIdx.x == 0) slot_lb[(size_t)b * nchunk + c] = (m <= chunk_n) ? surv[m - 1].key : 0u;
      return;
    }
    __syncthreads();                              // heavy ties: exact radix path below
  }
  uint32_t Tk = 0;
  int take = 0;
  block_radix_select(keys, valid, kPerThread, kk, hist, Tk, take);
  // count ties (key == T) per thread in index order; exclusive scan over threads
  int ties = 0;
#pragma unroll
  for (int i = 0; i < kPerThread; ++i) ties += (valid[i] && keys[i] == Tk);
  scan[threadIdx.x] = ties;
  if (threadIdx.x == 0) n_gt = 0;
  __syncthreads();
  for (int off = 1; off < 256; off <<= 1) {
    const int x = threadIdx.x >= off ? scan[threadIdx.x - off] : 0;
    __syncthreads();
    scan[threadIdx.x] += x;
    __syncthreads();
  }
  int tie_pos = scan[threadIdx.x] - ties;        // exclusive prefix
  const int n_greater = kk - take;
#pragma unroll
  for (int i = 0; i < kPerThread; ++i) {
    if (!valid[i]) continue;
    if (keys[i] > Tk) {
      const int pos = atomicAdd(&n_gt, 1);
      out[pos] = Cand{keys[i], v0 + i};
    } else if (keys[i] == Tk) {
      if (tie_pos < take) out[n_greater + tie_pos] = Cand{keys[i], v0 + i};
      ++tie_pos;
    }
  }
  for (int j = kk + (int)threadIdx.x; j < k; j += 256) out[j] = Cand{kKeyNone, -1};   // padding
  // the chunk's m-th largest key (m = ceil(k / #chunks)): the final kernel's lower bound for the
  // row's k-th key is the ceil(k/m)-th largest of these (0 = this chunk proves nothing)
  uint32_t Tm = 0u;
  if (m <= chunk_n) {
    __syncthreads();
    int tm;
    block_radix_select(keys, valid, kPerThread, m, hist, Tm, tm);
  }
  if (threadIdx.x == 0) slot_lb[(size_t)b * nchunk + c] = Tm;
}

constexpr int kFinalThreads = 512;
constexpr int kMaxTies = 1024;

constexpr int kMaxSlots = 256;

// Candidates of a row: cand[b][0, n_b), n_b = row_count[b] (atomically allocated by stage 1; reset
// to 0 here for the next call) or ncand (fixed layout, padding id -1).  A lower bound LB of the
// row's k-th key prunes them before the exact selection: slot s guarantees m elements with key
// >= slot_lb[s], so r = ceil(k/m) slots with slot_lb >= L prove k elements >= L; LB = the r-th
// largest slot_lb.  Survivors (key >= LB) are staged in shared memory when they fit, else every
// pass re-reads the row from L2 with the same filter.
template <bool PRQ>
__global__ void __launch_bounds__(kFinalThreads)
topk_final_kernel(const Cand* __restrict__ cand, int ncand, int* __restrict__ row_count, int k, float top_p,
                  const float* __restrict__ temperature, uint64_t seed, uint64_t step,
                  const uint64_t* __restrict__ seeds, const uint64_t* __restrict__ steps, int32_t* idx_out,
                  float* score_out, float* logZ_out, float* logprob_out, int row_offset, int smem_cand,
                  const uint32_t* __restrict__ slot_lb, int nslots, int m) {
  extern __shared__ Cand rowc[];
  __shared__ uint32_t hist[256];
  __shared__ uint32_t dsel[2];
  __shared__ Cand sel[kMaxK];
  __shared__ Cand ties[kMaxTies];
  __shared__ float red_f[kMaxK];
  __shared__ Cand red_c[kFinalThreads];
  __shared__ uint32_t lbv[kMaxSlots];
  __shared__ int cnt[3];
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31;
  sm100::pdl_wait();                          // stage-1 candidates are visible past this point
  const Cand* grow = cand + (size_t)b * ncand;
  const int nrow = row_count ? row_count[b] : ncand;
  uint32_t LB = 0u;
  const int r = (k + m - 1) / m;
  if (slot_lb && nslots <= kMaxSlots && r <= nslots) {
    for (int i = threadIdx.x; i < nslots; i += kFinalThreads) lbv[i] = slot_lb[(size_t)b * nslots + i];
    if (threadIdx.x == 0) dsel[0] = 0u;
    __syncthreads();
    for (int i = threadIdx.x; i < nslots; i += kFinalThreads) {
      const uint32_t x = lbv[i];
      int rank = 0;
      for (int j = 0; j < nslots; ++j) rank += (lbv[j] > x) || (lbv[j] == x && j < i);
      if (rank == r - 1) dsel[0] = x;
    }
    __syncthreads();
    LB = dsel[0];
  }
  if (threadIdx.x == 0) cnt[2] = 0;
  __syncthreads();
  constexpr int kBatch = 8;                    // loads in flight per thread
  for (int base0 = threadIdx.x & ~31; base0 < nrow; base0 += kFinalThreads * kBatch) {
    Cand cb[kBatch];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int i = base0 + j * kFinalThreads + lane;
      cb[j] = i < nrow ? grow[i] : Cand{kKeyNone, -1};
    }
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const Cand c = cb[j];
      const bool keep = c.idx >= 0 && c.key >= LB;
      const uint32_t bl = __ballot_sync(0xFFFFFFFFu, keep);
      if (bl) {
        int pos = 0;
        if (lane == 0) pos = atomicAdd(&cnt[2], __popc(bl));
        pos = __shfl_sync(0xFFFFFFFFu, pos, 0);
        const int at = pos + __popc(bl & ((1u << lane) - 1u));
        if (keep && at < smem_cand) rowc[at] = c;
      }
    }
  }
  __syncthreads();
  if (row_count && threadIdx.x == 0) row_count[b] = 0;   // ready for the next stage 1
  const bool staged = cnt[2] <= smem_cand;
  int n = staged ? cnt[2] : nrow;
  if (staged) LB = 0u;                         // staged entries are all valid and >= LB
  const Cand* row = staged ? rowc : grow;
  const Cand* selp;                            // the top k, sorted by (key desc, id asc)
  int nsel;
  if (staged && n <= kMaxK) {
    // few survivors (the usual case after pruning): sort them all, the first k are the top k
    int npow = 1;
    while (npow < n) npow <<= 1;
    for (int i = n + (int)threadIdx.x; i < npow; i += kFinalThreads) rowc[i] = Cand{0u, 0x7FFFFFFF};
    __syncthreads();
    bitonic_sort_desc(rowc, npow);
    selp = rowc;
    nsel = min(k, n);
  } else {
  // ---- radix select of the k largest keys over the row's candidates ----
  uint32_t prefix = 0, pmask = 0;
  int krem = k;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    if (threadIdx.x < 256) hist[threadIdx.x] = 0;
    __syncthreads();
    for (int base = threadIdx.x & ~31; base < n; base += kFinalThreads) {
      const int i = base + lane;
      const Cand c = i < n ? row[i] : Cand{kKeyNone, -1};
      warp_hist_add(hist, c.idx >= 0 && c.key >= LB && (c.key & pmask) == prefix, (c.key >> shift) & 255u, lane);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) { dsel[0] = 0; dsel[1] = (uint32_t)krem; }   // fewer than k: take all
      __syncwarp();
      warp_digit<true>(hist, krem, lane, dsel);
    }
    __syncthreads();
    prefix |= dsel[0] << shift;
    pmask |= 255u << shift;
    krem = (int)dsel[1];
  }
  const uint32_t Tk = prefix;
  // ---- collect key > T into sel, key == T into ties ----
  if (threadIdx.x < 3) cnt[threadIdx.x] = 0;
  int npow = 1;
  while (npow < k) npow <<= 1;
  for (int i = threadIdx.x; i < npow; i += kFinalThreads) sel[i] = Cand{0u, 0x7FFFFFFF};
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += kFinalThreads) {
    const Cand c = row[i];
    if (c.idx < 0 || c.key < LB) continue;
    if (c.key > Tk) {
      const int pos = atomicAdd(&cnt[0], 1);
      if (pos < kMaxK) sel[pos] = c;
    } else if (c.key == Tk) {
      const int pos = atomicAdd(&cnt[1], 1);
      if (pos < kMaxTies) ties[pos] = c;
    }
  }
  __syncthreads();
  const int n_gt = cnt[0], n_ties = cnt[1];
  if (n_ties <= krem || n_ties <= kMaxTies) {
    // boundary ties: the krem smallest ids (sort the ties by id when there are more than krem)
    if (n_ties > krem) {
      int tp = 1;
      while (tp < n_ties) tp <<= 1;
      for (int i = n_ties + (int)threadIdx.x; i < tp; i += kFinalThreads) ties[i] = Cand{0u, 0x7FFFFFFF};
      __syncthreads();
      bitonic_sort_desc(ties, tp);                  // equal keys: id ascending
    }
    const int take = min(krem, n_ties);
    for (int i = threadIdx.x; i < take; i += kFinalThreads) sel[n_gt + i] = ties[i];
    if (threadIdx.x == 0) cnt[0] = n_gt + take;
  } else {
    // more than kMaxTies boundary ties (degenerate rows): secondary radix select on the id
    uint32_t iprefix = 0, imask = 0;
    int irem = krem;
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass;
      if (threadIdx.x < 256) hist[threadIdx.x] = 0;
      __syncthreads();
      for (int base = threadIdx.x & ~31; base < n; base += kFinalThreads) {
        const int i = base + lane;
        const Cand c = i < n ? row[i] : Cand{kKeyNone, -1};
        const uint32_t id = (uint32_t)c.idx;
        warp_hist_add(hist, c.idx >= 0 && c.key == Tk && (id & imask) == iprefix, (id >> shift) & 255u, lane);
      }
      __syncthreads();
      if (threadIdx.x < 32) warp_digit<false>(hist, irem, lane, dsel);
      __syncthreads();
      iprefix |= dsel[0] << shift;
      imask |= 255u << shift;
      irem = (int)dsel[1];
    }
    for (int i = threadIdx.x; i < n; i += kFinalThreads) {
      const Cand c = row[i];
      if (c.idx >= 0 && c.key == Tk && (uint32_t)c.idx <= iprefix) {
        const int pos = atomicAdd(&cnt[0], 1);
        if (pos < kMaxK) sel[pos] = c;
      }
    }
  }
  __syncthreads();
  nsel = min(cnt[0], k);
  bitonic_sort_desc(sel, npow);
  selp = sel;
  }
  // ---- top-p on the sorted top k (finite l~ only), fp32: block scan of e_i = exp(l~_i - l~_0) ----
  __shared__ float wsum[kFinalThreads / 32];
  __shared__ uint32_t wkey[kFinalThreads / 32];
  __shared__ int widx[kFinalThreads / 32];
  __shared__ float wlt[kFinalThreads / 32];
  const int warp = threadIdx.x >> 5;
  const float tau = temperature ? temperature[b] : 1.0f;
  const float gsc = (tau == 0.0f) ? 0.0f : 1.0f;
  const float l0 = nsel > 0 && selp[0].key > kKeyNegInf ? key_to_float(selp[0].key) : -INFINITY;
  const int i0 = 2 * (int)threadIdx.x;         // nsel <= 1024 = 2 per thread
  const float e0 = (i0 < nsel && selp[i0].key > kKeyNegInf) ? __expf(key_to_float(selp[i0].key) - l0) : 0.0f;
  const float e1 = (i0 + 1 < nsel && selp[i0 + 1].key > kKeyNegInf) ? __expf(key_to_float(selp[i0 + 1].key) - l0) : 0.0f;
  float incl = e0 + e1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  if (threadIdx.x == 0) cnt[1] = nsel - 1;
  __syncthreads();
  if (warp == 0) {
    float w = lane < kFinalThreads / 32 ? wsum[lane] : 0.0f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const float v = __shfl_up_sync(0xFFFFFFFFu, w, o);
      if (lane >= o) w += v;
    }
    if (lane < kFinalThreads / 32) wsum[lane] = w;           // inclusive warp prefix
  }
  __syncthreads();
  const float Z = wsum[kFinalThreads / 32 - 1];
  const float before = (warp > 0 ? wsum[warp - 1] : 0.0f) + incl - (e0 + e1);
  const float c0 = before + e0, c1 = c0 + e1;
  // cut = first i with cumsum_i >= p * Z (all k when p >= 1)
  if (top_p < 1.0f) {
    const float thr = top_p * Z;
    if (i0 < nsel && c0 >= thr && before < thr) atomicMin(&cnt[1], i0);
    else if (i0 + 1 < nsel && c1 >= thr && c0 < thr) atomicMin(&cnt[1], i0 + 1);
  }
  __syncthreads();
  const int mcut = cnt[1];
  // ---- Gumbel-max over the kept set selp[0..mcut] ----
  State best = state_empty();
  float zk = 0.0f;
  for (int i = threadIdx.x; i <= mcut && i < nsel; i += kFinalThreads) {
    const Cand c = selp[i];
    if (c.key <= kKeyNegInf) continue;
    const float l = key_to_float(c.key);
    uint32_t rr;
    if (PRQ) {
      const uint64_t sd = seeds[b], st = steps ? steps[b] : step;
      const U4 o = philox4x32_10((uint32_t)c.idx >> 2, 0x80000000u, (uint32_t)st, (uint32_t)(st >> 32) & 0xFFFFFFu,
                                 (uint32_t)sd, (uint32_t)(sd >> 32));
      const uint32_t s4 = (uint32_t)c.idx & 3u;
      rr = s4 == 0 ? o.x : s4 == 1 ? o.y : s4 == 2 ? o.z : o.w;
    } else {
      const uint32_t bg = (uint32_t)(b + row_offset);
      const U4 o = philox4x32_10((uint32_t)c.idx, bg >> 2, (uint32_t)step,
                                 (uint32_t)(step >> 32) & 0xFFFFFFu, (uint32_t)seed, (uint32_t)(seed >> 32));
      const uint32_t s4 = bg & 3u;
      rr = s4 == 0 ? o.x : s4 == 1 ? o.y : s4 == 2 ? o.z : o.w;
    }
    const float sc = l + gumbel32(rr) * gsc;
    best = state_max(best, State{order_key(sc), c.idx, 0.0f, __float_as_uint(l)});
    zk += __expf(l - l0);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const State y{__shfl_xor_sync(0xFFFFFFFFu, best.key, o), __shfl_xor_sync(0xFFFFFFFFu, best.idx, o), 0.0f,
                  __shfl_xor_sync(0xFFFFFFFFu, best.lt, o)};
    best = state_max(best, y);
    zk += __shfl_xor_sync(0xFFFFFFFFu, zk, o);
  }
  __syncthreads();                             // wsum reads above are done
  if (lane == 0) { wkey[warp] = best.key; widx[warp] = best.idx; wlt[warp] = __uint_as_float(best.lt); wsum[warp] = zk; }
  __syncthreads();
  if (warp == 0) {
    const bool live = lane < kFinalThreads / 32;
    State x{live ? wkey[lane] : kKeyNone, live ? widx[lane] : -1, 0.0f, live ? __float_as_uint(wlt[lane]) : 0u};
    float z = live ? wsum[lane] : 0.0f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const State y{__shfl_xor_sync(0xFFFFFFFFu, x.key, o), __shfl_xor_sync(0xFFFFFFFFu, x.idx, o), 0.0f,
                    __shfl_xor_sync(0xFFFFFFFFu, x.lt, o)};
      x = state_max(x, y);
      z += __shfl_xor_sync(0xFFFFFFFFu, z, o);
    }
    if (lane == 0) {
      const bool defined = x.key > kKeyNegInf && x.idx >= 0;
      idx_out[b] = defined ? x.idx : -1;
      if (score_out) score_out[b] = defined ? key_to_float(x.key) : -INFINITY;
      const float lz = defined ? l0 + logf(z) : -INFINITY;      // log-mass of the kept set
      if (logZ_out) logZ_out[b] = lz;
      if (logprob_out) logprob_out[b] = defined ? __uint_as_float(x.lt) - lz : -INFINITY;
    }
  }
}

// Fused route with span maxima (stage 1 mode 2 + gmax): one block per row.  T = the k-th largest
// of the threads' largest span maxima (k spans hold an element >= T, so the row's k-th largest raw
// logit is >= T); relaxed by 8 key steps so that an element whose transformed value ties the k-th
// after fp32 rounding of l/tau is still gathered.  Only the spans at or above it are read back.
constexpr int kGatherThreads = 1024;
constexpr int kGatherPer = 32;            // most span entries per thread: V <= 16 * 1024 * 32
// PER span entries per thread (8 / 16 / 32 by V): fewer registers for V <= 262,144, so
// that two 1024-thread blocks (rows) fit on an SM (B = 256 in one wave)
template <int PER>
__global__ void __launch_bounds__(kGatherThreads, PER <= 16 ? 2 : 1)
topk_gather_kernel(const float* __restrict__ mat, int64_t ld, const uint32_t* __restrict__ gmax, int64_t gld,
                   const float* __restrict__ temperature, int V, int k, Cand* __restrict__ cand, int64_t stride,
                   int* __restrict__ row_count) {
  __shared__ uint32_t hist[258];
  __shared__ int cnt;
  const int b = blockIdx.x;
  const int64_t nunits = (V + 15) / 16;
  const uint32_t* g = gmax + (int64_t)b * gld;
  uint32_t keys[PER];
  bool valid[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int64_t u = threadIdx.x + (int64_t)j * kGatherThreads;
    keys[j] = u < nunits ? g[u] : 0u;
    valid[j] = keys[j] > 1u;               // 0 / 1: no span starts at this unit
  }
  if (threadIdx.x == 0) cnt = 0;
  // bound from the threads' maxima: k threads hold a span whose maximum is >= their k-th largest,
  // so k elements are >= it (a 1-key-per-thread select instead of 32)
  uint32_t tmax = 0u;
#pragma unroll
  for (int j = 0; j < PER; ++j) tmax = valid[j] && keys[j] > tmax ? keys[j] : tmax;
  const bool tvalid = tmax > 1u;
  uint32_t T = 0;
  int take = 0;
  block_radix_select(&tmax, &tvalid, 1, k, hist, T, take);   // T = 0 when fewer than k threads hold spans
  const uint32_t Tr = T > 8u ? T - 8u : 0u;
  float it = 1.0f;
  if (temperature) {
    const float t = temperature[b];
    it = (t == 0.0f) ? 1.0f : (t > 0.0f && isfinite(t)) ? 1.0f / t : __int_as_float(0x7FC00000);
  }
  const float* row = mat + (int64_t)b * ld;
  Cand* out = cand + (int64_t)b * stride;
  // the spans to read back as a bit mask (keys / valid stay in registers: they are only indexed in
  // unrolled loops; a rolled loop over them compiled to local-memory arrays)
  uint32_t sel = 0u;
#pragma unroll
  for (int j = 0; j < PER; ++j) sel |= (valid[j] && keys[j] >= Tr) ? (1u << j) : 0u;
#pragma unroll 1
  for (; sel != 0u; sel &= sel - 1u) {
    const int j = __ffs(sel) - 1;
    const int64_t u = threadIdx.x + (int64_t)j * kGatherThreads;
    const int64_t v0 = u * 16;
    const int64_t want = (u + 1 < nunits && g[u + 1] == 1u) ? 32 : 16;
    const int n = (int)(want < V - v0 ? want : V - v0);
#pragma unroll 1
    for (int i0 = 0; i0 < n; i0 += 8) {             // 8 loads in flight per round (few registers)
      float x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = i0 + i < n ? row[v0 + i0 + i] : -INFINITY;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float raw = x[i];
        if (isnan(raw)) raw = -INFINITY;
        if (i0 + i >= n || order_key(raw) < Tr) continue;
        float l = raw * it;
        if (isnan(l)) l = -INFINITY;
        const int pos = atomicAdd(&cnt, 1);
        out[pos] = Cand{order_key(l), (int32_t)(v0 + i0 + i)};
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) row_count[b] = cnt;
}

}  // namespace

int topk_chunks(int V) { return (V + kChunk - 1) / kChunk; }

cudaError_t launch_topk_gather(const float* mat, int64_t ld, const uint32_t* gmax, int64_t gld,
                               const float* temperature, int B, int V, int k, Cand* cand, int64_t stride,
                               int* row_count, cudaStream_t stream) {
  const int64_t units = (int64_t)(V + 15) / 16;
  if (units > (int64_t)kGatherThreads * kGatherPer) return cudaErrorInvalidValue;
  if (units <= (int64_t)kGatherThreads * 8)
    topk_gather_kernel<8><<<B, kGatherThreads, 0, stream>>>(mat, ld, gmax, gld, temperature, V, k, cand, stride,
                                                            row_count);
  else if (units <= (int64_t)kGatherThreads * 16)
    topk_gather_kernel<16><<<B, kGatherThreads, 0, stream>>>(mat, ld, gmax, gld, temperature, V, k, cand, stride,
                                                             row_count);
  else
    topk_gather_kernel<32><<<B, kGatherThreads, 0, stream>>>(mat, ld, gmax, gld, temperature, V, k, cand, stride,
                                                             row_count);
  return cudaGetLastError();
}
int topk_max_k() { return kMaxK; }

cudaError_t launch_topk_sample(fs_dtype dtype, const void* logits, int64_t ld, const float* bias,
                               const float* temperature, const uint32_t* mask, int64_t mask_words, int B, int V,
                               int k, float top_p, uint64_t seed, uint64_t step, const uint64_t* seeds,
                               const uint64_t* steps, void* cand_ws, int32_t* idx_out, float* score_out,
                               float* logZ_out, float* logprob_out, cudaStream_t stream, int row_offset) {
  const int nchunk = topk_chunks(V);
  Cand* cand = static_cast<Cand*>(cand_ws);
  uint32_t* thr = reinterpret_cast<uint32_t*>(cand + (size_t)B * nchunk * k);
  const int m = (k + nchunk - 1) / nchunk;
  const dim3 ga(nchunk, B);
  const bool xform = bias || temperature || mask;
  if (dtype == FS_BF16) {
    if (xform) topk_chunk_kernel<uint16_t, true><<<ga, 256, 0, stream>>>(static_cast<const uint16_t*>(logits), ld,
                   bias, temperature, mask, mask_words, V, k, nchunk, cand, thr, m);
    else topk_chunk_kernel<uint16_t, false><<<ga, 256, 0, stream>>>(static_cast<const uint16_t*>(logits), ld, bias,
                   temperature, mask, mask_words, V, k, nchunk, cand, thr, m);
  } else {
    if (xform) topk_chunk_kernel<float, true><<<ga, 256, 0, stream>>>(static_cast<const float*>(logits), ld, bias,
                   temperature, mask, mask_words, V, k, nchunk, cand, thr, m);
    else topk_chunk_kernel<float, false><<<ga, 256, 0, stream>>>(static_cast<const float*>(logits), ld, bias,
                   temperature, mask, mask_words, V, k, nchunk, cand, thr, m);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_topk_final(cand, nchunk * k, nullptr, B, k, top_p, temperature, seed, step, seeds, steps, idx_out,
                           score_out, logZ_out, logprob_out, stream, row_offset, false, thr, nchunk, m);
}

cudaError_t launch_topk_final(const Cand* cand, int ncand, int* row_count, int B, int k, float top_p,
                              const float* temperature, uint64_t seed, uint64_t step, const uint64_t* seeds,
                              const uint64_t* steps, int32_t* idx_out, float* score_out, float* logZ_out,
                              float* logprob_out, cudaStream_t stream, int row_offset, bool pdl,
                              const uint32_t* slot_lb, int nslots, int m) {
  // survivors are staged in shared memory next to the static arrays (~38 KB)
  constexpr int kDynMax = 180 * 1024;
  const int smem_cand = kDynMax / (int)sizeof(Cand);
  {
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(topk_final_kernel<true>), kDynMax);
    if (e == cudaSuccess) e = ensure_smem_attr(reinterpret_cast<const void*>(topk_final_kernel<false>), kDynMax);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.stream = stream;
  cfg.gridDim = dim3(B);
  cfg.blockDim = dim3(kFinalThreads);
  cfg.dynamicSmemBytes = kDynMax;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  if (seeds)
    return cudaLaunchKernelEx(&cfg, topk_final_kernel<true>, cand, ncand, row_count, k, top_p, temperature, seed,
                              step, seeds, steps, idx_out, score_out, logZ_out, logprob_out, row_offset, smem_cand,
                              slot_lb, nslots, m);
  return cudaLaunchKernelEx(&cfg, topk_final_kernel<false>, cand, ncand, row_count, k, top_p, temperature, seed,
                            step, seeds, steps, idx_out, score_out, logZ_out, logprob_out, row_offset, smem_cand,
                            slot_lb, nslots, m);
}

}  // namespace fs
