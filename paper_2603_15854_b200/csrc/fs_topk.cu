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

struct Cand {
  uint32_t key;
  int32_t idx;
};

template <typename T>
__device__ __forceinline__ float ldv(const T* p) {
  if constexpr (sizeof(T) == 2) return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(p));
  else return *p;
}

// Block-wide radix select over keys held by the calling threads (valid flags), 256 threads.
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
      if (valid[i] && (keys[i] & pmask) == prefix) atomicAdd(&hist[(keys[i] >> shift) & 255u], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0, d = 255;
      for (; d > 0; --d) {
        if (acc + (int)hist[d] >= krem) break;
        acc += (int)hist[d];
      }
      hist[256] = (uint32_t)d;
      hist[257] = (uint32_t)(krem - acc);
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

template <typename T, bool XFORM>
__global__ void __launch_bounds__(256)
topk_chunk_kernel(const T* __restrict__ logits, int64_t ld, const float* __restrict__ bias,
                  const float* __restrict__ temperature, const uint32_t* __restrict__ mask, int64_t mask_words, int V,
                  int k, int nchunk, Cand* __restrict__ cand) {
  __shared__ uint32_t hist[258];
  __shared__ int scan[256];
  __shared__ int n_gt;
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
#pragma unroll
  for (int i = 0; i < kPerThread; ++i) {
    const int v = v0 + i;
    valid[i] = v < V;
    float l = valid[i] ? ldv(logits + (int64_t)b * ld + v) : -INFINITY;
    if (XFORM && valid[i]) {
      l = (l + (bias ? bias[v] : 0.0f)) * it;
      if (mask && !((mask[(int64_t)b * mask_words + (v >> 5)] >> (v & 31)) & 1u)) l = -INFINITY;
    }
    if (isnan(l)) l = -INFINITY;
    keys[i] = order_key(l);
    nvalid += valid[i];
  }
  const int chunk_n = min(kChunk, V - c * kChunk);
  uint32_t Tk = 0;
  int take = 0;
  const int kk = min(k, chunk_n);
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
  Cand* out = cand + ((size_t)b * nchunk + c) * k;
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

template <bool PRQ>
__global__ void __launch_bounds__(512)
topk_final_kernel(const Cand* __restrict__ cand, int ncand, int k, float top_p, const float* __restrict__ temperature,
                  uint64_t seed, uint64_t step, const uint64_t* __restrict__ seeds, const uint64_t* __restrict__ steps,
                  int32_t* idx_out, float* score_out, float* logZ_out, float* logprob_out) {
  __shared__ uint32_t hist[258];
  __shared__ Cand sel[kMaxK];
  __shared__ float red_f[kMaxK];
  __shared__ Cand red_c[512];
  __shared__ int cnt[2];
  const int b = blockIdx.x;
  const Cand* row = cand + (size_t)b * ncand;
  // ---- radix select of the k largest keys over the row's candidates (streamed from L2) ----
  uint32_t prefix = 0, pmask = 0;
  int krem = k;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < ncand; i += blockDim.x) {
      const Cand c = row[i];
      if (c.idx >= 0 && (c.key & pmask) == prefix) atomicAdd(&hist[(c.key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0, d = 255;
      for (; d > 0; --d) {
        if (acc + (int)hist[d] >= krem) break;
        acc += (int)hist[d];
      }
      hist[256] = (uint32_t)d;
      hist[257] = (uint32_t)(krem - acc);
    }
    __syncthreads();
    prefix |= hist[256] << shift;
    pmask |= 255u << shift;
    krem = (int)hist[257];
    __syncthreads();
  }
  const uint32_t Tk = prefix;
  // secondary select on the id among boundary ties: the krem smallest ids with key == T
  uint32_t iprefix = 0, imask = 0;
  int irem = krem;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < ncand; i += blockDim.x) {
      const Cand c = row[i];
      const uint32_t id = (uint32_t)c.idx;
      if (c.idx >= 0 && c.key == Tk && (id & imask) == iprefix) atomicAdd(&hist[(id >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0, d = 0;
      for (; d < 255; ++d) {
        if (acc + (int)hist[d] >= irem) break;
        acc += (int)hist[d];
      }
      hist[256] = (uint32_t)d;
      hist[257] = (uint32_t)(irem - acc);
    }
    __syncthreads();
    iprefix |= hist[256] << shift;
    imask |= 255u << shift;
    irem = (int)hist[257];
    __syncthreads();
  }
  // ---- collect: key > T, or key == T and id <= id_T (the last boundary id, exactly `krem` ties) ----
  if (threadIdx.x == 0) cnt[0] = 0;
  int npow = 1;
  while (npow < k) npow <<= 1;
  for (int i = threadIdx.x; i < npow; i += blockDim.x) sel[i] = Cand{0u, 0x7FFFFFFF};
  __syncthreads();
  for (int i = threadIdx.x; i < ncand; i += blockDim.x) {
    const Cand c = row[i];
    if (c.idx < 0) continue;
    if (c.key > Tk || (c.key == Tk && (uint32_t)c.idx <= iprefix)) {
      const int pos = atomicAdd(&cnt[0], 1);
      if (pos < kMaxK) sel[pos] = c;
    }
  }
  __syncthreads();
  const int n = min(cnt[0], k);
  bitonic_sort_desc(sel, npow);
  // ---- top-p on the sorted survivors (finite l~ only), fp32 ----
  const float tau = temperature ? temperature[b] : 1.0f;
  const float gsc = (tau == 0.0f) ? 0.0f : 1.0f;
  const float l0 = n > 0 && sel[0].key > kKeyNegInf ? key_to_float(sel[0].key) : -INFINITY;
  for (int i = threadIdx.x; i < npow; i += blockDim.x)
    red_f[i] = (i < n && sel[i].key > kKeyNegInf) ? __expf(key_to_float(sel[i].key) - l0) : 0.0f;
  __syncthreads();
  // inclusive prefix sum (Hillis-Steele) over npow <= 1024 entries with 512 threads
  for (int off = 1; off < npow; off <<= 1) {
    float x[2] = {0.f, 0.f};
    for (int t = 0; t < 2; ++t) {
      const int i = threadIdx.x + t * 512;
      if (i < npow && i >= off) x[t] = red_f[i - off];
    }
    __syncthreads();
    for (int t = 0; t < 2; ++t) {
      const int i = threadIdx.x + t * 512;
      if (i < npow) red_f[i] += x[t];
    }
    __syncthreads();
  }
  const float Z = n > 0 ? red_f[n - 1] : 0.0f;
  // m = first j with cumsum_j >= p * Z (all finite survivors when p >= 1)
  if (threadIdx.x == 0) cnt[1] = n - 1;
  __syncthreads();
  if (top_p < 1.0f)
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      if (red_f[i] >= top_p * Z && (i == 0 || red_f[i - 1] < top_p * Z)) cnt[1] = i;
  __syncthreads();
  int m = cnt[1];
  // drop -inf survivors (fewer than k finite)
  // ---- Gumbel-max over the kept set ----
  State best = state_empty();
  float zk = 0.0f;
  for (int i = threadIdx.x; i <= m && i < n; i += blockDim.x) {
    const Cand c = sel[i];
    if (c.key <= kKeyNegInf) continue;
    const float l = key_to_float(c.key);
    uint32_t r;
    if (PRQ) {
      const uint64_t sd = seeds[b], st = steps ? steps[b] : step;
      const U4 o = philox4x32_10((uint32_t)c.idx >> 2, 0x80000000u, (uint32_t)st, (uint32_t)(st >> 32) & 0xFFFFFFu,
                                 (uint32_t)sd, (uint32_t)(sd >> 32));
      const uint32_t s4 = (uint32_t)c.idx & 3u;
      r = s4 == 0 ? o.x : s4 == 1 ? o.y : s4 == 2 ? o.z : o.w;
    } else {
      const U4 o = philox4x32_10((uint32_t)c.idx, (uint32_t)b >> 2, (uint32_t)step,
                                 (uint32_t)(step >> 32) & 0xFFFFFFu, (uint32_t)seed, (uint32_t)(seed >> 32));
      const uint32_t s4 = (uint32_t)b & 3u;
      r = s4 == 0 ? o.x : s4 == 1 ? o.y : s4 == 2 ? o.z : o.w;
    }
    const float s = l + gumbel32(r) * gsc;
    State x{order_key(s), c.idx, 0.0f, __float_as_uint(l)};
    best = state_max(best, x);
    zk += __expf(l - l0);
  }
  red_c[threadIdx.x] = Cand{best.key, best.idx};
  red_f[threadIdx.x] = zk;
  __syncthreads();
  for (int w = 256; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const Cand x = red_c[threadIdx.x], y = red_c[threadIdx.x + w];
      const bool take_y = y.key > x.key || (y.key == x.key && y.idx >= 0 && (x.idx < 0 || y.idx < x.idx));
      if (take_y) red_c[threadIdx.x] = y;
      red_f[threadIdx.x] += red_f[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const Cand w = red_c[0];
    const bool defined = w.key > kKeyNegInf && w.idx >= 0;
    idx_out[b] = defined ? w.idx : -1;
    if (score_out) score_out[b] = defined ? key_to_float(w.key) : -INFINITY;
    const float lz = defined ? l0 + logf(red_f[0]) : -INFINITY;      // log-mass of the kept set
    if (logZ_out) logZ_out[b] = lz;
    if (logprob_out) {
      float lw = -INFINITY;
      for (int i = 0; i <= m && i < n; ++i)
        if (sel[i].idx == w.idx) lw = key_to_float(sel[i].key);
      logprob_out[b] = defined ? lw - lz : -INFINITY;
    }
  }
}

}  // namespace

int topk_chunks(int V) { return (V + kChunk - 1) / kChunk; }
int topk_max_k() { return kMaxK; }

cudaError_t launch_topk_sample(fs_dtype dtype, const void* logits, int64_t ld, const float* bias,
                               const float* temperature, const uint32_t* mask, int64_t mask_words, int B, int V,
                               int k, float top_p, uint64_t seed, uint64_t step, const uint64_t* seeds,
                               const uint64_t* steps, void* cand_ws, int32_t* idx_out, float* score_out,
                               float* logZ_out, float* logprob_out, cudaStream_t stream) {
  const int nchunk = topk_chunks(V);
  Cand* cand = static_cast<Cand*>(cand_ws);
  const dim3 ga(nchunk, B);
  const bool xform = bias || temperature || mask;
  if (dtype == FS_BF16) {
    if (xform) topk_chunk_kernel<uint16_t, true><<<ga, 256, 0, stream>>>(static_cast<const uint16_t*>(logits), ld,
                   bias, temperature, mask, mask_words, V, k, nchunk, cand);
    else topk_chunk_kernel<uint16_t, false><<<ga, 256, 0, stream>>>(static_cast<const uint16_t*>(logits), ld, bias,
                   temperature, mask, mask_words, V, k, nchunk, cand);
  } else {
    if (xform) topk_chunk_kernel<float, true><<<ga, 256, 0, stream>>>(static_cast<const float*>(logits), ld, bias,
                   temperature, mask, mask_words, V, k, nchunk, cand);
    else topk_chunk_kernel<float, false><<<ga, 256, 0, stream>>>(static_cast<const float*>(logits), ld, bias,
                   temperature, mask, mask_words, V, k, nchunk, cand);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (seeds)
    topk_final_kernel<true><<<B, 512, 0, stream>>>(cand, nchunk * k, k, top_p, temperature, seed, step, seeds, steps,
                                                   idx_out, score_out, logZ_out, logprob_out);
  else
    topk_final_kernel<false><<<B, 512, 0, stream>>>(cand, nchunk * k, k, top_p, temperature, seed, step, seeds, steps,
                                                    idx_out, score_out, logZ_out, logprob_out);
  return cudaGetLastError();
}

}  // namespace fs
