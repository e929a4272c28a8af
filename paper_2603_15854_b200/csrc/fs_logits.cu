// fs_logits.cu -- standalone FlashSampling over materialised logits.
//
// Gumbel-max over a [B, V] logits matrix that some other kernel already wrote (§5.2
// P:490-493, Alg. A.1 P:747-763 parallelised like Alg. 2): same transform, RNG layout, tie rule
// and candidate format as the fused path, so fs_sample_logits(h W^T) == fs_sample(h, W) up to the
// fp32 rounding of the logits.  Optionally the log-normalizer and log p(idx) (App. E).
//
// HBM-bound (reads B*V*esz bytes once).  Grid (V blocks) x (B/4): a thread owns one vocabulary
// column v and 4 rows b0..b0+3, so one Philox call serves 4 rows (the counter layout's b>>2) and
// the 4 row reads are each coalesced along v.  Candidates: one per (V block, row).
#include <cuda_bf16.h>

#include <algorithm>

#include "fs_device.cuh"
#include "fs_epilogue.cuh"
#include "fs_sm100.cuh"
#include "fs_kernels.h"

namespace fs {

namespace {

template <typename T>
__device__ __forceinline__ float ld_logit(const T* p) {
  if constexpr (sizeof(T) == 2) return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(p));
  else return *p;
}

__device__ __forceinline__ State shfl_state(const State& a, int o) {
  State r;
  r.key = __shfl_xor_sync(0xFFFFFFFFu, a.key, o);
  r.idx = __shfl_xor_sync(0xFFFFFFFFu, a.idx, o);
  r.S = __shfl_xor_sync(0xFFFFFFFFu, a.S, o);
  r.lt = __shfl_xor_sync(0xFFFFFFFFu, a.lt, o);
  return r;
}

template <typename T, bool XFORM, bool LSE, bool PRQ>
__global__ void __launch_bounds__(256)
logits_sample_kernel(const T* __restrict__ logits, int64_t ld, const float* __restrict__ bias,
                     const float* __restrict__ temperature, const uint32_t* __restrict__ mask, int64_t mask_words,
                     int B, int V, int vpb, uint32_t k0, uint32_t k1, uint32_t c2, uint32_t c3, State* part,
                     int* part_group, const uint64_t* __restrict__ seeds, const uint64_t* __restrict__ steps,
                     uint64_t step, unsigned long long* fin_best, unsigned int* fin_ctr, int32_t* idx_out,
                     float* score_out) {
  __shared__ State red[8][4];
  __shared__ int fin_flag;
  const int b0 = blockIdx.y * 4;
  const int v_begin = blockIdx.x * vpb, v_end = min(V, v_begin + vpb);
  float it[4], gsc[4];
  uint32_t pk0[4], pk1[4], pc2[4], pc3[4];                  // per-request Philox words (R18)
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int b = b0 + j;
    it[j] = __int_as_float(0x7FC00000);
    gsc[j] = 1.0f;
    if (b < B) {
      const float t = (XFORM && temperature) ? temperature[b] : 1.0f;
      if (t == 0.0f) { it[j] = 1.0f; gsc[j] = 0.0f; }       // greedy row
      else if (t > 0.0f && isfinite(t)) it[j] = 1.0f / t;
    }
    if (PRQ) {
      const uint64_t sd = b < B ? seeds[b] : 0ull, st = b < B ? (steps ? steps[b] : step) : 0ull;
      pk0[j] = (uint32_t)sd; pk1[j] = (uint32_t)(sd >> 32);
      pc2[j] = (uint32_t)st; pc3[j] = (uint32_t)(st >> 32) & 0x00FFFFFFu;
    }
  }
  State st[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) st[j] = state_empty();
  // 4 columns per iteration (v, v+256, v+512, v+768): all 16 loads issued before the RNG work
  // warp-uniform trip count (the per-request exchange shuffles across the warp); lanes past
  // v_end load -inf and are masked below
  for (int vw = v_begin + (int)(threadIdx.x & ~31u); vw < v_end; vw += 1024) {
    const int v0 = vw + (int)(threadIdx.x & 31u);
    float lv[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int v = v0 + 256 * u;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        lv[u][j] = (v < v_end && b0 + j < B) ? ld_logit(logits + (int64_t)(b0 + j) * ld + v) : -INFINITY;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int v = v0 + 256 * u;
      uint32_t rr[4];
      if (PRQ) {
        // lane quartets hold v = 4m..4m+3 (v_begin % 4 == 0): one Philox per 4 elements, computed
        // before the range test so that the whole warp takes part in the exchange
        const int a = threadIdx.x & 3;
        prq_bits4((uint32_t)v >> 2, sel4(pk0[0], pk0[1], pk0[2], pk0[3], a), sel4(pk1[0], pk1[1], pk1[2], pk1[3], a),
                  sel4(pc2[0], pc2[1], pc2[2], pc2[3], a), sel4(pc3[0], pc3[1], pc3[2], pc3[3], a),
                  (int)(threadIdx.x & 31), rr);
      }
      if (v >= v_end) continue;
      if (!PRQ) {
        const U4 r4 = philox4x32_10((uint32_t)v, (uint32_t)b0 >> 2, c2, c3, k0, k1);
        rr[0] = r4.x; rr[1] = r4.y; rr[2] = r4.z; rr[3] = r4.w;
      }
      const float bv = (XFORM && bias) ? bias[v] : 0.0f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int b = b0 + j;
        if (b >= B) break;                                   // block-uniform
        float l = lv[u][j];
        if (XFORM) {
          l = (l + bv) * it[j];
          if (mask && !((mask[(int64_t)b * mask_words + (v >> 5)] >> (v & 31)) & 1u)) l = -INFINITY;
        }
        if (isnan(l)) l = -INFINITY;
        const float s = l + gumbel32(rr[j]) * gsc[j];
        const uint32_t key = order_key(s);
        if (key > st[j].key) {                               // v ascends per thread: ties keep smaller v
          if (LSE) {
            st[j].S = (st[j].key > kKeyNegInf ? st[j].S * fast_exp2((key_ref(st[j].key) - s) * kLog2e) : 0.0f) +
                      (s != -INFINITY ? fast_exp2((l - s) * kLog2e) : 0.0f);
            st[j].lt = __float_as_uint(l);
          }
          st[j].key = key;
          st[j].idx = v;
        } else if (LSE && st[j].key > kKeyNegInf) {
          st[j].S += fast_exp2((l - key_ref(st[j].key)) * kLog2e);
        }
      }
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    State x = st[j];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const State y = shfl_state(x, o);
      if (LSE) x = (lane & o) ? state_merge(y, x) : state_merge(x, y);
      else x = state_max(x, y);
    }
    if (lane == 0) red[warp][j] = x;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    const int j = threadIdx.x, b = b0 + j;
    State x = red[0][j];
#pragma unroll
    for (int w = 1; w < 8; ++w) x = LSE ? state_merge(x, red[w][j]) : state_max(x, red[w][j]);
    if (b < B) {
      if (!LSE && fin_best) {                   // one-kernel finalize (fs_epilogue.cuh)
        if (x.key != kKeyNone) atomicMax(&fin_best[b], pack_state(x));
      } else {
        part[(size_t)blockIdx.x * B + b] = x;
      }
    }
  }
  if (!LSE && fin_best) {
    finalize_last_cta(fin_best, fin_ctr, B, idx_out, score_out, threadIdx.x, 256, 1, &fin_flag,
                      gridDim.x * gridDim.y);
    return;
  }
  if (threadIdx.x == 0 && blockIdx.y == 0) part_group[blockIdx.x] = 0;
  sm100::pdl_launch_dependents();
}

}  // namespace

cudaError_t launch_logits_sample(fs_dtype dtype, const void* logits, int64_t ld, const float* bias,
                                 const float* temperature, const uint32_t* mask, int64_t mask_words, int B, int V,
                                 uint64_t seed, uint64_t step, bool lse, int nblk, State* part, int* part_group,
                                 cudaStream_t stream, const uint64_t* seeds, const uint64_t* steps,
                                 unsigned long long* fin_best, unsigned int* fin_ctr, int32_t* idx_out,
                                 float* score_out) {
  const int vpb = ((V + nblk - 1) / nblk + 255) / 256 * 256;
  const dim3 grid((V + vpb - 1) / vpb, (B + 3) / 4);
  const bool xform = bias || temperature || mask || seeds;
  const bool prq = seeds != nullptr;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const uint32_t c2 = (uint32_t)step, c3 = (uint32_t)(step >> 32) & 0x00FFFFFFu;
#define FS_LAUNCH(T, X, L, P)                                                                                 \
  logits_sample_kernel<T, X, L, P><<<grid, 256, 0, stream>>>(static_cast<const T*>(logits), ld, bias, temperature, \
                                                             mask, mask_words, B, V, vpb, k0, k1, c2, c3, part,  \
                                                             part_group, seeds, steps, step, fin_best, fin_ctr, \
                                                             idx_out, score_out)
#define FS_DISPATCH(T)                                                                                         \
  if (prq) { if (lse) FS_LAUNCH(T, true, true, true); else FS_LAUNCH(T, true, false, true); }                  \
  else if (xform) { if (lse) FS_LAUNCH(T, true, true, false); else FS_LAUNCH(T, true, false, false); }          \
  else { if (lse) FS_LAUNCH(T, false, true, false); else FS_LAUNCH(T, false, false, false); }
  if (dtype == FS_BF16) { FS_DISPATCH(uint16_t) } else { FS_DISPATCH(float) }
#undef FS_DISPATCH
#undef FS_LAUNCH
  return cudaGetLastError();
}

int logits_sample_blocks(int B, int V) {
  // ~16 columns per thread (4096 per block) so each thread has few dependent iterations, but at
  // least 2 waves of 148 SMs over (V blocks) x (B/4) and at least 256 columns per block
  const int rows4 = (B + 3) / 4;
  int nblk = std::max((V + 4095) / 4096, (2 * 148 + rows4 - 1) / rows4);
  nblk = std::max(1, std::min(nblk, (V + 255) / 256));
  const int vpb = ((V + nblk - 1) / nblk + 255) / 256 * 256;
  return (V + vpb - 1) / vpb;
}

}  // namespace fs
