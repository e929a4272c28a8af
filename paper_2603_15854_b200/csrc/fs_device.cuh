// fs_device.cuh -- per-element arithmetic of the fused epilogue (sm_100a).
//
// Philox4x32-10, the tail-accurate fp32 Gumbel map G32, the order-preserving score key and
// the running (key, idx, S) state used by both stage-1 kernels (tcgen05 and CUDA-core) and
// by the reduction kernels.  See include/flashsample.h for the conventions and DESIGN.md
// for the readings R1-R8 of PAPER.md.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fs {

// ---------------------------------------------------------------------------------------
// Philox4x32-10 ("counter-based RNG (e.g. Philox)"; reading R1).
// ---------------------------------------------------------------------------------------
constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                            uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(kPhiloxM0, c0), lo0 = kPhiloxM0 * c0;
    const uint32_t hi1 = __umulhi(kPhiloxM1, c2), lo1 = kPhiloxM1 * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += kPhiloxW0; k1 += kPhiloxW1;
  }
  return U4{c0, c1, c2, c3};
}

// Word i (0..3, lane-dependent) of (x, y, z, w) with mask arithmetic (3 LOP3 + 2 masks): the
// nested-ternary form compiled to divergent branches + warp reconvergence around the shuffles
// that consume it (ncu: BSSY/BSYNC + branch_resolving stalls in the per-request epilogue).
__device__ __forceinline__ uint32_t sel4(uint32_t x, uint32_t y, uint32_t z, uint32_t w, int i) {
  const uint32_t m1 = 0u - ((uint32_t)i & 1u), m2 = 0u - (((uint32_t)i >> 1) & 1u);
  const uint32_t lo = (x & ~m1) | (y & m1), hi = (z & ~m1) | (w & m1);
  return (lo & ~m2) | (hi & m2);
}

// Per-request draws (reading R18: key = seed_b, counter = (v >> 2, 2^31, step_b), word v & 3) of
// 4 batch columns for a warp whose lanes 4g..4g+3 hold vocabulary ids 4m..4m+3 (one counter per
// lane quartet).  Instead of 4 Philox calls per lane, lane a = lane & 3 evaluates the call of
// column a (its key / counter words k0..c3 are passed in) and 4 shuffle rounds hand every lane
// word (v & 3) of each column: round r, lane s sends word (a_s - r) & 3 and lane d reads lane
// (a_d + r) & 3 of its quartet, i.e. the word of column (a_d + r) & 3.  Warp-converged callers only.
__device__ __forceinline__ void prq_bits4(uint32_t vq, uint32_t k0, uint32_t k1, uint32_t c2, uint32_t c3, int lane,
                                          uint32_t (&rr)[4]);

// Counter words 2 and 3 for (step, tag).
__device__ __forceinline__ uint32_t ctr_step_lo(uint64_t step) { return (uint32_t)step; }
__device__ __forceinline__ uint32_t ctr_step_hi(uint64_t step, uint32_t tag) {
  return ((uint32_t)(step >> 32) & 0x00FFFFFFu) | (tag << 24);
}

__device__ __forceinline__ void prq_bits4(uint32_t vq, uint32_t k0, uint32_t k1, uint32_t c2, uint32_t c3, int lane,
                                          uint32_t (&rr)[4]) {
  const U4 o = philox4x32_10(vq, 0x80000000u, c2, c3, k0, k1);
  const int a = lane & 3;
  // y = (o) rotated left by a (two predicated rotation stages, 8 SEL), so y[r] = o[(a + r) & 3];
  // round r sends o[(a - r) & 3] = y[(4 - r) & 3]
  const bool s1 = a & 1, s2 = a & 2;
  uint32_t t0 = s1 ? o.y : o.x, t1 = s1 ? o.z : o.y, t2 = s1 ? o.w : o.z, t3 = s1 ? o.x : o.w;
  const uint32_t y0 = s2 ? t2 : t0, y1 = s2 ? t3 : t1, y2 = s2 ? t0 : t2, y3 = s2 ? t1 : t3;
  const uint32_t send[4] = {y0, y3, y2, y1};
  uint32_t got[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) got[r] = __shfl_sync(0xFFFFFFFFu, send[r], (lane & ~3) | ((a + r) & 3));
  // rr[c] = got[(c - a) & 3]: got rotated right by a
  t0 = s1 ? got[3] : got[0]; t1 = s1 ? got[0] : got[1]; t2 = s1 ? got[1] : got[2]; t3 = s1 ? got[2] : got[3];
  rr[0] = s2 ? t2 : t0; rr[1] = s2 ? t3 : t1; rr[2] = s2 ? t0 : t2; rr[3] = s2 ? t1 : t3;
}

// ---------------------------------------------------------------------------------------
// G32(r) = -log(-log u), u = (r+1)/(2^32+1)   (App. C; reading R2).
// fp32 with MUFU lg2 only where the result's absolute error is bounded:
//   r <  2^31 : u = (r+1)*2^-32 (1/(2^32+1) rounds to 2^-32 in fp32), E = -ln u >= ln 2,
//               so the abs error of ln u (~2^-22) is a small relative error of E.
//   r >= 2^31 : w = (2^32 - r)*2^-32 = 1 - u <= 1/2, E = -log1p(-w) = 2 atanh(s),
//               s = w/(2-w) <= 1/3, by the odd series 2 s (1 + s^2/3 + ... + s^10/11)
//               (truncation < 1.6e-7 relative), so E keeps full relative accuracy
//               even for w ~ 2^-32.
//   g = -ln E.   Budget |G32 - G64| <= 1e-5 (exhaustive test in tests/test_gpu_rng.py).
// Branch-free: both forms are evaluated and selected, which costs the same as the
// divergent branch in a warp and keeps the epilogue convergent.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ float fast_log2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fast_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

constexpr float kLn2 = 0.69314718055994530942f;
constexpr float kLog2e = 1.44269504088896340736f;
constexpr float kTwoM32 = 2.3283064365386963e-10f;   // 2^-32

__device__ __forceinline__ float gumbel32(uint32_t r) {
  // lower branch: E = -ln u = (32 - log2(r+1)) * ln2
  const float x_lo = (float)(r + 1u);                                // used only for r < 2^31
  const float E_lo = (32.0f - fast_log2(x_lo)) * kLn2;
  // upper branch: w = (2^32 - r) 2^-32, s = w/(2-w) <= 1/3, E = 2 s P(s^2) with
  // P(t) = 1 + t/3 + ... + t^5/11 (truncation <= t^6/13/(1-t) = 1.6e-7 relative at s = 1/3)
  const float w = (float)(0u - r) * kTwoM32;                         // 2^32 - r for r >= 2^31
  const float s = w * fast_rcp(2.0f - w);
  const float t = s * s;
  float p = 1.0f / 11.0f;
  p = fmaf(p, t, 1.0f / 9.0f);
  p = fmaf(p, t, 1.0f / 7.0f);
  p = fmaf(p, t, 1.0f / 5.0f);
  p = fmaf(p, t, 1.0f / 3.0f);
  p = fmaf(p, t, 1.0f);
  const float E_hi = 2.0f * s * p;
  const float E = (r < 0x80000000u) ? E_lo : E_hi;
  return -fast_log2(E) * kLn2;
}

// ---------------------------------------------------------------------------------------
// Order-preserving key: float order == uint32 order (for non-NaN inputs).
// ---------------------------------------------------------------------------------------
__device__ __host__ __forceinline__ uint32_t order_key_bits(uint32_t x) {
  return x ^ ((x & 0x80000000u) ? 0xFFFFFFFFu : 0x80000000u);
}
__device__ __forceinline__ uint32_t order_key(float f) { return order_key_bits(__float_as_uint(f)); }
__device__ __forceinline__ float key_to_float(uint32_t k) {
  const uint32_t x = (k & 0x80000000u) ? (k ^ 0x80000000u) : ~k;
  return __uint_as_float(x);
}
// key(-inf) = ~0xFF800000; key 0 marks "no element" (out-of-range rows), below every score.
constexpr uint32_t kKeyNegInf = 0x007FFFFFu;
constexpr uint32_t kKeyNone = 0u;

// Running state of a (row, vocabulary range): best key, its smallest global id, the log-mass
// S = sum exp(l~ - M) relative to M = key_to_float(key) (App. E), and the transformed
// logit l~ of the best element (float bits; gives log p(idx) = l~_idx - logZ).
struct State {
  uint32_t key;
  int32_t idx;
  float S;
  uint32_t lt;
};

__device__ __forceinline__ State state_empty() { return State{kKeyNone, -1, 0.0f, 0u}; }

__device__ __forceinline__ float key_ref(uint32_t key) {
  return key > kKeyNegInf ? key_to_float(key) : -INFINITY;
}

// Top-k candidate: order key of the transformed logit l~ and its global id.
struct Cand {
  uint32_t key;
  int32_t idx;
};

// Histogram increment of bin d by every active lane of a converged warp.  Radix digits of the
// top-k keys are highly concentrated (similar logits share sign, exponent and leading mantissa
// bits), and same-address shared atomics serialise: the lanes that agree with the first active
// lane's bin are folded into one atomic, the rest add individually.
__device__ __forceinline__ void warp_hist_add(uint32_t* hist, bool act, uint32_t d, int lane) {
  const uint32_t am = __ballot_sync(0xFFFFFFFFu, act);
  if (am == 0u) return;
  const int leader = __ffs(am) - 1;
  const uint32_t dl = __shfl_sync(0xFFFFFFFFu, d, leader);
  const uint32_t same = __ballot_sync(0xFFFFFFFFu, act && d == dl);
  if (lane == leader) atomicAdd(&hist[dl], (uint32_t)__popc(same));
  else if (act && d != dl) atomicAdd(&hist[d], 1u);
}

// Max-merge only (no log-mass): larger key wins, ties -> smaller id.
__device__ __forceinline__ State state_max(State a, State b) {
  const bool take_b = (b.key > a.key) || (b.key == a.key && b.idx >= 0 && (a.idx < 0 || b.idx < a.idx));
  return take_b ? b : a;
}

// Merge two states over disjoint vocabulary sets: max-merge (ties -> smaller id) and
// logaddexp of the masses (binary merge realised by max reuse).
__device__ __forceinline__ State state_merge(State a, State b) {
  const bool take_b = (b.key > a.key) || (b.key == a.key && b.idx >= 0 && (a.idx < 0 || b.idx < a.idx));
  State hi = take_b ? b : a;
  const State lo = take_b ? a : b;
  const float mh = key_ref(hi.key), ml = key_ref(lo.key);
  float S = hi.S;
  if (lo.S > 0.0f && ml != -INFINITY && mh != -INFINITY) S += lo.S * fast_exp2((ml - mh) * kLog2e);
  else if (mh == -INFINITY) S = 0.0f;
  hi.S = S;
  return hi;
}

}  // namespace fs
