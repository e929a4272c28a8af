// fs_epilogue.cuh -- the fused epilogue of Alg. 2 shared by the tcgen05
// stage-1 kernel and the CUDA-core stage-1 kernel.
//
// Thread <-> data mapping (swap-AB): one thread owns one vocabulary row v (a TMEM lane), a warp
// owns 32 consecutive rows; the accumulator columns are the batch rows b.  For each column b:
//   l~ = (acc + bias_v) * invtau_b, banned / NaN -> -inf          (Alg. 2 line 9; §4.6)
//   g  = G32(Philox(v, b>>2, step)[b&3])                           (line 10; App. C)
//   s  = l~ + g, key = order-preserving uint32 of s               (line 11)
//   warp max of key (redux.sync) + ballot -> smallest winning lane (= smallest v, reading R5)
//   lane (b mod 32) folds (kmax, v_win[, S_w]) into its running State for column b (line 14).
// With LSE the warp also sums exp(l~ - M_w) (App. E), M_w = warp max perturbed score:
// since -3.10 <= g <= 22.19, every l~ - M_w <= 3.1 and the max term is >= e^-22.2, so the
// fp32 sum neither overflows nor underflows (reading R9).
#pragma once
#include "../../include/flashsample.h"
#include "fs_device.cuh"
#include "fs_peer.cuh"
#include "fs_sm100.cuh"

namespace fs {

// Per-batch-column constants of one launch, staged in shared memory at kernel start.
struct RowTab {
  float invtau[256];        // 1/tau_b (1 for greedy rows), NaN for invalid or padding columns
  float gscale[256];        // noise scale: 1 sampled, 0 greedy (tau == 0; reading R18)
  uint32_t k0[256], k1[256], c2[256], c3[256];   // per-request Philox key / counter words (R18)
};

// Fill the table (all threads of the CTA; caller synchronises).
template <bool PRQ>
__device__ __forceinline__ void fill_rowtab(RowTab* t, int B, const float* temperature, const uint64_t* seeds,
                                            const uint64_t* steps, uint64_t step, int tid, int nthreads) {
  for (int b = tid; b < 256; b += nthreads) {
    float it = __int_as_float(0x7FC00000), gsc = 1.0f;
    if (b < B) {
      const float tau = temperature ? temperature[b] : 1.0f;
      if (tau == 0.0f) { it = 1.0f; gsc = 0.0f; }
      else if (tau > 0.0f && isfinite(tau)) it = 1.0f / tau;
    }
    t->invtau[b] = it;
    t->gscale[b] = gsc;
    if (PRQ) {
      const uint64_t sd = b < B ? seeds[b] : 0ull;
      const uint64_t st = b < B ? (steps ? steps[b] : step) : 0ull;
      t->k0[b] = (uint32_t)sd;
      t->k1[b] = (uint32_t)(sd >> 32);
      t->c2[b] = (uint32_t)st;
      t->c3[b] = (uint32_t)(st >> 32) & 0x00FFFFFFu;
    }
  }
}

// Per-request draw for (vocabulary id v, batch column b): Philox at counter
// (v >> 2, 2^31, step_b) under key seed_b, word v & 3 (reading R18).
__device__ __forceinline__ uint32_t per_request_bits(const RowTab* t, uint32_t v, int b) {
  const U4 o = philox4x32_10(v >> 2, 0x80000000u, t->c2[b], t->c3[b], t->k0[b], t->k1[b]);
  return sel4(o.x, o.y, o.z, o.w, (int)(v & 3u));
}

struct EpiArgs {
  const float* invtau;      // smem [BN]: 1/tau_b, NaN for invalid or padding columns
  const RowTab* tab;        // smem row table (invtau, gscale, per-request RNG words)
  const uint32_t* mask;     // global [rows][mask_words] for this launch's rows, or nullptr
  int64_t mask_words;
  int B;                    // valid columns in this launch
  int row_offset;           // global batch index of column 0 (RNG counter)
  uint32_t k0, k1, c2, c3;  // Philox key and counter words 2, 3
  int dbg_skip;             // debug: drain TMEM without computing (bounds the MMA+TMA-only time)
  int need_lt;              // log-mass epilogue: also carry the winner's l~ (only log-prob outputs read it)
};

// One-kernel finalize (StageOneParams::fin_best).  The candidate order of state_merge (larger key,
// then smaller id) is the unsigned order of (key << 32 | ~idx), so a 64-bit atomicMax per row
// reduces the per-CTA candidates in L2 in any arrival order with the same result as stage 2.
__device__ __forceinline__ unsigned long long pack_state(const State& s) {
  return ((unsigned long long)s.key << 32) | (unsigned long long)(s.idx >= 0 ? ~(uint32_t)s.idx : 0u);
}


struct RowArgs {
  bool valid;               // this lane's vocabulary row is inside the tile
  uint32_t v_lo;            // low word of the global vocabulary id (Philox counter word 0)
  int32_t v_global;         // global vocabulary id
  int32_t warp_v0;          // global id of lane 0's row (rows of a warp are consecutive)
  float bias;
};

// Fold the warp result for one column into the owning lane's running state.  Tiles reach a
// warp in increasing vocabulary order, so a strictly larger key wins and an equal key keeps
// the earlier (smaller) id.
template <bool LSE>
__device__ __forceinline__ void absorb(State& own, uint32_t kmax, int32_t widx, float S_w, float ltw = 0.0f) {
  if (kmax > own.key) {
    if (LSE) {
      const float m_old = key_ref(own.key), m_new = key_ref(kmax);
      own.S = (own.key > kKeyNegInf ? own.S * fast_exp2((m_old - m_new) * kLog2e) : 0.0f) + S_w;
      own.lt = __float_as_uint(ltw);
    }
    own.key = kmax;
    own.idx = widx;
  } else if (LSE) {
    if (kmax > kKeyNegInf) own.S += S_w * fast_exp2((key_ref(kmax) - key_ref(own.key)) * kLog2e);
  }
}

// Process NCOL (multiple of 4) consecutive accumulator columns [col0, col0+NCOL) of this lane's
// row; `own` is this lane's state for column col0 + lane.
template <int NCOL, bool LSE, bool PRQ = false>
__device__ __forceinline__ void epi_columns(const float* acc, int col0, const RowArgs& ra,
                                            const EpiArgs& ea, State& own, int lane) {
#pragma unroll
  for (int j = 0; j < NCOL; j += 4) {
    const int b0 = col0 + j;
    if (b0 >= ea.B) break;                                   // warp-uniform
    uint32_t rr[4];
    if (PRQ) {
      if (ra.warp_v0 & 3) {
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) rr[jj] = per_request_bits(ea.tab, ra.v_lo, b0 + jj);
      } else {
        const int bq = b0 + (lane & 3);
        prq_bits4(ra.v_lo >> 2, ea.tab->k0[bq], ea.tab->k1[bq], ea.tab->c2[bq], ea.tab->c3[bq], lane, rr);
      }
    } else {
      const U4 r4 = philox4x32_10(ra.v_lo, (uint32_t)(ea.row_offset + b0) >> 2, ea.c2, ea.c3, ea.k0, ea.k1);
      rr[0] = r4.x; rr[1] = r4.y; rr[2] = r4.z; rr[3] = r4.w;
    }
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int b = b0 + jj;
      float lt = (acc[j + jj] + ra.bias) * ea.invtau[b];
      if (ea.mask != nullptr && b < ea.B && ra.valid) {     // padding rows past V read no mask word
        const uint32_t w = __ldg(ea.mask + (int64_t)b * ea.mask_words + (ra.v_global >> 5));
        if (!((w >> (ra.v_global & 31)) & 1u)) lt = -INFINITY;
      }
      if (isnan(lt)) lt = -INFINITY;
      const float s = lt + gumbel32(rr[jj]) * ea.tab->gscale[b];
      const uint32_t key = ra.valid ? order_key(s) : kKeyNone;
      const uint32_t kmax = __reduce_max_sync(0xFFFFFFFFu, key);
      const uint32_t ball = __ballot_sync(0xFFFFFFFFu, key == kmax);
      const int32_t widx = kmax > kKeyNone ? ra.warp_v0 + (__ffs(ball) - 1) : -1;
      float S_w = 0.0f;
      if (LSE) {
        const float m = key_ref(kmax);
        float e = (ra.valid && m != -INFINITY) ? fast_exp2((lt - m) * kLog2e) : 0.0f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xFFFFFFFFu, e, o);
        S_w = e;
      }
      const float ltw = LSE ? __shfl_sync(0xFFFFFFFFu, lt, kmax > kKeyNone ? __ffs(ball) - 1 : 0) : 0.0f;
      if (lane == ((j + jj) & 31)) absorb<LSE>(own, kmax, widx, S_w, ltw);
    }
  }
}

// Merge the per-warp states of the 4 TMEM lane quadrants (one epilogue warp each) for every
// column and write one candidate per column to `part_row` (Alg. 2 line 15).
template <int NCHUNK, int COLS_PER_CHUNK>
__device__ __forceinline__ void flush_states(State (&st)[NCHUNK], State* scratch, int BN, int q, int lane,
                                             int epi_tid, int B, State* part_row, uint32_t bar_id) {
#pragma unroll
  for (int c = 0; c < NCHUNK; ++c) {
    if (lane < COLS_PER_CHUNK) scratch[q * BN + c * COLS_PER_CHUNK + lane] = st[c];
    st[c] = state_empty();
  }
  sm100::named_bar_sync(bar_id, 128);
  for (int b = epi_tid; b < B; b += 128) {
    State m = scratch[b];
#pragma unroll
    for (int qq = 1; qq < 4; ++qq) m = state_merge(m, scratch[qq * BN + b]);
    part_row[b] = m;
  }
  sm100::named_bar_sync(bar_id, 128);
}

// ---------------------------------------------------------------------------------------------
// tcgen05 epilogue: one warp processes its 32 TMEM lanes (vocabulary rows) x all B columns of one
// accumulator tile, in rolled groups of 8 columns.  Per group: issue the TMEM load, generate the
// 8 Philox/Gumbel draws (independent of the accumulator, so they overlap the load), wait, then
// transform + key + warp argmax for the 8 columns back to back (independent chains).
// Running states: st[c] holds this lane's state for column 32c + lane; chunk c is processed at
// st[0] and the array is rotated, so the loops stay rolled (small code, no local memory).
// ---------------------------------------------------------------------------------------------
template <int NST>
__device__ __forceinline__ void rotate_states(State (&st)[NST]) {
  const State t = st[0];
#pragma unroll
  for (int i = 0; i < NST - 1; ++i) st[i] = st[i + 1];
  st[NST - 1] = t;
}

// Release of the accumulator buffer after the tile's last TMEM read: every thread arrives on the
// local barrier (1-CTA kernel, count 128) or lane 0 of each warp arrives on the pair leader's
// barrier (CTA-pair kernel, count 8); tempty_cluster != 0 selects the latter.
__device__ __forceinline__ void release_tmem(uint64_t* tempty, uint32_t tempty_cluster, int lane) {
  sm100::tc_fence_before();
  if (tempty_cluster) {
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive_cluster(tempty_cluster);
  } else {
    sm100::mbar_arrive(tempty);
  }
}

// NG groups of 8 columns per iteration (NG = 2 doubles the independent work in flight: 4 Philox
// chains, 16 Gumbel evaluations, 16 warp reductions -- the epilogue is latency-bound at one warp
// pair per SM sub-partition).  Columns >= B are computed on padding and never stored.
// The warp processes the 32-column chunks c = chunk0, chunk0 + cstep, ... (cstep 2: two warps
// per TMEM lane quadrant split a tile's columns); st[i] holds its i-th chunk.
template <bool LSE, bool XFORM, int NG, bool PRQ = false, int NST = 8>
__device__ __forceinline__ void epi_tile_tc(uint32_t taddr, const RowArgs& ra, const EpiArgs& ea, State (&st)[NST],
                                            int lane, uint64_t* tempty, uint32_t tempty_cluster = 0, int chunk0 = 0,
                                            int cstep = 1) {
  constexpr int NC = 8 * NG;
  const int B = ea.B;
  const int nch = (B + 31) >> 5;
  const int nmine = nch > chunk0 ? (nch - chunk0 + cstep - 1) / cstep : 0;
  if (nmine == 0) {                                   // nothing in this tile for this warp
    release_tmem(tempty, tempty_cluster, lane);
    return;
  }
#pragma unroll 1
  for (int c = chunk0; c < nch; c += cstep) {
    State own = st[0];
#pragma unroll 1
    for (int g = 0; g < 4; g += NG) {
      const int col0 = c * 32 + g * 8;
      if (col0 >= B) break;
      uint32_t r[NC];
#pragma unroll
      for (int i = 0; i < NG; ++i)
        sm100::tmem_ld_32x32b_x8(taddr + (uint32_t)(col0 + 8 * i), *reinterpret_cast<uint32_t(*)[8]>(&r[8 * i]));
      if (ea.dbg_skip) {
        sm100::tmem_wait_ld();
        if (col0 + NC >= B || (c + cstep >= nch && g + NG >= 4)) release_tmem(tempty, tempty_cluster, lane);
        if (r[0] == 0x7FFFFFFFu && r[NC - 1] == 0x7FFFFFFFu) own.key = 1u;   // keep the loads live
        continue;
      }
      // mask words for these columns: lane j < 16 holds word (col0+j, w0), lane 16+j word
      // (col0+j, w0+1), w0 = first word of the warp's 32 rows (rows may straddle two words)
      uint32_t mw = 0xFFFFFFFFu;
      const int wshift = ra.warp_v0 & 31;
      const int msrc = ((lane + wshift) >> 5) << 4, mbit = (lane + wshift) & 31;
      if (XFORM && ea.mask != nullptr) {
        const int jb = col0 + (lane & 15);
        const int64_t w = (int64_t)(ra.warp_v0 >> 5) + (lane >> 4);
        mw = 0u;
        if ((lane & 15) < NC && jb < B && w < ea.mask_words) mw = __ldg(ea.mask + (int64_t)jb * ea.mask_words + w);
      }
      // randomness: independent of the accumulator, overlaps the TMEM load
      uint32_t rb[NC];
      if (PRQ && (ra.warp_v0 & 3)) {             // unaligned shard offset: one Philox per element
#pragma unroll
        for (int jj = 0; jj < NC; ++jj) rb[jj] = per_request_bits(ea.tab, ra.v_lo, col0 + jj);
      } else if (PRQ) {                          // lane quartets share v >> 2: one Philox per 4 elements
#pragma unroll
        for (int qq = 0; qq < NC / 4; ++qq) {
          const int bq = col0 + 4 * qq + (lane & 3);
          uint32_t rr[4];
          prq_bits4(ra.v_lo >> 2, ea.tab->k0[bq], ea.tab->k1[bq], ea.tab->c2[bq], ea.tab->c3[bq], lane, rr);
#pragma unroll
          for (int c = 0; c < 4; ++c) rb[4 * qq + c] = rr[c];
        }
      } else {
        const uint32_t qd = (uint32_t)(ea.row_offset + col0) >> 2;
#pragma unroll
        for (int qq = 0; qq < NC / 4; ++qq) {
          const U4 p4 = philox4x32_10(ra.v_lo, qd + (uint32_t)qq, ea.c2, ea.c3, ea.k0, ea.k1);
          rb[4 * qq + 0] = p4.x;
          rb[4 * qq + 1] = p4.y;
          rb[4 * qq + 2] = p4.z;
          rb[4 * qq + 3] = p4.w;
        }
      }
      float gm[NC];
#pragma unroll
      for (int jj = 0; jj < NC; ++jj) gm[jj] = gumbel32(rb[jj]);
      sm100::tmem_wait_ld();
      if (col0 + NC >= B || (c + cstep >= nch && g + NG >= 4))        // this warp's last TMEM read
        release_tmem(tempty, tempty_cluster, lane);
      uint32_t key[NC];
      float lt[NC];
#pragma unroll
      for (int jj = 0; jj < NC; ++jj) {
        float l = __uint_as_float(r[jj]);
        float gj = gm[jj];
        if (XFORM) {
          l = (l + ra.bias) * ea.invtau[col0 + jj];
          gj *= ea.tab->gscale[col0 + jj];              // 0 on greedy rows
          if (ea.mask != nullptr) {
            // bit of row warp_v0 + lane sits in word (lane + wshift) >> 5 (lanes 0-15 / 16-31)
            const uint32_t w = __shfl_sync(0xFFFFFFFFu, mw, msrc + jj);
            if (!((w >> mbit) & 1u)) l = -INFINITY;
          }
        }
        if (isnan(l)) l = -INFINITY;
        lt[jj] = l;
        key[jj] = ra.valid ? order_key(l + gj) : kKeyNone;
      }
      uint32_t kmax[NC], ball[NC];
#pragma unroll
      for (int jj = 0; jj < NC; ++jj) kmax[jj] = __reduce_max_sync(0xFFFFFFFFu, key[jj]);
#pragma unroll
      for (int jj = 0; jj < NC; ++jj) ball[jj] = __ballot_sync(0xFFFFFFFFu, key[jj] == kmax[jj]);
      // the owner lane of column col0+jj is g*8+jj: select its column's result (no branches)
      const int jo = lane - g * 8;
      uint32_t km = 0u, bl = 0u;
#pragma unroll
      for (int jj = 0; jj < NC; ++jj) {
        km = (jo == jj) ? kmax[jj] : km;
        bl = (jo == jj) ? ball[jj] : bl;
      }
      const int32_t wi = km > kKeyNone ? ra.warp_v0 + (__ffs(bl) - 1) : -1;
      const bool mine = (unsigned)jo < (unsigned)NC;
      if (LSE) {
        // e = exp(l~ - M_col) per element; warp sums by a reduce-scatter butterfly: after log2(NC)
        // halving steps lane L holds column L >> (5 - log2 NC), the remaining xor steps finish
        // the 32-lane sum (2 shuffles per column instead of 5).
        float ev[NC];
#pragma unroll
        for (int jj = 0; jj < NC; ++jj) {
          const float m = key_ref(kmax[jj]);
          ev[jj] = (ra.valid && m != -INFINITY) ? fast_exp2((lt[jj] - m) * kLog2e) : 0.0f;
        }
        int n = NC, bit = 16;
#pragma unroll
        for (int st2 = 0; st2 < 4; ++st2) {
          if (n > 1) {
            const bool upper = (lane & bit) != 0;
            const int h2 = n >> 1;
#pragma unroll
            for (int i2 = 0; i2 < 8; ++i2) {
              if (i2 < h2) {
                const float keep = upper ? ev[h2 + i2] : ev[i2];
                const float send = upper ? ev[i2] : ev[h2 + i2];
                ev[i2] = keep + __shfl_xor_sync(0xFFFFFFFFu, send, bit);
              }
            }
            n = h2;
            bit >>= 1;
          }
        }
        float v = ev[0];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
          if (o <= bit) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        constexpr int kShift = (NC == 16) ? 1 : 2;          // column of lane L = L >> kShift
        const float Sw = __shfl_sync(0xFFFFFFFFu, v, (jo & (NC - 1)) << kShift);
        float ltw = 0.0f;                                    // l~ of each column's winner (log-prob only)
        if (ea.need_lt) {
#pragma unroll
          for (int jj = 0; jj < NC; ++jj) {
            const float x = __shfl_sync(0xFFFFFFFFu, lt[jj], kmax[jj] > kKeyNone ? __ffs(ball[jj]) - 1 : 0);
            ltw = (jo == jj) ? x : ltw;
          }
        }
        if (mine) absorb<true>(own, km, wi, Sw, ltw);
      } else {
        const bool upd = mine && (km > own.key);       // ties keep the earlier (smaller) id
        own.key = upd ? km : own.key;
        own.idx = upd ? wi : own.idx;
      }
    }
    st[0] = own;
    if (nmine > 1) rotate_states(st);
  }
  if (nmine > 1)
#pragma unroll 1
    for (int i = nmine; i < NST; ++i) rotate_states(st);    // restore chunk order
}

// Write this warp's states (one candidate per column for its 32 rows of every tile it saw in
// the segment) to its own candidate slot; stage 2 merges slots (no intra-CTA barrier needed).
template <int NST>
__device__ __forceinline__ void flush_warp(State (&st)[NST], int lane, int B, State* part_row, int chunk0 = 0,
                                           int cstep = 1) {
#pragma unroll
  for (int c = 0; c < NST; ++c) {
    const int b = (chunk0 + c * cstep) * 32 + lane;
    if (b < B) part_row[b] = st[c];
    st[c] = state_empty();
  }
}

// One-kernel finalize, last step (pack_state above).
// Called by all `nthr` epilogue threads (ids et) of every CTA after their atomicMax calls: the last
// CTA to arrive (threadFenceReduction pattern) converts the row maxima to (idx, score) exactly as
// stage 2's to_summary does, and leaves fin_best / fin_ctr at 0 for the next call.
// With in-kernel staging (h_bar != nullptr), h_bar[1] is the staging-timeout flag (wait_h_staged):
// when set, h was not fully staged before some CTA's first h load, so every row is reported
// undefined (idx -1, score -inf) and h_bar[2] counts the event (fs_ctx_query "staging_timeouts").
// With sum_out (a TP shard step that needs no log-mass, fs_sample_tp without logZ) the row maxima are
// written as the shard's exchange records {M, I, L = NaN} instead of idx / score.
// With done_flag (option "done_flag", pinned host memory): 1 is stored with system-scope release
// after the outputs, so a serving loop can spin on it instead of synchronising the stream.
// With push->peers (f2 fully fused, a TP step without log-mass): the records also go into every
// peer's exchange window, and the same CTA then waits for the n ranks' records, runs the outer
// selection (Alg. A.4 lines 5-7) into idx_out / score_out and acknowledges the epoch -- the whole
// sharded step is this one kernel per rank.  `flag` needs 2 ints of shared scratch.
__device__ __forceinline__ void finalize_last_cta(unsigned long long* best, unsigned int* ctr, int B,
                                                  int32_t* idx_out, float* score_out, int et, int nthr,
                                                  uint32_t bar_id, volatile int* flag, unsigned n_ctas,
                                                  unsigned int* h_bar = nullptr, fs_summary* sum_out = nullptr,
                                                  const PushCtx* push = nullptr,
                                                  unsigned long long* done_flag = nullptr) {
  __threadfence();
  sm100::named_bar_sync(bar_id, nthr);
  if (et == 0) *flag = (atomicAdd(ctr, 1u) == n_ctas - 1) ? 1 : 0;
  sm100::named_bar_sync(bar_id, nthr);
  if (*flag) {
    __threadfence();
    const bool timed_out = h_bar != nullptr && *reinterpret_cast<volatile unsigned int*>(h_bar + 1) != 0u;
    const bool pushing = push != nullptr && push->peers != nullptr;
    if (pushing) {                             // readers are done with this parity slot
      if (et == 0) flag[1] = 1;
      push_wait_readers(*push, et);
      sm100::named_bar_sync(bar_id, nthr);
    }
    for (int b = et; b < B; b += nthr) {
      const unsigned long long v = atomicExch(&best[b], 0ull);
      const uint32_t key = (uint32_t)(v >> 32);
      const bool defined = key > kKeyNegInf && !timed_out;
      const int32_t id = defined ? (int32_t)~(uint32_t)v : -1;
      const float sc = defined ? key_to_float(key) : -INFINITY;
      const fs_summary f{sc, id, __int_as_float(0x7FC00000)};
      if (!pushing) {
        if (idx_out) idx_out[b] = id;
        if (score_out) score_out[b] = sc;
      }
      if (sum_out) sum_out[b] = f;
      if (pushing) push_record(*push, b, f);
    }
    sm100::named_bar_sync(bar_id, nthr);     // every thread read the timeout flag
    if (done_flag && !pushing && et == 0) {   // host completion flag (pinned): after every output store
      __threadfence_system();
      st_release_sys(reinterpret_cast<uint64_t*>(done_flag), 1ull);
    }
    if (pushing) {
      if (et == 0) push_release(*push);        // fence.sys + this rank's flag in every window
      sm100::named_bar_sync(bar_id, nthr);
      const int par = (int)(push->epoch & 1);
      const PeerTab& pt = *push->peers;
      if (et < push->world &&
          !wait_flag(pt.flags[push->rank] + par * push->world + et, [&](uint64_t v) { return v == push->epoch; }))
        flag[1] = 0;
      sm100::named_bar_sync(bar_id, nthr);
      const bool ok = flag[1] != 0;
      const fs_summary* rec = pt.rec[push->rank] + (size_t)par * push->world * push->B_max;
      for (int b = et; b < B; b += nthr) {
        State acc = state_empty();
        for (int k = 0; k < push->world; ++k) {
          const fs_summary m = rec[(size_t)k * push->B_max + b];
          State s1 = state_empty();
          if (m.idx >= 0 && !(m.max_score == -INFINITY)) {
            s1.key = order_key(m.max_score);
            s1.idx = m.idx;
          }
          acc = state_max(acc, s1);            // ties -> smaller global id (reading R5)
        }
        const bool defined = acc.key > kKeyNegInf && ok;
        if (idx_out) idx_out[b] = defined ? acc.idx : -1;
        if (score_out) score_out[b] = defined ? key_to_float(acc.key) : -INFINITY;
      }
      sm100::named_bar_sync(bar_id, nthr);
      if (et == 0) {
        if (!ok) atomicAdd(push->timeouts, 1u);
        for (int q = 0; q < push->world; ++q) st_release_sys(pt.acks[q] + push->rank, push->epoch);
      }
    }
    if (et == 0) {
      atomicExch(ctr, 0u);
      if (h_bar) {
        atomicExch(h_bar, 0u);               // every CTA passed the staging barrier long ago
        if (timed_out) {
          atomicExch(h_bar + 1, 0u);
          atomicAdd(h_bar + 2, 1u);
        }
      }
    }
  }
}

// Summary record of a state (Lemma P:254-270): M, I, L = M + log S; undefined -> (-inf, -1, -inf).
__device__ __forceinline__ fs_summary to_summary(const State& s) {
  fs_summary o;
  const bool defined = s.key > kKeyNegInf;
  o.max_score = defined ? key_to_float(s.key) : -INFINITY;
  o.idx = defined ? s.idx : -1;
  o.log_mass = (defined && s.S > 0.0f) ? o.max_score + logf(s.S) : -INFINITY;
  return o;
}

// log p(idx) = l~_idx - logZ (App. E); -inf when the row is undefined.
__device__ __forceinline__ float logprob_of(const State& s) {
  const fs_summary f = to_summary(s);
  return f.idx >= 0 && f.log_mass > -INFINITY ? __uint_as_float(s.lt) - f.log_mass : -INFINITY;
}

// Stage 2 of one batch row b (Alg. 2; App. E), one warp: lane L merges slots L, L+32, ...
// (L2 loads, so a last CTA of the same grid may call it), then a fixed xor tree -- deterministic,
// so logZ is bit-reproducible and identical whichever kernel runs it.
// With `push` (f2), the row's summary record is also stored into every peer's exchange window.
__device__ __forceinline__ void reduce_row(const State* part, const int* part_group, int n_slots, int B, int b,
                                           int lane, int32_t* idx_out, float* score_out, float* logZ_out,
                                           fs_summary* groups_out, float* logprob_out,
                                           const PushCtx* push = nullptr) {
  State acc = state_empty();
#pragma unroll 4
  for (int s = lane; s < n_slots; s += 32)
    if (__ldcg(part_group + s) >= 0) {
      const uint4 u = __ldcg(reinterpret_cast<const uint4*>(part + (size_t)s * B + b));
      acc = state_merge(acc, State{u.x, (int32_t)u.y, __uint_as_float(u.z), u.w});
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    State other;
    other.key = __shfl_xor_sync(0xFFFFFFFFu, acc.key, o);
    other.idx = __shfl_xor_sync(0xFFFFFFFFu, acc.idx, o);
    other.S = __shfl_xor_sync(0xFFFFFFFFu, acc.S, o);
    other.lt = __shfl_xor_sync(0xFFFFFFFFu, acc.lt, o);
    acc = (lane & o) ? state_merge(other, acc) : state_merge(acc, other);
  }
  if (lane == 0) {
    const fs_summary f = to_summary(acc);
    if (idx_out) idx_out[b] = f.idx;
    if (score_out) score_out[b] = f.max_score;
    if (logZ_out) logZ_out[b] = f.log_mass;
    if (groups_out) groups_out[b] = f;
    if (logprob_out) logprob_out[b] = logprob_of(acc);
    if (push) push_record(*push, b, f);
  }
}

// One-kernel finalize with log-mass (single group, small B): every CTA has written its candidate
// slot (part, part_group); the last CTA to arrive runs stage 2's reduce_row for every row, one warp
// per row, and resets the counter.
// With push.peers (f2, a TP shard step) the same CTA stores every row's summary into the peers'
// exchange windows and releases this rank's flags: the exchange needs no extra kernel before the
// wait + combine.
__device__ __forceinline__ void finalize_lse_last_cta(const State* part, const int* part_group, int B,
                                                      unsigned int* ctr, int32_t* idx_out, float* score_out,
                                                      float* logZ_out, fs_summary* groups_out, float* logprob_out,
                                                      int et, int nthr, uint32_t bar_id, volatile int* flag,
                                                      const PushCtx& push) {
  __threadfence();
  sm100::named_bar_sync(bar_id, nthr);
  if (et == 0) *flag = (atomicAdd(ctr, 1u) == gridDim.x - 1) ? 1 : 0;
  sm100::named_bar_sync(bar_id, nthr);
  if (*flag) {
    __threadfence();
    const bool pushing = push.peers != nullptr;
    if (pushing) {                             // readers are done with this parity slot
      push_wait_readers(push, et);
      sm100::named_bar_sync(bar_id, nthr);
    }
    const int w = et >> 5, nw = nthr >> 5, lane = et & 31;
    for (int b = w; b < B; b += nw)
      reduce_row(part, part_group, gridDim.x, B, b, lane, idx_out, score_out, logZ_out, groups_out, logprob_out,
                 pushing ? &push : nullptr);
    if (pushing) sm100::named_bar_sync(bar_id, nthr);
    if (et == 0) {
      atomicExch(ctr, 0u);
      if (pushing) push_release(push);
    }
  }
}

// In-kernel input staging (StageOneParams::h_host): the `nthr` non-producer threads of every CTA
// copy this CTA's slice of the pinned host h into the device h (past the dependency wait, so the
// previous kernel no longer reads it), fence, and one thread arrives on the grid counter.
__device__ __forceinline__ void stage_h_slice(const void* h_host, const void* h_dev, size_t bytes, int et, int nthr,
                                              uint32_t bar_id, unsigned int* h_bar) {
  const size_t n16 = bytes / 16;
  const size_t per = (n16 + gridDim.x - 1) / gridDim.x;
  const size_t lo = per * blockIdx.x, hi = min(n16, lo + per);
  const uint4* src = static_cast<const uint4*>(h_host);
  uint4* dst = static_cast<uint4*>(const_cast<void*>(h_dev));
  for (size_t i = lo + et; i < hi; i += nthr) dst[i] = src[i];
  if (blockIdx.x == 0)                       // bytes % 16 (D % 8 == 0 for bf16 makes this 0)
    for (size_t i = n16 * 16 + et; i < bytes; i += nthr)
      static_cast<uint8_t*>(const_cast<void*>(h_dev))[i] = static_cast<const uint8_t*>(h_host)[i];
  __threadfence();
  sm100::named_bar_sync(bar_id, nthr);
  if (et == 0) atomicAdd(h_bar, 1u);
}
// Producer side: wait until every CTA staged its slice, then order the TMA reads after it.
// The host launches in-kernel staging only when the whole grid fits on the device at once
// (fs_api.cu run_path); should the CTAs still not be co-resident (a GPU shared through MPS or
// green contexts), the wait gives up after ~5 s instead of hanging or trapping: it raises the
// timeout flag h_bar[1] and proceeds, the CTAs drain, and the finalizing CTA reports every row
// as undefined (finalize_last_cta) -- a recoverable per-call failure, no sticky CUDA error.
__device__ __forceinline__ void wait_h_staged(unsigned int* h_bar) {
  const uint64_t t0 = sm100::globaltimer();
  while (sm100::ld_acquire_gpu(h_bar) < gridDim.x) {
    __nanosleep(64);
    if (sm100::globaltimer() - t0 > 5000000000ull) {
      atomicExch(h_bar + 1, 1u);
      break;
    }
  }
  sm100::fence_proxy_async_global();
}

// Persistent-CTA vocabulary partition: CTA c of G owns rows [u*floor(c*U/G), u*floor((c+1)*U/G))
// (U = ceil(V/u) units of u rows, u in {16, 32, 64, 128}), clipped to V.  No split-K: every
// logit's fp32 sum is independent of G and of the partition.
__device__ __forceinline__ void cta_rows(int cta, int G, int V, int unit, int& r0, int& r1) {
  const int64_t U = (V + unit - 1) / unit;
  r0 = (int)(unit * ((int64_t)cta * U / G));
  const int64_t e = unit * ((int64_t)(cta + 1) * U / G);
  r1 = (int)(e < (int64_t)V ? e : (int64_t)V);
}

}  // namespace fs
