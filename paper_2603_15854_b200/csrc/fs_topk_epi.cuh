// fs_topk_epi.cuh -- top-k candidates inside the fused LM-head epilogue (
// PAPER.md §4.6: "each tile computes top-k candidates locally, a second stage reduces
// all per-tile candidates into a global top-k"; reading R19) and the raw-logit store
// used when the candidate lists do not fit in shared memory.
//
// Top-k mode of the 1-CTA tcgen05 kernel: every epilogue warp sees every tile; warp quad qd
// (warps 4qd+2 .. 4qd+5, one per TMEM lane quadrant) handles the 8-column groups g = qd, qd+2, ...
// Per batch column the CTA keeps, in shared memory, a list of (key(l~), id) candidates of
// capacity cap >= k_pad + 128, a count and an append threshold thr:
//   * append: a row of the tile enters the list iff key(l~) > thr (thr starts at key(-inf), so
//     only finite l~ enter -- R19 keeps finite logits only);
//   * compaction (tile end, when the list might not hold another full tile of 128 rows): exact
//     warp radix select of the k best by (key desc, id asc); thr := key of the k-th.  A later row
//     with key == thr has a larger id than every kept row (tiles reach a CTA in increasing id
//     order), so it ranks below all k kept rows: the strict test is exact.
// At the end each CTA writes its k best per column (padded with id -1) to
// cand[b][cta * k + j]; topk_final_kernel (fs_topk.cu) merges the G*k candidates of a row,
// applies top-p and draws the Gumbel-max over the kept set.
#pragma once
#include "fs_epilogue.cuh"

namespace fs {

struct TopkSmem {
  uint32_t* thr;    // [BN] append threshold (order key)
  int* cnt;         // [BN] list lengths
  uint32_t* hist;   // [8 warps][256] radix histograms (warp-private)
  Cand* buf;        // [BN][cap]
  int cap;
  int k;
};

__device__ __forceinline__ uint32_t lanemask_lt(int lane) { return (1u << lane) - 1u; }

// k-th largest key among buf[0, n) (n >= k): returns T and `take` = how many elements equal to
// T belong to the k largest.  Warp-cooperative 4 x 8-bit radix select; hist = 256 words.
__device__ __forceinline__ void warp_select_key(const Cand* buf, int n, int k, uint32_t* hist, int lane,
                                                uint32_t& T, int& take) {
  uint32_t prefix = 0, pmask = 0;
  int krem = k;
#pragma unroll 1
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
#pragma unroll
    for (int i = 0; i < 8; ++i) hist[lane * 8 + i] = 0u;
    __syncwarp();
    for (int base = 0; base < n; base += 32) {
      const int i = base + lane;
      const uint32_t key = i < n ? buf[i].key : 0u;
      warp_hist_add(hist, i < n && (key & pmask) == prefix, (key >> shift) & 255u, lane);
    }
    __syncwarp();
    int h[8], sum = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) { h[i] = (int)hist[lane * 8 + i]; sum += h[i]; }
    int incl = sum;                                  // elements with digit in bins >= 8*lane
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_down_sync(0xFFFFFFFFu, incl, o);
      if (lane + o < 32) incl += v;
    }
    const int above = incl - sum;
    const bool here = above < krem && incl >= krem;
    int d = 0, nk = 0, acc = above;
#pragma unroll
    for (int i = 7; i >= 0; --i) {
      const bool hit = here && nk == 0 && acc + h[i] >= krem;
      d = hit ? lane * 8 + i : d;
      nk = hit ? krem - acc : nk;
      acc += h[i];
    }
    const int src = __ffs(__ballot_sync(0xFFFFFFFFu, here)) - 1;
    d = __shfl_sync(0xFFFFFFFFu, d, src);
    krem = __shfl_sync(0xFFFFFFFFu, nk, src);
    prefix |= (uint32_t)d << shift;
    pmask |= 255u << shift;
    __syncwarp();
  }
  T = prefix;
  take = krem;
}

// The take-th smallest id among the elements with key == T (ascending radix select).
__device__ __forceinline__ uint32_t warp_select_id(const Cand* buf, int n, uint32_t T, int take, uint32_t* hist,
                                                   int lane) {
  uint32_t prefix = 0, pmask = 0;
  int krem = take;
#pragma unroll 1
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
#pragma unroll
    for (int i = 0; i < 8; ++i) hist[lane * 8 + i] = 0u;
    __syncwarp();
    for (int base = 0; base < n; base += 32) {
      const int i = base + lane;
      const Cand c = i < n ? buf[i] : Cand{kKeyNone, -1};
      const uint32_t id = (uint32_t)c.idx;
      warp_hist_add(hist, i < n && c.key == T && (id & pmask) == prefix, (id >> shift) & 255u, lane);
    }
    __syncwarp();
    int h[8], sum = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) { h[i] = (int)hist[lane * 8 + i]; sum += h[i]; }
    int incl = sum;                                  // elements with digit in bins <= 8*lane+7
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += v;
    }
    const int below = incl - sum;
    const bool here = below < krem && incl >= krem;
    int d = 0, nk = 0, acc = below;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool hit = here && nk == 0 && acc + h[i] >= krem;
      d = hit ? lane * 8 + i : d;
      nk = hit ? krem - acc : nk;
      acc += h[i];
    }
    const int src = __ffs(__ballot_sync(0xFFFFFFFFu, here)) - 1;
    d = __shfl_sync(0xFFFFFFFFu, d, src);
    krem = __shfl_sync(0xFFFFFFFFu, nk, src);
    prefix |= (uint32_t)d << shift;
    pmask |= 255u << shift;
    __syncwarp();
  }
  return prefix;
}

// Keep exactly the k best of buf[0, n) by (key desc, id asc), order-preserving, in place.
// Returns the new length (k if n > k) and sets thr to the k-th key.  Warp-uniform.
__device__ __forceinline__ int warp_compact(Cand* buf, int n, int k, uint32_t* hist, int lane, uint32_t& thr) {
  if (n <= k) return n;
  uint32_t T;
  int take;
  warp_select_key(buf, n, k, hist, lane, T, take);
  unsigned ties = 0;
  for (int i = lane; i < n; i += 32) ties += buf[i].key == T;
  ties = __reduce_add_sync(0xFFFFFFFFu, ties);
  const uint32_t idT = (int)ties > take ? warp_select_id(buf, n, T, take, hist, lane) : 0xFFFFFFFFu;
  int out = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const Cand c = i < n ? buf[i] : Cand{kKeyNone, -1};
    const bool keep = i < n && (c.key > T || (c.key == T && (uint32_t)c.idx <= idT));
    const uint32_t bl = __ballot_sync(0xFFFFFFFFu, keep);
    __syncwarp();
    if (keep) buf[out + __popc(bl & lanemask_lt(lane))] = c;
    out += __popc(bl);
    __syncwarp();
  }
  thr = T;
  return out;
}

// One tile of the top-k epilogue for this warp: 32 rows x the quad's 8-column groups.
template <bool XFORM>
__device__ __forceinline__ void epi_tile_topk(uint32_t taddr, const RowArgs& ra, const EpiArgs& ea,
                                              const TopkSmem& ts, int lane, int qd) {
  const int B = ea.B;
  const int wshift = ra.warp_v0 & 31;
  const int msrc = ((lane + wshift) >> 5) << 4, mbit = (lane + wshift) & 31;
#pragma unroll 1
  for (int g = qd; g * 8 < B; g += 2) {
    const int col0 = g * 8;
    uint32_t r[8];
    sm100::tmem_ld_32x32b_x8(taddr + (uint32_t)col0, r);
    uint32_t mw = 0xFFFFFFFFu;
    if (XFORM && ea.mask != nullptr) {               // same word staging as epi_tile_tc
      const int jb = col0 + (lane & 15);
      const int64_t w = (int64_t)(ra.warp_v0 >> 5) + (lane >> 4);
      mw = 0u;
      if ((lane & 15) < 8 && jb < B && w < ea.mask_words) mw = __ldg(ea.mask + (int64_t)jb * ea.mask_words + w);
    }
    sm100::tmem_wait_ld();
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int col = col0 + jj;
      if (col >= B) break;                           // warp-uniform
      float l = __uint_as_float(r[jj]);
      if (XFORM) {
        l = (l + ra.bias) * ea.invtau[col];
        if (ea.mask != nullptr) {
          // bit of row warp_v0 + lane sits in word (lane + wshift) >> 5 (lanes 0-15 / 16-31)
          const uint32_t w = __shfl_sync(0xFFFFFFFFu, mw, msrc + jj);
          if (!((w >> mbit) & 1u)) l = -INFINITY;
        }
      }
      if (isnan(l)) l = -INFINITY;
      const uint32_t key = ra.valid ? order_key(l) : kKeyNone;
      const bool pass = key > ts.thr[col];
      const uint32_t bl = __ballot_sync(0xFFFFFFFFu, pass);
      if (bl) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&ts.cnt[col], __popc(bl));
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        if (pass) ts.buf[(size_t)col * ts.cap + base + __popc(bl & lanemask_lt(lane))] = Cand{key, ra.v_global};
      }
    }
  }
}

// Compact the columns of quad qd owned by warp wq (column jj of a group with jj % 4 == wq) whose
// list exceeds `limit`.  Caller brackets with the quad's named barrier.
__device__ __forceinline__ void topk_compact_cols(const TopkSmem& ts, int B, int qd, int wq, int limit,
                                                  uint32_t* hist, int lane) {
#pragma unroll 1
  for (int g = qd; g * 8 < B; g += 2)
#pragma unroll 1
    for (int jj = wq; jj < 8; jj += 4) {
      const int col = g * 8 + jj;
      if (col >= B) break;
      const int n = ts.cnt[col];
      if (n <= limit) continue;
      uint32_t t = ts.thr[col];
      const int nn = warp_compact(ts.buf + (size_t)col * ts.cap, n, ts.k, hist, lane, t);
      __syncwarp();
      if (lane == 0) { ts.cnt[col] = nn; ts.thr[col] = t; }
      __syncwarp();
    }
}

// Write this CTA's list of every column of the quad/warp (no final compaction: the merge kernel
// selects exactly): append the cnt entries at an atomically allocated offset of the row, and the
// list's m-th largest key (the merge kernel's pruning bound; 0 if the list is shorter).
__device__ __forceinline__ void topk_write_cols(const TopkSmem& ts, int B, int qd, int wq, int lane, Cand* cand,
                                                int stride, int* rowcnt, uint32_t* slot_lb, int nslot, int slot,
                                                int m, uint32_t* hist) {
#pragma unroll 1
  for (int g = qd; g * 8 < B; g += 2)
#pragma unroll 1
    for (int jj = wq; jj < 8; jj += 4) {
      const int col = g * 8 + jj;
      if (col >= B) break;
      const int n = ts.cnt[col];
      const Cand* src = ts.buf + (size_t)col * ts.cap;
      uint32_t lb = 0u;
      if (n >= m) {
        if (m == 1) {
          uint32_t mx = 0u;
          for (int j = lane; j < n; j += 32) mx = max(mx, src[j].key);
          lb = __reduce_max_sync(0xFFFFFFFFu, mx);
        } else {
          int take;
          warp_select_key(src, n, m, hist, lane, lb, take);
        }
      }
      int off = 0;
      if (lane == 0) {
        off = n > 0 ? atomicAdd(rowcnt + col, n) : 0;
        slot_lb[(size_t)col * nslot + slot] = lb;
      }
      off = __shfl_sync(0xFFFFFFFFu, off, 0);
      Cand* out = cand + (size_t)col * stride + off;
      for (int j = lane; j < n; j += 32) out[j] = src[j];
    }
}

// Raw-logit store (fallback when the candidate lists do not fit): this warp's 32 rows x all B
// columns of one tile, acc (fp32, untransformed) -> out[b * ld + row]; coalesced per column.
// gmax (optional): this warp's 32-row span starts at local row 16*u0 (span_rows valid rows, 0 =
// empty span -> nothing written); per column the span's max order key of the raw logit goes to
// gmax[col][u0] and the marker 1 to gmax[col][u0 + 1] when the span covers a second 16-row unit.
__device__ __forceinline__ void epi_tile_store(uint32_t taddr, bool valid, int row, int B, float* out, int64_t ld,
                                               uint32_t* gmax = nullptr, int64_t gld = 0, int64_t u0 = 0,
                                               int span_rows = 0, int lane = 0, int col_first = 0,
                                               int col_step = 8) {
#pragma unroll 1
  for (int col0 = col_first; col0 < B; col0 += col_step) {
    uint32_t r[8];
    sm100::tmem_ld_32x32b_x8(taddr + (uint32_t)col0, r);
    sm100::tmem_wait_ld();
#pragma unroll
    for (int jj = 0; jj < 8; ++jj)
      if (valid && col0 + jj < B) out[(int64_t)(col0 + jj) * ld + row] = __uint_as_float(r[jj]);
    if (gmax != nullptr && span_rows > 0) {
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        float x = __uint_as_float(r[jj]);
        if (isnan(x)) x = -INFINITY;
        const uint32_t km = __reduce_max_sync(0xFFFFFFFFu, valid ? order_key(x) : kKeyNone);
        if (lane == jj && col0 + jj < B) {
          gmax[(int64_t)(col0 + jj) * gld + u0] = km;
          if (span_rows > 16) gmax[(int64_t)(col0 + jj) * gld + u0 + 1] = 1u;
        }
      }
    }
  }
}

}  // namespace fs
