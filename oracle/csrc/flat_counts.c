/*
 * flat_counts.c -- TEST INFRASTRUCTURE ONLY (part of oracle/, see oracle/__init__.py).
 *
 * A plain C restatement of the oracle's flat sampler for ONE row, used where the numpy oracle
 * is too slow: the north-star chi-square pins need 1e6 draws (reading R16), i.e.
 * up to 1e9 Gumbel evaluations for the tiny config (V = 1000).  Same definitions as
 * oracle/philox.py, oracle/rng.py and oracle/sampler.py, written out again (no shared code with
 * the CUDA path, no blocking or reordering):
 *
 *   Philox4x32-10 (Salmon et al. SC'11; "counter-based RNG (e.g. Philox)", reading R1)
 *   r    = Philox(ctr = (v, b >> 2, step lo, (step hi & 0xFFFFFF) | tag << 24), key = seed)[b & 3]
 *   u    = (r + 1) / (2^32 + 1)                         App. C
 *   g    = -log(-log u), evaluated without cancellation  App. C, reading R2:
 *          r <  2^31: E = -log((r+1)/(2^32+1));  r >= 2^31: E = -log1p(-(2^32-r)/(2^32+1)); g = -log E
 *   s_v  = l~_v + g_v  (-inf stays -inf)                 Alg. 2 line 11
 *   idx  = smallest v attaining max_v s_v (-1 if all -inf)    Alg. A.1, reading R5
 *
 * Draw d of oracle_flat_counts uses step = step0 + d (row b fixed): the draws are the sampler's
 * outputs at consecutive decode steps, exactly what the GPU chi-square tests count.
 * Pinned in tests/test_oracle_flat_c.py against the Random123 known answers, the numpy oracle's
 * gumbel64 (itself pinned to 50-digit Decimal) and draw-by-draw equality with sampler.flat_sample.
 * Built by __graft_entry__.build() (gcc -O2 -fopenmp), loaded with ctypes by the tests only.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static void philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;                    /* Weyl increments W0, W1 */
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;   /* M0 * c0 */
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;   /* M1 * c2 */
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

void oracle_philox(const uint32_t* ctr, const uint32_t* key, uint32_t* out) { philox4x32_10(ctr, key, out); }

double oracle_gumbel64(uint32_t r) {
  const double den = 4294967297.0;          /* 2^32 + 1 */
  double E;
  if (r < 2147483648u)
    E = -log(((double)r + 1.0) / den);
  else
    E = -log1p(-(4294967296.0 - (double)r) / den);
  return -log(E);
}

void oracle_gumbel64_array(const uint32_t* r, double* g, int64_t n) {
  for (int64_t i = 0; i < n; ++i) g[i] = oracle_gumbel64(r[i]);
}

/* draw of row b at `step` for vocabulary id v (shared-stream layout, tag 0) */
static uint32_t bits(uint64_t seed, uint64_t step, uint32_t b, uint32_t v) {
  const uint32_t ctr[4] = {v, b >> 2, (uint32_t)step, (uint32_t)((step >> 32) & 0x00FFFFFFu)};
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t o[4];
  philox4x32_10(ctr, key, o);
  return o[b & 3];
}

int64_t oracle_flat_sample(const double* lt, int V, uint64_t seed, uint64_t step, uint32_t b) {
  int64_t idx = -1;
  double best = -INFINITY;
  for (int v = 0; v < V; ++v) {
    if (lt[v] == -INFINITY) continue;       /* s = -inf never wins */
    const double s = lt[v] + oracle_gumbel64(bits(seed, step, b, (uint32_t)v));
    if (idx < 0 || s > best) {             /* strict: ties keep the smaller id */
      best = s;
      idx = v;
    }
  }
  return idx;
}

/* counts[v] += #{d in [0, n): oracle_flat_sample(lt, step0 + d) == v}; counts[V] collects -1 */
void oracle_flat_counts(const double* lt, int V, uint64_t seed, uint64_t step0, int64_t n, uint32_t b,
                        int64_t* counts) {
#pragma omp parallel
  {
    int64_t* mine = (int64_t*)calloc((size_t)V + 1, sizeof(int64_t));
#pragma omp for schedule(static)
    for (int64_t d = 0; d < n; ++d) {
      const int64_t i = oracle_flat_sample(lt, V, seed, step0 + (uint64_t)d, b);
      mine[i < 0 ? V : i] += 1;
    }
#pragma omp critical
    for (int v = 0; v <= V; ++v) counts[v] += mine[v];
    free(mine);
  }
}
