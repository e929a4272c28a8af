"""Flat definition of the fused LM-head + exact Gumbel-max sampler (test infrastructure only).

The fused two-stage kernel (Alg. 2) is exact *pathwise*: by the
"Max over vocabulary tiles" lemma (applied at P:391) it returns exactly
    idx_b = argmax_v ( l~_{b,v} + g_{b,v} )
so the oracle is that definition written out over the whole row, in fp64, with no
tiling.  Steps:

  O1  inputs: exact bf16 bit patterns (or fp32) -> fp64 (exact)
  O2  l[b,v]  = sum_d h[b,d] W[v,d]                     Y = H W^T; Alg. 2
  O3  l~      = (l + bias_v) / tau_b; mask bit 0 or NaN -> -inf     P:41, Alg. 2, §4.6
              (order: DESIGN.md reading R3; tau <= 0 or non-finite -> row undefined, R7)
  O4  g[b,v]  = gumbel64(r(seed, step, b, v))           Alg. 2, App. C
  O5  s       = l~ + g                                   Alg. 2
  O6  idx     = smallest v attaining max s; s1, s2, gap, near-tie set     Alg. A.1
              (ties -> smaller index: DESIGN.md reading R5; no finite l~ -> idx -1: R7)
  O7  grouped: M_k = max_{G_k} s, I_k = argmax, L_k = logsumexp_{G_k} l~   §4.1 P:211-217,
              Lemma P:254-270; outer selection reuses the maxima (reading R8)
  O8  TP: shards are groups (Alg. A.4); idx_TP == idx_flat
  logZ = logsumexp_v l~                                  App. E
"""
from __future__ import annotations

import dataclasses
import numpy as np

from . import rng

NEAR_TIE = 1e-2       # north-star parity rule: bit-exact index when top-2 gap > 1e-2


def to_f64(a) -> np.ndarray:
    """O1: bf16 bit patterns (uint16) or fp32/fp64 values -> exact fp64."""
    a = np.asarray(a)
    if a.dtype == np.uint16:
        return (a.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)
    return a.astype(np.float64)


def logits(h, W, rows=None, v_chunk: int = 16384) -> np.ndarray:
    """O2: l = H W^T in fp64 for the selected batch rows.  h [B,D], W [V,D]."""
    hf = to_f64(h)
    if rows is not None:
        hf = hf[np.asarray(rows)]
    V = W.shape[0]
    out = np.empty((hf.shape[0], V), dtype=np.float64)
    for v0 in range(0, V, v_chunk):
        v1 = min(V, v0 + v_chunk)
        out[:, v0:v1] = hf @ to_f64(W[v0:v1]).T
    return out


def allowed_bits(mask, rows, v_global) -> np.ndarray:
    """Mask bit for (row, global vocab id): bit v%32 of word v/32, 1 = allowed (reading R4)."""
    words = np.asarray(mask, dtype=np.uint32)[np.asarray(rows)]          # [R, nw]
    w = words[:, v_global // 32]
    return ((w >> (v_global % 32).astype(np.uint32)) & np.uint32(1)).astype(bool)


def greedy_rows(temperature, rows):
    """Rows sampled greedily: tau == 0 exactly (reading R18; "greedy ... would
    disable FlashSampling" -- greedy is argmax without noise)."""
    if temperature is None:
        return np.zeros(len(np.atleast_1d(rows)), dtype=bool)
    return np.asarray(temperature, dtype=np.float64)[np.asarray(rows)] == 0.0


def transform(ell, rows, v_global, bias=None, temperature=None, mask=None):
    """O3: l~ = (l + bias_v)/tau_b, banned or NaN -> -inf.  Returns (l~, row_valid).
    tau == 0: greedy row, l~ = l + bias_v (no scaling); tau < 0 or non-finite: undefined row."""
    lt = ell.copy()
    if bias is not None:
        lt = lt + np.asarray(bias, dtype=np.float64)[None, :]
    row_valid = np.ones(lt.shape[0], dtype=bool)
    if temperature is not None:
        tau = np.asarray(temperature, dtype=np.float64)[np.asarray(rows)]
        greedy = tau == 0.0
        row_valid = np.isfinite(tau) & (tau >= 0)
        safe = np.where(row_valid & ~greedy, tau, 1.0)
        lt = lt / safe[:, None]
    if mask is not None:
        lt = np.where(allowed_bits(mask, rows, v_global), lt, -np.inf)
    lt = np.where(np.isnan(lt), -np.inf, lt)
    lt[~row_valid, :] = -np.inf
    return lt, row_valid


@dataclasses.dataclass
class Scores:
    rows: np.ndarray          # batch row ids [R]
    v_global: np.ndarray      # global vocab ids [Vl]
    ltilde: np.ndarray        # [R, Vl] transformed logits (fp64)
    g: np.ndarray             # [R, Vl] Gumbel noise (fp64)
    s: np.ndarray             # [R, Vl] perturbed scores (fp64)


def noise(seed, step, rows, v_global, seeds=None, steps=None, temperature=None) -> np.ndarray:
    """O4: Gumbel noise [R, V]: shared layout (R1) or per-request layout (R18) when `seeds`
    ([B] uint64) is given (`steps` [B] or None -> the scalar step); 0 on greedy rows."""
    rows = np.asarray(rows)
    if seeds is None:
        g = rng.gumbel_at(seed, step, rows[:, None], v_global[None, :])
    else:
        sd = np.asarray(seeds).astype(np.uint64)[rows]
        stp = (np.full(len(rows), int(step) & 0xFFFFFFFFFFFFFFFF, np.uint64) if steps is None
               else np.asarray(steps).astype(np.uint64)[rows])
        g = rng.gumbel64(rng.random_bits_per_request(sd[:, None], stp[:, None], v_global[None, :]))
    g = np.where(greedy_rows(temperature, rows)[:, None], 0.0, g)
    return g


def scores(h, W, *, seed: int, step: int, rows=None, bias=None, temperature=None,
           mask=None, vocab_offset: int = 0, seeds=None, steps=None) -> Scores:
    """O1-O5 for the selected rows.  W (and bias) may be a vocabulary shard whose first
    row has global id `vocab_offset`; the RNG and the mask are keyed by global ids."""
    B = np.asarray(h).shape[0]
    rows = np.arange(B) if rows is None else np.asarray(rows)
    V_local = W.shape[0]
    v_global = np.arange(vocab_offset, vocab_offset + V_local, dtype=np.int64)
    ell = logits(h, W, rows)
    lt, _ = transform(ell, rows, v_global, bias, temperature, mask)
    g = noise(seed, step, rows, v_global, seeds, steps, temperature)
    s = lt + g                      # -inf + finite = -inf
    return Scores(rows=rows, v_global=v_global, ltilde=lt, g=g, s=s)


def scores_from_logits(logits, *, seed: int, step: int, rows=None, bias=None, temperature=None,
                       mask=None, seeds=None, steps=None) -> Scores:
    """O3-O5 on pre-materialised logits l [B, V] (standalone sampling, §5.2 P:490-493 /
    Alg. A.1): the same transform, RNG layout and perturbation as the fused path."""
    lg = to_f64(logits)
    B, V = lg.shape
    rows = np.arange(B) if rows is None else np.asarray(rows)
    v_global = np.arange(V, dtype=np.int64)
    lt, _ = transform(lg[rows], rows, v_global, bias, temperature, mask)
    g = noise(seed, step, rows, v_global, seeds, steps, temperature)
    return Scores(rows=rows, v_global=v_global, ltilde=lt, g=g, s=lt + g)


@dataclasses.dataclass
class TopKResult:
    idx: np.ndarray           # [R] sampled global id (-1: no finite l~)
    s1: np.ndarray            # [R] winning perturbed score over the kept set
    gap: np.ndarray           # [R] s1 - second best over the kept set (inf if one survivor)
    kept: list                # per row: global ids of the kept set (top-k, then top-p), sorted
    kth_margin: np.ndarray    # [R] l~ gap at the top-k boundary (rank k vs k+1; inf if none)
    p_margin: np.ndarray      # [R] |cumsum before the top-p cut - p| (decision margin)
    near: list = None         # per row: kept ids with s >= s1 - NEAR_TIE (the north-star near-tie set)


def topk_topp_sample(sc: Scores, top_k: int, top_p: float = 1.0) -> TopKResult:
    """Top-k then top-p (nucleus) sampling, exactly (§4.6; reading R19):
      1. rank tokens by l~ descending, ties by smaller id; keep the first k with finite l~;
      2. q = softmax of l~ over those k (fp64); keep the shortest prefix whose cumulative q >= p;
      3. idx = argmax over the kept set of l~ + g (the same per-token Gumbels as the flat
         sampler; Gumbel-max restricted to a subset samples the renormalised subset exactly)."""
    R, V = sc.s.shape
    idx = np.full(R, -1, np.int64)
    s1 = np.full(R, -np.inf)
    gap = np.full(R, np.inf)
    kth = np.full(R, np.inf)
    pm = np.full(R, np.inf)
    kept_all = []
    near_all = []
    for r in range(R):
        lt = sc.ltilde[r]
        order = np.lexsort((sc.v_global, -lt))               # l~ desc, id asc
        k = min(int(top_k), V)
        cand = order[:k]
        if k < V and np.isfinite(lt[order[k - 1]]):
            kth[r] = lt[order[k - 1]] - lt[order[k]]
        cand = cand[np.isfinite(lt[cand])]
        if cand.size == 0:
            kept_all.append([])
            near_all.append([])
            continue
        q = np.exp(lt[cand] - lt[cand[0]])
        q = q / q.sum()
        c = np.cumsum(q)
        m = int(np.searchsorted(c, top_p, side="left")) if top_p < 1.0 else cand.size - 1
        m = min(m, cand.size - 1)
        keep = cand[:m + 1]
        if top_p < 1.0:
            before = c[m - 1] if m > 0 else 0.0
            pm[r] = min(abs(c[m] - top_p), abs(before - top_p))
        s = lt[keep] + sc.g[r, keep]
        best = s.max()
        win = keep[s == best]
        j = win[np.argmin(sc.v_global[win])]
        idx[r] = sc.v_global[j]
        s1[r] = best
        rest = s[keep != j]
        gap[r] = best - rest.max() if rest.size else np.inf
        kept_all.append(sorted(int(sc.v_global[x]) for x in keep))
        near_all.append(sorted(int(sc.v_global[x]) for x, sx in zip(keep, s) if sx >= best - NEAR_TIE))
    return TopKResult(idx=idx, s1=s1, gap=gap, kept=kept_all, kth_margin=kth, p_margin=pm, near=near_all)


def log_prob(sc: Scores, res: "FlatResult") -> np.ndarray:
    """log p(idx) = l~_idx - logsumexp(l~)  (App. E: log-normalizer -> log-probabilities);
    -inf for undefined rows."""
    out = np.full(len(res.idx), -np.inf)
    for r, i in enumerate(res.idx):
        if i >= 0:
            j = int(np.nonzero(sc.v_global == i)[0][0])
            out[r] = sc.ltilde[r, j] - res.logZ[r]
    return out


def logsumexp(x, axis=-1) -> np.ndarray:
    """Max-shifted log(sum(exp(x))); -inf for an all -inf (or empty) slice."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape[axis] == 0:
        return np.full(np.delete(np.array(x.shape), axis % x.ndim), -np.inf)
    m = np.max(x, axis=axis, keepdims=True)
    finite = np.isfinite(m)
    msafe = np.where(finite, m, 0.0)
    with np.errstate(divide="ignore"):
        out = np.log(np.sum(np.exp(x - msafe), axis=axis, keepdims=True)) + msafe
    out = np.where(finite, out, m)
    return np.squeeze(out, axis=axis)


@dataclasses.dataclass
class FlatResult:
    idx: np.ndarray           # [R] global id, -1 when the row has no finite l~
    s1: np.ndarray            # [R] winning perturbed score (-inf for undefined rows)
    s2: np.ndarray            # [R] second-largest perturbed score over v != idx
    gap: np.ndarray           # [R] s1 - s2
    near: list                # per row: global ids with s >= s1 - NEAR_TIE (capped)
    logZ: np.ndarray          # [R] logsumexp of l~ (App. E)


def flat_sample(sc: Scores, near_cap: int = 64, want_near: bool = True) -> FlatResult:
    """O6: argmax over the whole row; ties -> smallest global id."""
    R, V = sc.s.shape
    j = np.argmax(sc.s, axis=1)                    # first occurrence = smallest id
    top = sc.s[np.arange(R), j]
    defined = ~np.isneginf(top)
    idx = np.where(defined, sc.v_global[j], -1)
    s1 = np.where(defined, top, -np.inf)
    rest = sc.s.copy()
    rest[np.arange(R), j] = -np.inf
    s2 = rest.max(axis=1) if V > 1 else np.full(R, -np.inf)
    s2 = np.where(defined, s2, -np.inf)
    with np.errstate(invalid="ignore"):
        gap = s1 - s2
    near = []
    if want_near:
        for r in range(R):
            if not defined[r]:
                near.append([])
                continue
            cand = np.nonzero(sc.s[r] >= s1[r] - NEAR_TIE)[0][:near_cap]
            near.append([int(sc.v_global[c]) for c in cand])
    return FlatResult(idx=idx, s1=s1, s2=s2, gap=gap, near=near, logZ=logsumexp(sc.ltilde, axis=1))


@dataclasses.dataclass
class GroupResult:
    M: np.ndarray             # [R, K] group max perturbed score (Lemma P:258)
    I: np.ndarray             # [R, K] its smallest argmax (global id), -1 if empty
    L: np.ndarray             # [R, K] group log-mass logsumexp(l~_{G_k})
    idx: np.ndarray           # [R] I at argmax_k M_k (ties -> smaller k)
    logZ: np.ndarray          # [R] logsumexp_k L_k


def group_summaries(sc: Scores, group_size: int) -> GroupResult:
    """O7: contiguous groups [k g, min((k+1) g, V)) of the (local) vocabulary axis."""
    R, V = sc.s.shape
    K = (V + group_size - 1) // group_size
    M = np.full((R, K), -np.inf)
    I = np.full((R, K), -1, np.int64)
    L = np.full((R, K), -np.inf)
    for k in range(K):
        a, b = k * group_size, min(V, (k + 1) * group_size)
        blk = sc.s[:, a:b]
        j = np.argmax(blk, axis=1)
        m = blk[np.arange(R), j]
        M[:, k] = m
        I[:, k] = np.where(np.isneginf(m), -1, sc.v_global[a + j])
        L[:, k] = logsumexp(sc.ltilde[:, a:b], axis=1)
    kstar = np.argmax(M, axis=1)
    idx = np.where(np.isneginf(M[np.arange(R), kstar]), -1, I[np.arange(R), kstar])
    return GroupResult(M=M, I=I, L=L, idx=idx, logZ=logsumexp(L, axis=1))


def shard_bounds(V: int, n: int):
    """Alg. A.4: rank k holds [k V/n, (k+1) V/n) (floor division; last shard ragged)."""
    return [(k * V // n, (k + 1) * V // n) for k in range(n)]


def combine_shard_summaries(M, I, L):
    """Alg. A.4 P:830-833 with max reuse (reading R8): winner = argmax_k M_k
    (ties -> smaller global id), logZ = logsumexp_k L_k.  M, I, L: [n, R]."""
    M = np.asarray(M, np.float64)
    I = np.asarray(I, np.int64)
    n, R = M.shape
    idx = np.full(R, -1, np.int64)
    best = np.full(R, -np.inf)
    for k in range(n):
        for r in range(R):
            if I[k, r] < 0:
                continue
            if M[k, r] > best[r] or (M[k, r] == best[r] and (idx[r] < 0 or I[k, r] < idx[r])):
                best[r], idx[r] = M[k, r], I[k, r]
    return idx, best, logsumexp(np.asarray(L, np.float64).T, axis=1)


def tp_sample(h, W, n: int, **kw):
    """O8: run the flat definition on each vocabulary shard and combine the 3-scalar
    summaries.  Returns (idx, score, logZ, per-rank (M, I, L))."""
    V = W.shape[0]
    bias = kw.pop("bias", None)
    Ms, Is, Ls = [], [], []
    R = len(kw["rows"]) if kw.get("rows") is not None else np.asarray(h).shape[0]
    for a, b in shard_bounds(V, n):
        if b == a:                                   # empty shard: zero mass
            Ms.append(np.full(R, -np.inf)); Is.append(np.full(R, -1)); Ls.append(np.full(R, -np.inf))
            continue
        sc = scores(h, W[a:b], bias=None if bias is None else np.asarray(bias)[a:b],
                    vocab_offset=a, **kw)
        gr = group_summaries(sc, max(1, b - a))
        Ms.append(gr.M[:, 0]); Is.append(gr.I[:, 0]); Ls.append(gr.L[:, 0])
    idx, best, logZ = combine_shard_summaries(Ms, Is, Ls)
    return idx, best, logZ, (np.array(Ms), np.array(Is), np.array(Ls))
