"""GPU parity of top-k / top-p sampling THROUGH the LM head (SURVEY §8(f) f1 in the fused
epilogue; reading R19) against oracle.sampler.topk_topp_sample on
the exact h, W the GPU saw.  Both stage-1 routes are covered: candidate lists in the epilogue
(topk_mode 1) and raw fp32 logits + chunked selection (topk_mode 2); they must agree bit for bit
(same accumulator, same transform)."""
import numpy as np
import pytest
import torch

import synth
from oracle import sampler, stats
from parity import SCORE_TOL, oracle_inputs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2603_15854_b200 as fs

# boundary decisions (k-th element, top-p cut) are taken on fp32 l~ from an fp32 MMA sum; the
# oracle's fp64 margin must exceed the fp32 accumulation error (|l| ~ 1, D <= 4096: << 1e-4)
MARGIN = 1e-4


@pytest.fixture(autouse=True)
def _reset():
    yield
    if torch.cuda.is_available():
        fs.set_option("topk_mode", 0)
        fs.set_option("force_simt", 0)
        fs.set_option("max_ctas", 0)
        fs.set_option("topk_spans", 1)
        fs.set_option("pair", -1)


def _dev(t):
    return None if t is None else t.cuda()


def _run(wl, k, p, step=3, seeds=None, temperature=None):
    tau = wl.temperature if temperature is None else temperature
    return fs.sample(_dev(wl.h), _dev(wl.W), bias=_dev(wl.bias), temperature=_dev(tau), mask=_dev(wl.mask),
                     seed=wl.seed, step=step, seeds=seeds, top_k=k, top_p=p, return_score=True,
                     return_logprob=True)


def _oracle(wl, k, p, step=3, seeds=None, temperature=None):
    a = oracle_inputs(wl)
    tau = a["temperature"] if temperature is None else temperature.numpy()
    sc = sampler.scores(a["h"], a["W"], seed=wl.seed, step=step, bias=a["bias"], temperature=tau, mask=a["mask"],
                        seeds=None if seeds is None else seeds.cpu().numpy().astype(np.uint64))
    return sc, sampler.topk_topp_sample(sc, k, p)


def _check(idx, score, res):
    idx = idx.cpu().numpy()
    score = score.cpu().numpy()
    exact = decisive = 0
    for r in range(len(res.idx)):
        if res.idx[r] < 0:
            assert idx[r] == -1, (r, idx[r])
            continue
        if not ((res.kth_margin[r] > MARGIN or res.kth_margin[r] == 0) and res.p_margin[r] > MARGIN):
            continue                                      # boundary within fp32 rounding
        decisive += 1
        assert idx[r] in res.kept[r], (r, idx[r])
        assert abs(score[r] - res.s1[r]) <= SCORE_TOL, (r, score[r], res.s1[r])
        if res.gap[r] > 1e-2:
            assert idx[r] == res.idx[r], (r, idx[r], res.idx[r])
            exact += 1
        else:                                             # near tie: one of the near-tied kept ids
            assert int(idx[r]) in res.near[r], (r, idx[r], res.near[r])
    return exact, decisive


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("cfg,B,V,D,k,p", [
    ("llama3_8b", 1, 5000, 128, 50, 0.95),
    ("llama3_8b", 13, 20000, 256, 50, 1.0),
    ("qwen25_7b", 32, 9000, 128, 20, 0.8),          # bias + tau + mask
    ("llama3_8b", 8, 3000, 64, 1, 1.0),             # k = 1: argmax of l~
    ("llama3_8b", 4, 7000, 192, 200, 0.9),          # k > 128: list capacity > 2 tiles
    ("qwen25_7b", 3, 300, 64, 500, 0.99),           # k > V
])
def test_fused_topk_matches_oracle(mode, cfg, B, V, D, k, p):
    fs.set_option("topk_mode", mode)
    wl = synth.make_workload(cfg, B, V=V, D=D, seed_offset=k + B, pattern="peaked")
    idx, score, logZ, logprob = _run(wl, k, p)
    _, res = _oracle(wl, k, p)
    exact, decisive = _check(idx, score, res)
    assert decisive >= 0.5 * B - 1 and exact >= 0.3 * decisive, (exact, decisive, B)


def test_lists_and_raw_logits_agree_bit_exact():
    wl = synth.make_workload("qwen25_7b", 24, V=30011, D=512, seed_offset=7, pattern="peaked")
    out = {}
    for mode in (1, 2):
        fs.set_option("topk_mode", mode)
        out[mode] = _run(wl, 64, 0.9, step=11)
    for a, b in zip(out[1], out[2]):
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))


def test_fused_topk_ties_and_increasing_logits():
    # (1) all-equal logits: the k smallest ids form the top-k (secondary id select in compaction)
    B, V, D, k = 5, 4000, 64, 37
    h = torch.zeros(B, D, dtype=torch.bfloat16)
    W = torch.zeros(V, D, dtype=torch.bfloat16)
    idx = fs.sample(h.cuda(), W.cuda(), seed=1, step=2, top_k=k)
    assert bool((idx.cpu() < k).all()) and bool((idx.cpu() >= 0).all())
    # (2) l~ increasing in v: every tile's rows beat all earlier ones (a compaction every tile)
    h = torch.ones(B, D, dtype=torch.bfloat16)
    ramp = torch.linspace(-4, 4, V).to(torch.bfloat16)
    W = torch.zeros(V, D, dtype=torch.bfloat16)
    W[:, 0] = ramp
    for mode in (1, 2):
        fs.set_option("topk_mode", mode)
        idx, score, logZ, logprob = fs.sample(h.cuda(), W.cuda(), seed=5, step=1, top_k=k, return_score=True,
                                              return_logprob=True)
        sc = sampler.scores(synth.as_numpy_exact(h), synth.as_numpy_exact(W), seed=5, step=1)
        res = sampler.topk_topp_sample(sc, k, 1.0)
        for r in range(B):
            assert int(idx[r]) in res.kept[r]
            if res.gap[r] > 1e-2:
                assert int(idx[r]) == res.idx[r]


def test_fused_topk_edges_greedy_per_request_masked():
    wl = synth.make_workload("qwen25_7b", 12, V=3000, D=64, pattern="edge")
    tau = wl.temperature.clone()
    tau[5] = 0.0                                                      # greedy row
    seeds = torch.arange(12, dtype=torch.int64) * 977 + 5
    for mode in (1, 2):
        fs.set_option("topk_mode", mode)
        idx, score, logZ, logprob = _run(wl, 30, 0.9, step=9, seeds=seeds.cuda(), temperature=tau)
        sc, res = _oracle(wl, 30, 0.9, step=9, seeds=seeds, temperature=tau)
        _check(idx, score, res)
        assert idx[0].item() == -1 and idx[1].item() == (3000 * 5) // 7   # fully masked / single allowed
        assert idx[5].item() == int(np.argmax(sc.ltilde[5]))


def test_fused_topk_simt_and_chunked_batches():
    # fp32 operands -> CUDA-core kernel (raw logits route); B > 256 -> row chunks (RNG row offset)
    wl = synth.make_workload("tiny", 300, V=1000, D=64, seed_offset=3)
    idx, score = fs.sample(_dev(wl.h), _dev(wl.W), seed=wl.seed, step=4, top_k=10, top_p=0.9, return_score=True)
    a = oracle_inputs(wl)
    res = sampler.topk_topp_sample(sampler.scores(a["h"], a["W"], seed=wl.seed, step=4), 10, 0.9)
    exact, decisive = _check(idx, score, res)
    assert decisive >= 150
    wl = synth.make_workload("llama3_8b", 260, V=2000, D=64, seed_offset=4)
    idx, score = fs.sample(_dev(wl.h), _dev(wl.W), seed=wl.seed, step=4, top_k=8, return_score=True)
    a = oracle_inputs(wl)
    res = sampler.topk_topp_sample(sampler.scores(a["h"], a["W"], seed=wl.seed, step=4), 8, 1.0)
    exact, decisive = _check(idx, score, res)
    assert decisive >= 200


def test_fused_topk_logZ_logprob():
    wl = synth.make_workload("llama3_8b", 6, V=5000, D=128, pattern="peaked")
    idx, score, logZ, logprob = _run(wl, 40, 0.7)
    sc, res = _oracle(wl, 40, 0.7)
    for r in range(6):
        kept = np.asarray(res.kept[r])
        lz = sampler.logsumexp(sc.ltilde[r, kept])
        assert abs(float(logZ[r]) - lz) <= 1e-3
        assert abs(float(logprob[r]) - (sc.ltilde[r, int(idx[r])] - lz)) <= 1e-3


def test_fused_topk_chi_square_1e6():
    lt = np.array([0.5, -1.0, 2.0, 0.0, 1.5, -0.5, 1.0, 0.25], np.float32)
    order = np.lexsort((np.arange(8), -lt.astype(np.float64)))[:5]
    q = np.exp(lt[order] - lt[order].max()).astype(np.float64)
    q /= q.sum()
    keep = order[:int(np.searchsorted(np.cumsum(q), 0.8)) + 1]
    target = np.zeros(8)
    target[keep] = stats.softmax_probs(lt[keep])
    B = 250
    h = torch.tensor(np.tile(lt, (B, 1))).to(torch.bfloat16).cuda()
    W = torch.eye(8).to(torch.bfloat16).cuda()
    counts = torch.zeros(8, dtype=torch.int64, device="cuda")
    for s in range(4000):
        counts += torch.bincount(fs.sample(h, W, seed=3, step=s, top_k=5, top_p=0.8).long(), minlength=8)
    c = counts.cpu().numpy()
    assert c[np.setdiff1d(np.arange(8), keep)].sum() == 0
    _, pv = stats.chi_square(c, target)
    assert pv > 1e-3


def test_topk_errors():
    wl = synth.make_workload("llama3_8b", 4, V=1000, D=64)
    with pytest.raises(fs.FlashSampleError):
        fs.sample(_dev(wl.h), _dev(wl.W), top_k=2000)
    with pytest.raises(fs.FlashSampleError):
        fs.sample(_dev(wl.h), _dev(wl.W), top_p=0.5)                  # top_p needs top_k


@pytest.mark.parametrize("B,V,k,p", [(1, 5000, 50, 0.95), (40, 20011, 50, 0.9), (256, 9000, 1, 1.0),
                                     (7, 3001, 1024, 0.5), (33, 129, 64, 1.0)])
def test_raw_route_span_gather_equals_chunk_selection(B, V, k, p):
    # raw-logit route: span maxima written by stage 1 + gather of the spans at or above the k-th
    # largest (topk_spans=1) vs the full chunk selection (topk_spans=0) -- identical results, with
    # per-row temperature incl. a greedy row (tau = 0) and an invalid row (tau < 0)
    fs.set_option("topk_mode", 2)
    wl = synth.make_workload("llama3_8b", B, V=V, D=128, seed_offset=B + k, pattern="peaked")
    tau = torch.rand(B, generator=torch.Generator().manual_seed(B)) + 0.5
    if B > 2:
        tau[1], tau[2] = 0.0, -1.0
    out = {}
    for spans in (0, 1):
        fs.set_option("topk_spans", spans)
        out[spans] = _run(wl, k, p, temperature=tau)
    fs.set_option("topk_spans", 1)
    for a, b in zip(out[0], out[1]):
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))
    sc, res = _oracle(wl, k, p, temperature=tau)
    _check(out[1][0], out[1][1], res)


def test_raw_route_span_gather_all_ties():
    # all-equal logits: every span reaches the threshold, the whole row is gathered; the k smallest
    # ids are the top-k
    fs.set_option("topk_mode", 2)
    B, V, D, k = 3, 6000, 64, 37
    h = torch.zeros(B, D, dtype=torch.bfloat16).cuda()
    W = torch.zeros(V, D, dtype=torch.bfloat16).cuda()
    idx = fs.sample(h, W, seed=1, step=2, top_k=k)
    assert bool((idx.cpu() < k).all()) and bool((idx.cpu() >= 0).all())


@pytest.mark.parametrize("B,V", [(17, 4099), (64, 20011), (128, 9000), (256, 5003)])
def test_raw_route_pair_kernel_equals_single_cta(B, V):
    # raw-logit route on the CTA-pair kernel (32-row pair tile units, span maxima per CTA half) vs the
    # 1-CTA kernel: the same stored logits and span bounds, hence identical samples; and the oracle
    fs.set_option("topk_mode", 2)
    wl = synth.make_workload("llama3_8b", B, V=V, D=192, seed_offset=3 * B + 1, pattern="peaked")
    out = {}
    for pair in (0, 1):                       # 1 forces the pair kernel from B = 17 (auto: B > 128)
        fs.set_option("pair", pair)
        out[pair] = _run(wl, 50, 0.95, step=5)
    fs.set_option("pair", -1)
    for a, b in zip(out[0], out[1]):
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))
    _, res = _oracle(wl, 50, 0.95, step=5)
    _check(out[1][0], out[1][1], res)
