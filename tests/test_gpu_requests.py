"""GPU parity of SURVEY §8(f) f4 (reading R18): per-request RNG streams (batch-position
invariant) and greedy rows (temperature == 0), for the fused tcgen05 / CTA-pair / CUDA-core kernels
and the standalone logits sampler."""
import numpy as np
import pytest
import torch

import synth
from oracle import sampler, stats
from parity import check_flat, oracle_inputs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2603_15854_b200 as fs


def _dev(t):
    return None if t is None else t.cuda()


def _seeds(B, salt=0):
    rs = np.random.default_rng(1234 + salt)
    return rs.integers(0, 2**63, B, dtype=np.int64)


@pytest.fixture(autouse=True)
def _reset():
    yield
    if torch.cuda.is_available():
        fs.set_option("pair", -1)
        fs.set_option("force_simt", 0)


@pytest.mark.parametrize("B,pair,simt", [(5, 0, 0), (40, 0, 0), (40, 1, 0), (200, 1, 0), (13, 0, 1)])
def test_per_request_streams_match_oracle(B, pair, simt):
    fs.set_option("pair", pair)
    fs.set_option("force_simt", simt)
    wl = synth.make_workload("qwen25_7b", B, V=3000 + B, D=128, seed_offset=B)
    seeds = _seeds(B, B)
    steps = np.arange(B, dtype=np.int64) * 3 + 7
    idx, score = fs.sample(_dev(wl.h), _dev(wl.W), bias=_dev(wl.bias), temperature=_dev(wl.temperature),
                           mask=_dev(wl.mask), seeds=torch.tensor(seeds).cuda(), steps=torch.tensor(steps).cuda(),
                           return_score=True)
    a = oracle_inputs(wl)
    flat = sampler.flat_sample(sampler.scores(a["h"], a["W"], seed=0, step=0, bias=a["bias"],
                                              temperature=a["temperature"], mask=a["mask"],
                                              seeds=seeds.astype(np.uint64), steps=steps.astype(np.uint64)))
    check_flat(idx.cpu().numpy(), score.cpu().numpy(), flat)


def test_per_request_batch_position_invariance_bit_exact():
    wl = synth.make_workload("llama3_8b", 48, V=5000, D=256)
    h, W = _dev(wl.h), _dev(wl.W)
    seeds = torch.tensor(_seeds(48)).cuda()
    idx, score = fs.sample(h, W, seeds=seeds, step=11, return_score=True)
    perm = torch.randperm(48, generator=torch.Generator().manual_seed(0)).cuda()
    idx2, score2 = fs.sample(h[perm].contiguous(), W, seeds=seeds[perm].contiguous(), step=11, return_score=True)
    assert torch.equal(idx[perm], idx2)
    assert torch.equal(score[perm].view(torch.int32), score2.view(torch.int32))


@pytest.mark.parametrize("pair", [0, 1])
def test_greedy_rows(pair):
    fs.set_option("pair", pair)
    wl = synth.make_workload("qwen25_7b", 36, V=4000, D=128)
    tau = wl.temperature.clone()
    tau[::3] = 0.0                                           # every third row greedy
    idx, score = fs.sample(_dev(wl.h), _dev(wl.W), bias=_dev(wl.bias), temperature=_dev(tau), mask=_dev(wl.mask),
                           seed=wl.seed, step=4, return_score=True)
    idx_b, _ = fs.sample(_dev(wl.h), _dev(wl.W), bias=_dev(wl.bias), temperature=_dev(tau), mask=_dev(wl.mask),
                         seed=wl.seed + 1, step=99, return_score=True)
    a = oracle_inputs(wl)
    flat = sampler.flat_sample(sampler.scores(a["h"], a["W"], seed=wl.seed, step=4, bias=a["bias"],
                                              temperature=tau.numpy(), mask=a["mask"]))
    check_flat(idx.cpu().numpy(), score.cpu().numpy(), flat)
    g = (tau == 0).numpy()
    assert np.array_equal(idx.cpu().numpy()[g], idx_b.cpu().numpy()[g])    # greedy ignores the RNG


def test_logits_sampler_per_request_and_greedy():
    wl = synth.make_workload("qwen25_7b", 21, V=3000, D=96)
    lg = (wl.h.float() @ wl.W.float().t())
    tau = wl.temperature.clone()
    tau[1::4] = 0.0
    seeds = _seeds(21, 5)
    idx, score, logZ, logprob = fs.sample_logits(lg.cuda(), bias=_dev(wl.bias), temperature=_dev(tau),
                                                 mask=_dev(wl.mask), seeds=torch.tensor(seeds).cuda(), step=8,
                                                 return_all=True)
    a = oracle_inputs(wl)
    flat = sampler.flat_sample(sampler.scores_from_logits(lg.numpy(), seed=0, step=8, bias=a["bias"],
                                                          temperature=tau.numpy(), mask=a["mask"],
                                                          seeds=seeds.astype(np.uint64)))
    check_flat(idx.cpu().numpy(), score.cpu().numpy(), flat)


def test_per_request_chi_square_1e6():
    lt = np.array([0.5, -1.0, 2.0, 0.0, 1.5, -0.5, 1.0, 0.25], np.float32)
    B = 256
    h = torch.tensor(np.tile(lt, (B, 1))).to(torch.bfloat16).cuda()
    W = torch.eye(8).to(torch.bfloat16).cuda()
    seeds = torch.tensor(_seeds(B, 9)).cuda()
    counts = torch.zeros(8, dtype=torch.int64, device="cuda")
    out = torch.empty(B, dtype=torch.int32, device="cuda")
    for s in range(4000):
        counts += torch.bincount(fs.sample(h, W, seeds=seeds, step=s).long(), minlength=8)
    _, p = stats.chi_square(counts.cpu().numpy(), stats.softmax_probs(lt))
    assert p > 1e-3
