"""Exact Gumbel pruning in the one-kernel epilogue (csrc/fs_epilogue.cuh `gumbel_upper`): an element
whose bound l~ + (clz(~r) + 1) ln 2 does not exceed a recorded best score is skipped without
evaluating G32.  The pruned sampler must return the SAME idx and score bits as the unpruned one
on every row -- plain, transformed (bias / tau / mask, greedy rows), per-request streams, peaked and
duplicate-row logits (ties), both stage-1 kernels, ragged shapes -- and still satisfy the parity
rule against the fp64 oracle."""
import numpy as np
import pytest
import torch

import synth
from parity import check_flat, oracle_flat

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2603_15854_b200 as fs


@pytest.fixture(autouse=True)
def _reset():
    yield
    if torch.cuda.is_available():
        for k, v in (("prune", 0), ("pair", -1), ("pdl_w", 0)):
            fs.set_option(k, v)


def _run(wl, step, prune, seeds=None, **kw):
    d = {k: (getattr(wl, k).cuda() if getattr(wl, k) is not None else None)
         for k in ("h", "W", "bias", "temperature", "mask")}
    fs.set_option("prune", prune)
    idx, score = fs.sample(d["h"], d["W"], bias=d["bias"], temperature=d["temperature"], mask=d["mask"],
                           seed=wl.seed, step=step, seeds=seeds, return_score=True, **kw)
    torch.cuda.synchronize()
    return idx.cpu().numpy(), score.cpu().numpy()


CASES = [("llama3_8b", "default", B, V, D) for B, V, D in [(1, 20011, 256), (16, 9000, 128), (40, 30000, 64),
                                                         (256, 12000, 128), (300, 5003, 64)]] + \
        [("qwen25_7b", "default", 33, 15001, 128), ("qwen25_7b", "edge", 64, 8000, 64),
         ("llama3_8b", "peaked", 32, 20000, 256), ("llama3_8b", "duplicate", 24, 16000, 128)]


@pytest.mark.parametrize("cfg,pattern,B,V,D", CASES)
@pytest.mark.parametrize("pair", [0, 1])
def test_pruned_equals_unpruned_bit_for_bit(cfg, pattern, B, V, D, pair):
    wl = synth.make_workload(cfg, B, V=V, D=D, pattern=pattern, seed_offset=B + V)
    fs.set_option("pair", pair)
    for step in (0, 5):
        ref = _run(wl, step, prune=0)
        got = _run(wl, step, prune=1)
        assert np.array_equal(got[0], ref[0])
        assert np.array_equal(got[1].view(np.uint32), ref[1].view(np.uint32))
    _, flat = oracle_flat(wl, 5)
    check_flat(*got, flat)


def test_pruned_greedy_ties_keep_smallest_id():
    # tau = 0 rows are greedy (s = l~, no noise): duplicate W rows give exact ties, and the pruning
    # test (l~ + margin > best) must still let the smaller id win
    wl = synth.make_workload("llama3_8b", 12, V=9000, D=128, pattern="duplicate", seed_offset=3)
    wl.temperature = torch.zeros(12, dtype=torch.float32)
    wl.temperature[::2] = 0.9
    for pair in (0, 1):
        fs.set_option("pair", pair)
        ref = _run(wl, 2, prune=0)
        got = _run(wl, 2, prune=1)
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1].view(np.uint32), ref[1].view(np.uint32))
        greedy = got[0][1::2]
        assert np.all(greedy % 2 == 0)            # of each duplicate pair the even (smaller) id wins


def test_pruned_per_request_streams():
    wl = synth.make_workload("llama3_8b", 40, V=12345, D=128, seed_offset=9)
    seeds = torch.arange(40, dtype=torch.int64, device="cuda") * 7919 + 5
    ref = _run(wl, 3, prune=0, seeds=seeds)
    got = _run(wl, 3, prune=1, seeds=seeds)
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1].view(np.uint32), ref[1].view(np.uint32))


def test_pruned_full_vocab_back_to_back_steps():
    # full Llama vocabulary, PDL across steps: the published bests of one step never leak into the next
    wl = synth.make_workload("llama3_8b", 64, V=128256, D=256, seed_offset=77)
    d = {k: getattr(wl, k).cuda() for k in ("h", "W")}
    outs = {}
    for prune in (0, 1):
        fs.set_option("prune", prune)
        fs.set_option("pdl_w", 1)
        res = []
        for step in range(6):
            idx, score = fs.sample(d["h"], d["W"], seed=wl.seed, step=step, return_score=True)
            res.append((idx.clone(), score.clone()))
        torch.cuda.synchronize()
        outs[prune] = res
    for (a, sa), (b, sb) in zip(outs[0], outs[1]):
        assert torch.equal(a, b) and torch.equal(sa.view(torch.int32), sb.view(torch.int32))
