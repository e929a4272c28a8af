"""GPU: seeded random configurations against the fp64 oracle -- shapes, ragged tails, transforms,
per-request streams, kernel choices (1-CTA / CTA pair / CUDA core), grid caps and CTA range
granularity drawn together, so that combinations no hand-written case covers are exercised.  Every
case applies the north-star parity rule (tests/parity.py) and, for the tensor-core variants, checks
bit-identity with the default launch of the same inputs (the partition and kernel never change a
logit's accumulation)."""
import numpy as np
import pytest
import torch

import synth
from parity import check_flat, oracle_flat
from oracle import sampler

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2603_15854_b200 as fs

OPTS = {"pair": [-1, 0, 1], "whole_tiles": [0, 1], "max_ctas": [0, 0, 3, 17, 64], "unit_rows": [0, 0, 32, 64],
        "kbps": [0, 0, 1, 2], "pdl_w": [0, 1]}
N_CASES = 40


def _case(i):
    r = np.random.default_rng(0xF0CC + i)
    config = ["llama3_8b", "qwen25_7b"][i % 2]
    B = int(r.choice([1, 2, 7, 16, 17, 31, 33, 64, 100, 128, 200, 256, 257]))
    V = int(r.integers(200, 24000))
    D = int(r.choice([64, 72, 136, 256, 520]))
    opts = {k: v[int(r.integers(len(v)))] for k, v in OPTS.items()}
    per_request = bool(r.random() < 0.25)
    return config, B, V, D, opts, per_request


@pytest.fixture(autouse=True)
def _reset():
    yield
    if torch.cuda.is_available():
        for k in OPTS:
            fs.set_option(k, -1 if k == "pair" else (1 if k == "whole_tiles" else 0))


@pytest.mark.parametrize("i", range(N_CASES))
def test_random_configuration_matches_oracle(i):
    config, B, V, D, opts, per_request = _case(i)
    wl = synth.make_workload(config, B, V=V, D=D, seed_offset=500 + i)
    g = {k: (getattr(wl, k).cuda() if getattr(wl, k) is not None else None)
         for k in ("h", "W", "bias", "temperature", "mask")}
    seeds = steps = None
    if per_request:
        seeds = torch.arange(B, dtype=torch.int64, device="cuda") * 7919 + 11
        steps = torch.full((B,), 3, dtype=torch.int64, device="cuda")

    def run():
        idx, score = fs.sample(g["h"], g["W"], bias=g["bias"], temperature=g["temperature"], mask=g["mask"],
                               seed=wl.seed, step=3, seeds=seeds, steps=steps, return_score=True)
        torch.cuda.synchronize()
        return idx.cpu().numpy(), score.cpu().numpy()
    ref = run()                                   # default launch
    for k, v in opts.items():
        fs.set_option(k, v)
    got = run()
    assert np.array_equal(got[0], ref[0]), (config, B, V, D, opts)
    assert np.array_equal(got[1].view(np.uint32), ref[1].view(np.uint32)), (config, B, V, D, opts)
    if per_request:
        a = {k: synth.as_numpy_exact(getattr(wl, k)) for k in ("h", "W", "bias", "temperature", "mask")}
        sc = sampler.scores(a["h"], a["W"], seed=0, step=0, bias=a["bias"], temperature=a["temperature"],
                            mask=a["mask"], seeds=seeds.cpu().numpy(), steps=steps.cpu().numpy())
        flat = sampler.flat_sample(sc)
    else:
        _, flat = oracle_flat(wl, 3)
    check_flat(*got, flat)
