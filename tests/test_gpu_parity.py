"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded
inputs, element by element, at sizes spanning several tiles and ragged tails; plus the
invariances the method guarantees (tiling/grid independence, TP shards == 1 GPU, grouped ==
flat).  Parity rule in tests/parity.py."""
import numpy as np
import pytest
import torch

import synth
from oracle import sampler
from parity import GAP, LOGMASS_TOL, SCORE_TOL, check_flat, oracle_flat, oracle_inputs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2603_15854_b200 as fs


def _gpu(wl):
    return synth.Workload(**{**wl.__dict__, **{k: (getattr(wl, k).cuda() if getattr(wl, k) is not None else None)
                                               for k in ("h", "W", "bias", "temperature", "mask")}})


def _run(wl, step, **kw):
    g = _gpu(wl)
    idx, score = fs.sample(g.h, g.W, bias=g.bias, temperature=g.temperature, mask=g.mask, seed=wl.seed,
                           step=step, return_score=True, **kw)
    torch.cuda.synchronize()
    return idx.cpu().numpy(), score.cpu().numpy()


@pytest.fixture(autouse=True)
def _reset_options():
    yield
    if torch.cuda.is_available():
        for k, v in (("force_simt", 0), ("max_ctas", 0), ("pdl", 1), ("stages", 0), ("pair", -1), ("kbps", 0), ("fuse_reduce", 1), ("pdl_w", 0),
                     ("whole_tiles", 1)):
            fs.set_option(k, v)


def test_tiny_fp32_config():
    wl = synth.make_workload("tiny", 4)
    tot = 0
    for step in range(8):
        idx, score = _run(wl, step)
        _, flat = oracle_flat(wl, step)
        e, n = check_flat(idx, score, flat)
        tot += e
    assert tot >= 24


@pytest.mark.parametrize("B", [1, 3, 16, 17, 32, 33, 64, 100, 128, 200, 256, 300])
def test_bf16_tensor_core_shapes(B):
    # V=1000 (ragged last tile), D=200 (K tail: 64+64+64+8), several 16-row units per CTA
    wl = synth.make_workload("llama3_8b", B, V=1000, D=200, seed_offset=B)
    idx, score = _run(wl, 11)
    _, flat = oracle_flat(wl, 11)
    check_flat(idx, score, flat)


@pytest.mark.parametrize("V,D,B", [(4096, 64, 8), (5000, 512, 40), (7777, 136, 5), (129, 4096, 2)])
def test_bf16_more_shapes(V, D, B):
    wl = synth.make_workload("llama3_8b", B, V=V, D=D, seed_offset=V)
    idx, score = _run(wl, 3)
    _, flat = oracle_flat(wl, 3)
    check_flat(idx, score, flat)


def test_bf16_cuda_core_fallback_odd_D():
    wl = synth.make_workload("llama3_8b", 6, V=3000, D=100)   # D % 8 != 0 -> CUDA-core kernel
    idx, score = _run(wl, 5)
    _, flat = oracle_flat(wl, 5)
    check_flat(idx, score, flat)


@pytest.mark.parametrize("B", [8, 40])
def test_transforms_bias_temperature_mask(B):
    wl = synth.make_workload("qwen25_7b", B, V=3000, D=256)
    for step in (0, 1):
        idx, score = _run(wl, step)
        _, flat = oracle_flat(wl, step)
        check_flat(idx, score, flat)


@pytest.mark.parametrize("pattern", ["edge", "peaked", "duplicate"])
def test_patterns(pattern):
    wl = synth.make_workload("llama3_8b", 12, V=2000, D=128, pattern=pattern,
                             with_transforms=(pattern == "edge"))
    idx, score = _run(wl, 2)
    _, flat = oracle_flat(wl, 2)
    check_flat(idx, score, flat)
    if pattern == "edge":
        assert idx[0] == -1 and idx[1] == (2000 * 5) // 7


def test_degenerate_single_token_vocab():
    wl = synth.make_workload("llama3_8b", 3, V=1, D=64)
    idx, score = _run(wl, 0)
    assert idx.tolist() == [0, 0, 0]
    _, flat = oracle_flat(wl, 0)
    check_flat(idx, score, flat)


@pytest.mark.parametrize("V,D,B,pair", [(2, 8, 1, 0), (7, 16, 17, 1), (127, 8, 33, 1), (128, 24, 3, 0),
                                        (129, 8, 64, 1), (255, 16, 2, 0), (256, 8, 100, 1), (257, 24, 256, 1),
                                        (383, 8, 16, 0), (513, 16, 31, -1)])
def test_tiny_vocab_and_width_around_tile_boundaries(V, D, B, pair):
    # smallest TMA-legal widths (D = 8 bf16 = 16 B rows) and V around the 128 / 256-row tile edges, on
    # the 1-CTA and the CTA-pair kernel; whole-tile and 16-row partitions agree bit for bit
    wl = synth.make_workload("qwen25_7b", B, V=V, D=D, seed_offset=V * 3 + D)
    fs.set_option("pair", pair)
    idx, score = _run(wl, 1)
    _, flat = oracle_flat(wl, 1)
    check_flat(idx, score, flat)
    fs.set_option("whole_tiles", 0)
    idx2, score2 = _run(wl, 1)
    assert np.array_equal(idx, idx2) and np.array_equal(score.view(np.uint32), score2.view(np.uint32))


def test_invalid_temperature_rows():
    wl = synth.make_workload("llama3_8b", 4, V=500, D=64)
    wl.temperature = torch.tensor([1.0, -0.5, -1.0, float("nan")])
    idx, score = _run(wl, 0)
    assert idx[1:].tolist() == [-1, -1, -1] and idx[0] >= 0
    assert np.all(np.isneginf(score[1:]))


@pytest.mark.parametrize("max_ctas", [1, 5, 37, 0])
def test_grid_invariance_bit_exact(max_ctas):
    wl = synth.make_workload("llama3_8b", 20, V=6000, D=256)
    ref_idx, ref_score = _run(wl, 9)
    fs.set_option("max_ctas", max_ctas)
    idx, score = _run(wl, 9)
    assert np.array_equal(idx, ref_idx)
    assert np.array_equal(score.view(np.uint32), ref_score.view(np.uint32))


@pytest.mark.parametrize("config,B,V", [("llama3_8b", 1, 152064), ("qwen25_7b", 32, 152064), ("llama3_8b", 256, 151936),
                                        ("qwen25_7b", 8, 16032), ("llama3_8b", 64, 1000), ("qwen25_7b", 200, 40000)])
def test_whole_tile_grid_bit_exact(config, B, V):
    # whole_tiles (default): fewest CTAs (pairs) with whole 128/256-row tiles; 0: 16-row ranges on
    # every SM.  The partition never changes a logit's accumulation -> identical results.
    wl = synth.make_workload(config, B, V=V, D=64, seed_offset=77 + B)
    fs.set_option("whole_tiles", 0)
    ref = _run(wl, 3)
    fs.set_option("whole_tiles", 1)
    got = _run(wl, 3)
    assert np.array_equal(got[0], ref[0])
    assert np.array_equal(got[1].view(np.uint32), ref[1].view(np.uint32))
    if V <= 40000:
        _, flat = oracle_flat(wl, 3)
        check_flat(*got, flat)


def test_stage_ring_depth_and_pdl_invariance():
    wl = synth.make_workload("llama3_8b", 24, V=3000, D=320)
    ref = _run(wl, 4)
    for opt, val in (("stages", 2), ("stages", 3), ("pdl", 0)):
        fs.set_option(opt, val)
        got = _run(wl, 4)
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])


def test_tensor_core_vs_cuda_core_kernel():
    wl = synth.make_workload("llama3_8b", 16, V=2500, D=256)
    tc = _run(wl, 6)
    fs.set_option("force_simt", 1)
    simt = _run(wl, 6)
    _, flat = oracle_flat(wl, 6)
    check_flat(*tc, flat)
    check_flat(*simt, flat)


def test_steps_and_seeds_change_samples():
    wl = synth.make_workload("llama3_8b", 64, V=4000, D=64)
    a = _run(wl, 0)[0]
    b = _run(wl, 1)[0]
    assert (a != b).mean() > 0.5
    again = _run(wl, 0)[0]
    assert np.array_equal(a, again)


def test_cuda_graph_capture_replay():
    wl = _gpu(synth.make_workload("llama3_8b", 8, V=3000, D=128))
    idx = torch.empty(8, dtype=torch.int32, device="cuda")
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        # contexts are per (device, stream): grow this stream's workspace outside capture
        fs.sample(wl.h, wl.W, seed=wl.seed, step=5, out=idx)
        s.synchronize()
        ref = idx.clone()
        idx.zero_()
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            fs.sample(wl.h, wl.W, seed=wl.seed, step=5, out=idx)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(idx, ref)


@pytest.mark.parametrize("B", [1, 16, 40, 100, 128, 200, 256])
def test_cta_pair_kernel_matches_oracle_and_single_cta(B):
    # cta_group::2 (M=256) kernel vs oracle, and bit-identical to the 1-CTA kernel
    wl = synth.make_workload("llama3_8b", B, V=5000 + B, D=320, seed_offset=1000 + B)
    fs.set_option("pair", 0)
    ref = _run(wl, 6)
    fs.set_option("pair", 1)
    got = _run(wl, 6)
    assert np.array_equal(got[0], ref[0])
    assert np.array_equal(got[1].view(np.uint32), ref[1].view(np.uint32))
    _, flat = oracle_flat(wl, 6)
    check_flat(*got, flat)


@pytest.mark.parametrize("max_ctas", [2, 6, 38, 0])
def test_cta_pair_grid_invariance(max_ctas):
    wl = synth.make_workload("qwen25_7b", 64, V=9000, D=192)
    ref = _run(wl, 2)
    fs.set_option("pair", 1)
    fs.set_option("max_ctas", max_ctas)
    got = _run(wl, 2)
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
