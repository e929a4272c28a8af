"""GPU parity of the grouped/online variant (per-group log-mass summaries, §4.1, App. E) and the
vocabulary-sharded TP variant (Alg. A.4) simulated shard by shard on one GPU.

Pathwise claims checked bit-exactly (max reuse, P:286 / reading R8):
  grouped idx and score == fs_sample idx and score;  TP combine(idx, score) == fs_sample.
Against the oracle: group (M, I, L) and logZ within the parity tolerances."""
import numpy as np
import pytest
import torch

import synth
from oracle import sampler
from parity import GAP, LOGMASS_TOL, SCORE_TOL, check_flat, oracle_flat, oracle_inputs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2603_15854_b200 as fs


def _dev(t):
    return None if t is None else t.cuda()


def _groups_vs_oracle(groups, sc, g):
    ref = sampler.group_summaries(sc, g)
    M = groups.max_score.cpu().numpy()
    I = groups.idx.cpu().numpy()
    L = groups.log_mass.cpu().numpy()
    assert M.shape == ref.M.shape
    fin = np.isfinite(ref.M)
    assert np.array_equal(np.isfinite(M), fin)
    assert np.all(np.abs(M[fin] - ref.M[fin]) <= SCORE_TOL)
    assert np.all(np.abs(L[fin] - ref.L[fin]) <= LOGMASS_TOL)
    assert np.all(I[~fin] == -1)
    # group argmax: exact where the in-group top-2 gap exceeds 1e-2
    R, K = ref.M.shape
    for r in range(R):
        for k in range(K):
            if not fin[r, k]:
                continue
            blk = sc.s[r, k * g:(k + 1) * g]
            top2 = np.sort(blk)[-2:] if blk.size > 1 else np.array([-np.inf, blk[0]])
            if top2[1] - top2[0] > GAP:
                assert I[r, k] == ref.I[r, k]
            else:
                assert blk[I[r, k] - k * g] >= top2[1] - GAP


@pytest.mark.parametrize("V,g", [(5000, 128), (5000, 1024), (5064, 4096), (262208 // 16, 4096)])
def test_grouped_matches_flat_and_oracle(V, g):
    wl = synth.make_workload("gemma3_27b", 6, V=V, D=192)
    h, W = wl.h.cuda(), wl.W.cuda()
    idx, score, logZ, groups = fs.sample_grouped(h, W, group_size=g, seed=wl.seed, step=3)
    fidx, fscore = fs.sample(h, W, seed=wl.seed, step=3, return_score=True)
    torch.cuda.synchronize()
    assert torch.equal(idx, fidx)
    assert torch.equal(score.view(torch.int32), fscore.view(torch.int32))
    sc, flat = oracle_flat(wl, 3)
    check_flat(idx.cpu().numpy(), score.cpu().numpy(), flat)
    assert np.all(np.abs(logZ.cpu().numpy() - flat.logZ) <= LOGMASS_TOL)
    _groups_vs_oracle(groups, sc, g)


def test_grouped_with_transforms_and_edges():
    wl = synth.make_workload("qwen25_7b", 10, V=3000, D=128, pattern="edge")
    a = oracle_inputs(wl)
    idx, score, logZ, groups = fs.sample_grouped(wl.h.cuda(), wl.W.cuda(), group_size=512, bias=_dev(wl.bias),
                                                 temperature=_dev(wl.temperature), mask=_dev(wl.mask),
                                                 seed=wl.seed, step=1)
    sc, flat = oracle_flat(wl, 1)
    check_flat(idx.cpu().numpy(), score.cpu().numpy(), flat)
    lz = logZ.cpu().numpy()
    assert lz[0] == -np.inf
    fin = np.isfinite(flat.logZ)
    assert np.all(np.abs(lz[fin] - flat.logZ[fin]) <= LOGMASS_TOL)
    _groups_vs_oracle(groups, sc, 512)


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_tp_shards_reproduce_single_gpu_bit_exact(n):
    V, D, B = 6000, 256, 33
    wl = synth.make_workload("llama3_70b", B, V=V, D=D, with_transforms=True)
    h, W, bias, tau, mask = (x.cuda() for x in (wl.h, wl.W, wl.bias, wl.temperature, wl.mask))
    ref_idx, ref_score = fs.sample(h, W, bias=bias, temperature=tau, mask=mask, seed=wl.seed, step=7,
                                   return_score=True)
    parts = []
    for a, b in sampler.shard_bounds(V, n):
        parts.append(fs.sample_shard(h, W[a:b].contiguous(), a, V, bias_shard=bias[a:b].contiguous(),
                                     temperature=tau, mask=mask, seed=wl.seed, step=7).raw)
    gathered = torch.stack(parts)
    idx, score, logZ = fs.combine_summaries(gathered, return_all=True)
    torch.cuda.synchronize()
    assert torch.equal(idx, ref_idx)
    assert torch.equal(score.view(torch.int32), ref_score.view(torch.int32))
    sc, flat = oracle_flat(wl, 7)
    check_flat(idx.cpu().numpy(), score.cpu().numpy(), flat)
    fin = np.isfinite(flat.logZ)
    assert np.all(np.abs(logZ.cpu().numpy()[fin] - flat.logZ[fin]) <= LOGMASS_TOL)
    # per-rank summaries vs the oracle's shard summaries (O8)
    _, _, _, (Ms, Is, Ls) = sampler.tp_sample(**{k: v for k, v in oracle_inputs(wl).items() if k != "h"},
                                              h=oracle_inputs(wl)["h"], n=n, seed=wl.seed, step=7)
    G = fs.Summaries(gathered)
    fin = np.isfinite(Ms)
    assert np.all(np.abs(G.max_score.cpu().numpy()[fin] - Ms[fin]) <= SCORE_TOL)
    assert np.all(np.abs(G.log_mass.cpu().numpy()[fin] - Ls[fin]) <= LOGMASS_TOL)


def test_merge_summaries_online():
    wl = synth.make_workload("gemma3_27b", 5, V=4096, D=128)
    h, W = wl.h.cuda(), wl.W.cuda()
    idx, score, logZ, groups = fs.sample_grouped(h, W, group_size=512, seed=1, step=0)
    run = fs.Summaries(groups.raw[:, 0].contiguous())
    for k in range(1, 8):                                   # Alg. A.3 stream over groups
        run = fs.merge_summaries(run, fs.Summaries(groups.raw[:, k].contiguous()))
    torch.cuda.synchronize()
    assert torch.equal(run.idx, idx)
    assert torch.allclose(run.log_mass, logZ, atol=1e-4)


@pytest.fixture
def pair_on():
    fs.set_option("pair", 1)
    yield
    fs.set_option("pair", -1)


def test_grouped_and_tp_on_cta_pairs(pair_on):
    wl = synth.make_workload("gemma3_27b", 40, V=9000, D=128, with_transforms=True)
    h, W, bias, tau, mask = (x.cuda() for x in (wl.h, wl.W, wl.bias, wl.temperature, wl.mask))
    idx, score, logZ, groups = fs.sample_grouped(h, W, group_size=1024, bias=bias, temperature=tau, mask=mask,
                                                 seed=wl.seed, step=2)
    fidx, fscore = fs.sample(h, W, bias=bias, temperature=tau, mask=mask, seed=wl.seed, step=2, return_score=True)
    assert torch.equal(idx, fidx) and torch.equal(score, fscore)
    sc, flat = oracle_flat(wl, 2)
    check_flat(idx.cpu().numpy(), score.cpu().numpy(), flat)
    _groups_vs_oracle(groups, sc, 1024)
    parts = [fs.sample_shard(h, W[a:b].contiguous(), a, wl.V, bias_shard=bias[a:b].contiguous(), temperature=tau,
                             mask=mask, seed=wl.seed, step=2).raw for a, b in sampler.shard_bounds(wl.V, 4)]
    tidx, tscore, _ = fs.combine_summaries(torch.stack(parts), return_all=True)
    assert torch.equal(tidx, fidx) and torch.equal(tscore, fscore)


@pytest.fixture
def grp_ranges_reset():
    yield
    fs.set_option("grp_ranges", 1)


@pytest.mark.parametrize("B", [65, 128, 256])
@pytest.mark.parametrize("ranges", [1, 0])
def test_grouped_large_batch_stage2_vs_oracle(B, ranges, grp_ranges_reset):
    """B > 64 takes the block-per-row stage 2 (reduce_groups_kernel, host slot ranges or the device
    binary search); every row, every group against the oracle (O7, §4.1)."""
    fs.set_option("grp_ranges", ranges)
    wl = synth.make_workload("gemma3_27b", B, V=9000 + 64, D=128, with_transforms=True)
    h, W, bias, tau, mask = (x.cuda() for x in (wl.h, wl.W, wl.bias, wl.temperature, wl.mask))
    idx, score, logZ, groups, logprob = fs.sample_grouped(h, W, group_size=1024, bias=bias, temperature=tau,
                                                          mask=mask, seed=wl.seed, step=4, return_logprob=True)
    fidx, fscore = fs.sample(h, W, bias=bias, temperature=tau, mask=mask, seed=wl.seed, step=4, return_score=True)
    torch.cuda.synchronize()
    assert torch.equal(idx, fidx) and torch.equal(score.view(torch.int32), fscore.view(torch.int32))
    sc, flat = oracle_flat(wl, 4)
    check_flat(idx.cpu().numpy(), score.cpu().numpy(), flat)
    fin = np.isfinite(flat.logZ)
    assert np.all(np.abs(logZ.cpu().numpy()[fin] - flat.logZ[fin]) <= LOGMASS_TOL)
    lp_ref = sampler.log_prob(sc, flat)
    same = idx.cpu().numpy() == flat.idx
    assert np.all(np.abs(logprob.cpu().numpy()[same] - lp_ref[same]) <= LOGMASS_TOL + SCORE_TOL)
    _groups_vs_oracle(groups, sc, 1024)
