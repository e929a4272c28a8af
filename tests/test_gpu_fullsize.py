"""GPU parity at BASELINE.json's full sizes, EVERY row, in the launch configuration bench.py times
(fuse_reduce = 1, the one-kernel finalize; pdl_w = 0, the headline, and pdl_w = 1, the pipelined period).

For each configuration the oracle (fp64 over the whole vocabulary, oracle/sampler.py) is run once
on B = 256 rows, in chunks of 32 rows; the GPU is then run at B in {1, 32, 128, 256} on the first
B rows.  A row's noise depends only on its index b (RNG layout R1), so the oracle's first B rows are
exactly the B-row problem.  The north-star rule (parity.check_flat) is applied to every row.

  Llama-3-8B   D=4096 V=128256          fs_sample
  Qwen2.5-7B   D=3584 V=152064          fs_sample, tau 0.7 + bias + 25% mask (transform, R3)
  Gemma-3-27B  D=5376 V=262208          fs_sample_grouped g=4096 (65 groups, ragged last group):
                                        idx, score, logZ, log-prob and every group (M, I, L)
  Llama-3-70B  D=8192 V=128256          fs_sample (n=1) and vocabulary shards n=2,4,8
                                        (fs_sample_shard + fs_combine_summaries) == n=1 bit for bit
"""
import numpy as np
import pytest
import torch

import synth
from oracle import sampler
from parity import GAP, LOGMASS_TOL, SCORE_TOL, check_flat, oracle_inputs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2603_15854_b200 as fs

BS = (1, 32, 128, 256)
STEP = 7
_cache = {}


def _group_near(sc, g):
    """Per (row, group): ids with s >= group max - GAP (capped), for the in-group near-tie rule."""
    R, V = sc.s.shape
    K = (V + g - 1) // g
    near = [[None] * K for _ in range(R)]
    for k in range(K):
        blk = sc.s[:, k * g:min(V, (k + 1) * g)]
        m = blk.max(axis=1)
        for r in range(R):
            ids = np.nonzero(blk[r] >= m[r] - GAP)[0][:16]
            near[r][k] = set(int(sc.v_global[k * g + i]) for i in ids)
    return near


def _oracle(name):
    """Workload (B = 256 rows) on the device + the oracle over every row (cached per config)."""
    if name in _cache:
        return _cache[name]
    wl = synth.make_workload(name, 256)
    a = oracle_inputs(wl)
    flats, groups, gnear, lt_at = [], [], [], []
    ell = sampler.logits(a["h"], a["W"])            # O2 once for all rows (fp64 [256, V])
    for r0 in range(0, 256, 32):
        rows = np.arange(r0, r0 + 32)
        # O3-O5 on those logits (== sampler.scores, pinned in test_oracle_sampler.py)
        sc = sampler.scores_from_logits(ell, seed=wl.seed, step=STEP, rows=rows, bias=a["bias"],
                                        temperature=a["temperature"], mask=a["mask"])
        flat = sampler.flat_sample(sc)
        flats.append(flat)
        lt_at.append(np.array([sc.ltilde[i, flat.idx[i]] if flat.idx[i] >= 0 else -np.inf
                               for i in range(len(rows))]))
        if wl.group_size:
            groups.append(sampler.group_summaries(sc, wl.group_size))
            gnear.extend(_group_near(sc, wl.group_size))
        del sc
    del ell
    flat = sampler.FlatResult(idx=np.concatenate([f.idx for f in flats]), s1=np.concatenate([f.s1 for f in flats]),
                              s2=np.concatenate([f.s2 for f in flats]), gap=np.concatenate([f.gap for f in flats]),
                              near=sum((f.near for f in flats), []), logZ=np.concatenate([f.logZ for f in flats]))
    grp = None
    if groups:
        grp = sampler.GroupResult(M=np.concatenate([g.M for g in groups]), I=np.concatenate([g.I for g in groups]),
                                  L=np.concatenate([g.L for g in groups]), idx=np.concatenate([g.idx for g in groups]),
                                  logZ=np.concatenate([g.logZ for g in groups]))
    dev = {k: (getattr(wl, k).cuda() if getattr(wl, k) is not None else None)
           for k in ("h", "W", "bias", "temperature", "mask")}
    _cache.clear()                       # keep one full-size W on the device at a time
    torch.cuda.empty_cache()
    _cache[name] = (wl, dev, flat, grp, gnear, np.concatenate(lt_at))
    return _cache[name]


def _rows(flat, B):
    return sampler.FlatResult(idx=flat.idx[:B], s1=flat.s1[:B], s2=flat.s2[:B], gap=flat.gap[:B],
                              near=flat.near[:B], logZ=flat.logZ[:B])


@pytest.fixture(autouse=True, params=[0, 1], ids=["pdl0", "pdl1"])
def _bench_launch_config(request):
    # bench.py's two launch configurations: the headline (no cross-step overlap, pdl_w = 0) and the
    # pipelined period (pdl_w = 1: PDL for batch chunks <= 128), both with the one-kernel finalize
    fs.set_option("pdl_w", request.param)
    fs.set_option("fuse_reduce", 1)
    yield
    fs.set_option("pdl_w", 0)


def _sub(t, B):
    return None if t is None else t[:B].contiguous()


@pytest.mark.parametrize("name,B", [(n, b) for n in ("llama3_8b", "qwen25_7b") for b in BS])
def test_fused_sample_every_row(name, B):
    wl, dev, flat, _, _, _ = _oracle(name)
    h = _sub(dev["h"], B)
    for rep in range(2):                 # back-to-back calls (PDL overlap of the W stream)
        idx, score = fs.sample(h, dev["W"], bias=dev["bias"], temperature=_sub(dev["temperature"], B),
                               mask=_sub(dev["mask"], B), seed=wl.seed, step=STEP, return_score=True)
    torch.cuda.synchronize()
    exact, near = check_flat(idx.cpu().numpy(), score.cpu().numpy(), _rows(flat, B))
    assert exact + near == B
    if dev["mask"] is not None:          # a banned token is never sampled
        allowed = synth.unpack_allowed_bits(wl.mask[:B], wl.V)
        assert bool(allowed[torch.arange(B), idx.cpu().long()].all())


@pytest.mark.parametrize("B", BS)
def test_gemma_grouped_every_row_and_group(B):
    wl, dev, flat, grp, gnear, lt_at = _oracle("gemma3_27b")
    h = _sub(dev["h"], B)
    idx, score, logZ, groups, logprob = fs.sample_grouped(h, dev["W"], group_size=wl.group_size, seed=wl.seed,
                                                          step=STEP, return_logprob=True)
    torch.cuda.synchronize()
    check_flat(idx.cpu().numpy(), score.cpu().numpy(), _rows(flat, B))
    assert np.all(np.abs(logZ.cpu().numpy() - flat.logZ[:B]) <= LOGMASS_TOL)
    same = idx.cpu().numpy() == flat.idx[:B]
    lp = logprob.cpu().numpy()
    assert np.all(np.abs(lp[same] - (lt_at[:B] - flat.logZ[:B])[same]) <= LOGMASS_TOL + SCORE_TOL)
    M, I, L = (groups.max_score.cpu().numpy(), groups.idx.cpu().numpy(), groups.log_mass.cpu().numpy())
    assert M.shape == (B, 65)
    assert np.all(np.abs(M - grp.M[:B]) <= SCORE_TOL)
    assert np.all(np.abs(L - grp.L[:B]) <= LOGMASS_TOL)
    for r in range(B):
        for k in range(65):
            assert I[r, k] == grp.I[r, k] or int(I[r, k]) in gnear[r][k], (r, k, I[r, k], grp.I[r, k])
    # max reuse (R8): the grouped sample is the flat sample, bit for bit
    fidx, fscore = fs.sample(h, dev["W"], seed=wl.seed, step=STEP, return_score=True)
    assert torch.equal(idx, fidx) and torch.equal(score.view(torch.int32), fscore.view(torch.int32))


@pytest.mark.parametrize("B", BS)
def test_llama70b_single_and_shards_every_row(B):
    wl, dev, flat, _, _, _ = _oracle("llama3_70b")
    h = _sub(dev["h"], B)
    ref_idx, ref_score = fs.sample(h, dev["W"], seed=wl.seed, step=STEP, return_score=True)
    torch.cuda.synchronize()
    check_flat(ref_idx.cpu().numpy(), ref_score.cpu().numpy(), _rows(flat, B))
    for n in (2, 4, 8):
        parts = [fs.sample_shard(h, dev["W"][a:b], a, wl.V, seed=wl.seed, step=STEP).raw
                 for a, b in sampler.shard_bounds(wl.V, n)]
        idx, score, logZ = fs.combine_summaries(torch.stack(parts), return_all=True)
        assert torch.equal(idx, ref_idx), n
        assert torch.equal(score.view(torch.int32), ref_score.view(torch.int32)), n
        assert np.all(np.abs(logZ.cpu().numpy() - flat.logZ[:B]) <= LOGMASS_TOL), n
