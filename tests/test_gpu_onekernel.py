"""GPU: the one-kernel finalize (the last stage-1 CTA reduces the per-CTA candidates through a
64-bit atomicMax per row; no stage-2 launch) and PDL-launched stage 1 (W streamed before the
dependency wait, every other input after it) give exactly the two-kernel results, and the
oracle's (parity rule in tests/parity.py)."""
import numpy as np
import pytest
import torch

import synth
from parity import check_flat, oracle_flat

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2603_15854_b200 as fs

OPTS = (("fuse_reduce", 1), ("pdl_w", 0), ("pdl", 1), ("pair", -1), ("max_ctas", 0), ("staging_check", 1))


@pytest.fixture(autouse=True)
def _reset_options():
    yield
    if torch.cuda.is_available():
        for k, v in OPTS:
            fs.set_option(k, v)


def _gpu(wl):
    return {k: (getattr(wl, k).cuda() if getattr(wl, k) is not None else None)
            for k in ("h", "W", "bias", "temperature", "mask")}


def _sample(g, wl, step, **kw):
    idx, score = fs.sample(g["h"], g["W"], bias=g["bias"], temperature=g["temperature"], mask=g["mask"],
                           seed=wl.seed, step=step, return_score=True, **kw)
    torch.cuda.synchronize()
    return idx.cpu().numpy(), score.cpu().numpy()


@pytest.mark.parametrize("B", [1, 5, 32, 33, 100, 256, 300])
@pytest.mark.parametrize("config", ["llama3_8b", "qwen25_7b"])
def test_one_kernel_equals_two_kernels_and_oracle(B, config):
    wl = synth.make_workload(config, B, V=5000, D=256, seed_offset=7 * B)
    g = _gpu(wl)
    fs.set_option("fuse_reduce", 0)
    i2, s2 = _sample(g, wl, 3)
    fs.set_option("fuse_reduce", 1)
    i1, s1 = _sample(g, wl, 3)
    np.testing.assert_array_equal(i1, i2)
    np.testing.assert_array_equal(s1.view(np.uint32), s2.view(np.uint32))
    if B <= 33:
        _, flat = oracle_flat(wl, 3)
        check_flat(i1, s1, flat)


@pytest.mark.parametrize("pair", [0, 1])
def test_one_kernel_undefined_rows_and_many_calls(pair):
    # edge pattern: one fully masked row (-> -1), one single-token row, per-row tau; 40 calls in a
    # row must keep the finalize buffer / counter consistent (reset by the last CTA)
    fs.set_option("pair", pair)
    wl = synth.make_workload("qwen25_7b", 40, V=3000, D=128, pattern="edge", seed_offset=3)
    g = _gpu(wl)
    outs = []
    for step in range(40):
        outs.append(_sample(g, wl, step))
    fs.set_option("fuse_reduce", 0)
    for step in (0, 17, 39):
        i2, s2 = _sample(g, wl, step)
        np.testing.assert_array_equal(outs[step][0], i2)
        np.testing.assert_array_equal(outs[step][1].view(np.uint32), s2.view(np.uint32))
    _, flat = oracle_flat(wl, 17)
    check_flat(outs[17][0], outs[17][1], flat)
    assert (outs[17][0] == -1).any()


@pytest.mark.parametrize("B", [8, 64])
def test_pdl_w_respects_producer_kernels(B):
    # Each call's h and temperature are written by a torch kernel IMMEDIATELY before the call on the
    # same stream; with pdl_w the stage-1 kernel streams W before its dependency wait, so any read
    # of h / tau before it would see stale values and change the sample.
    wl = synth.make_workload("qwen25_7b", B, V=20000, D=512, seed_offset=B)
    g = _gpu(wl)
    h0, t0 = g["h"].clone(), g["temperature"].clone()
    ref = []
    for step in range(6):
        g["h"].copy_(h0 * (1.0 + 0.25 * step))
        g["temperature"].copy_(t0 * (1.0 + 0.1 * step))
        ref.append(_sample(g, wl, step))
    fs.set_option("pdl_w", 1)
    got = []
    for step in range(6):
        g["h"].copy_(h0 * (1.0 + 0.25 * step))
        g["temperature"].copy_(t0 * (1.0 + 0.1 * step))
        idx, score = fs.sample(g["h"], g["W"], bias=g["bias"], temperature=g["temperature"], mask=g["mask"],
                               seed=wl.seed, step=step, return_score=True)
        got.append((idx, score))                       # no host sync between steps
    torch.cuda.synchronize()
    for (ir, sr), (ig, sg) in zip(ref, got):
        np.testing.assert_array_equal(ir, ig.cpu().numpy())
        np.testing.assert_array_equal(sr.view(np.uint32), sg.cpu().numpy().view(np.uint32))


def test_pdl_w_back_to_back_full_size_and_graph():
    # Llama-3-8B LM head, B=32: 20 back-to-back PDL calls into distinct outputs, then the same loop
    # captured in a CUDA graph and replayed -- all equal the two-kernel results per step.
    D, V, B = 4096, 128256, 32
    gen = torch.Generator(device="cuda").manual_seed(5)
    W = (torch.randn(V, D, device="cuda", generator=gen) * 0.02).to(torch.bfloat16)
    h = torch.randn(B, D, device="cuda", generator=gen).to(torch.bfloat16)
    fs.set_option("fuse_reduce", 0)
    ref = [fs.sample(h, W, seed=9, step=s) for s in range(20)]
    torch.cuda.synchronize()
    fs.set_option("fuse_reduce", 1)
    fs.set_option("pdl_w", 1)
    outs = [torch.empty(B, dtype=torch.int32, device="cuda") for _ in range(20)]
    for s in range(20):
        fs.sample(h, W, seed=9, step=s, out=outs[s])
    torch.cuda.synchronize()
    for s in range(20):
        assert torch.equal(ref[s], outs[s]), s
    stream = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    for o in outs:
        o.fill_(-7)
    with torch.cuda.stream(stream):
        fs.sample(h, W, seed=9, step=0, out=outs[0])      # warm-up on the capture stream
        stream.synchronize()
        with torch.cuda.graph(graph, stream=stream):
            for s in range(20):
                fs.sample(h, W, seed=9, step=s, out=outs[s])
    graph.replay()
    torch.cuda.synchronize()
    for s in range(20):
        assert torch.equal(ref[s], outs[s]), s


@pytest.mark.parametrize("nbytes", [16, 4096 + 16, 262144, 3 * 1048576 + 48])
def test_copy_async_pinned_and_device(nbytes):
    src = torch.randint(0, 256, (nbytes,), dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    fs.copy_async(dst, src)
    torch.cuda.synchronize()
    assert torch.equal(dst.cpu(), src)
    dst2 = torch.empty_like(dst)
    fs.set_option("pdl_w", 1)
    fs.copy_async(dst2, dst)
    torch.cuda.synchronize()
    assert torch.equal(dst2, dst)


def test_copy_async_rejects_pageable_and_misaligned():
    dst = torch.empty(64, dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        fs.copy_async(dst, torch.zeros(64, dtype=torch.uint8))          # pageable host memory
    src = torch.zeros(80, dtype=torch.uint8).pin_memory()
    with pytest.raises(fs._lib.FlashSampleError):
        fs.copy_async(dst, src[1:65])                                  # misaligned source


@pytest.mark.parametrize("pdl_w", [0, 1])
def test_sample_from_host_equals_device_path(pdl_w):
    # end-to-end path: inputs staged by the copy kernel, ids written by the sampling kernel straight
    # into pinned host memory; each step's host inputs change and no host sync happens in between
    fs.set_option("pdl_w", pdl_w)
    wl = synth.make_workload("qwen25_7b", 24, V=20000, D=512, seed_offset=11)
    g = _gpu(wl)
    hs = [(wl.h * (1.0 + 0.2 * s)).to(wl.h.dtype).pin_memory() for s in range(5)]
    ts = [(wl.temperature * (1.0 + 0.1 * s)).pin_memory() for s in range(5)]
    m_host = wl.mask.pin_memory()
    h_dev, t_dev, m_dev = torch.empty_like(g["h"]), torch.empty_like(g["temperature"]), torch.empty_like(g["mask"])
    outs = [torch.empty(24, dtype=torch.int32).pin_memory() for _ in range(5)]
    for s in range(5):
        fs.sample_from_host(hs[s], g["W"], temperature_host=ts[s], mask_host=m_host, bias=g["bias"], seed=wl.seed,
                            step=s, h_dev=h_dev, t_dev=t_dev, m_dev=m_dev, idx_host=outs[s])
    torch.cuda.synchronize()
    for s in range(5):
        ref = fs.sample(hs[s].cuda(), g["W"], bias=g["bias"], temperature=ts[s].cuda(), mask=g["mask"],
                        seed=wl.seed, step=s)
        assert torch.equal(ref.cpu(), outs[s]), s


@pytest.mark.parametrize("B", [1, 7, 64, 256, 300])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_logits_sampler_one_kernel_equals_two_kernels(B, dtype):
    # fs_sample_logits: the last block finalizes (B <= 256) == the stage-2 reduce kernel, bit for bit
    wl = synth.make_workload("qwen25_7b", B, V=9000, D=64, seed_offset=B)
    lg = (wl.h.float() @ wl.W.float().t() * 3.0).to(dtype).cuda()
    kw = dict(bias=wl.bias.cuda(), temperature=wl.temperature.cuda(), mask=wl.mask.cuda(), seed=wl.seed, step=4)
    seeds = torch.arange(B, device="cuda", dtype=torch.int64) * 31 + 7
    res = {}
    for fuse in (0, 1):
        fs.set_option("fuse_reduce", fuse)
        res[fuse] = [fs.sample_logits(lg, return_score=True, **kw),
                     fs.sample_logits(lg, seeds=seeds, return_score=True, **kw),
                     fs.sample_logits(lg, return_all=True, **kw)[:2]]          # log-mass: stage 2 both times
        torch.cuda.synchronize()
    for (i0, s0), (i1, s1) in zip(res[0], res[1]):
        assert torch.equal(i0, i1)
        assert torch.equal(s0.view(torch.int32), s1.view(torch.int32))


@pytest.mark.parametrize("B", [1, 32, 64, 300])
@pytest.mark.parametrize("pdl_w", [0, 1])
def test_sample_staged_in_kernel_equals_device_path(B, pdl_w):
    # fs_sample_staged: every CTA copies its slice of the pinned host h into the device buffer after the
    # dependency wait, a grid counter orders it before the first h load; temperature read from pinned
    # host memory; ids written into pinned host memory.  5 steps with changing inputs, no host syncs.
    fs.set_option("pdl_w", pdl_w)
    wl = synth.make_workload("qwen25_7b", B, V=20000, D=512, seed_offset=13 + B)
    W, bias = wl.W.cuda(), wl.bias.cuda()
    hs = [(wl.h * (1.0 + 0.2 * s)).to(wl.h.dtype).pin_memory() for s in range(5)]
    ts = [(wl.temperature * (1.0 + 0.1 * s)).pin_memory() for s in range(5)]
    h_dev = torch.empty(hs[0].shape, dtype=hs[0].dtype, device="cuda")
    outs = [torch.full((B,), -7, dtype=torch.int32).pin_memory() for _ in range(5)]
    for s in range(5):
        fs.sample_from_host(hs[s], W, temperature_host=ts[s], bias=bias, seed=wl.seed, step=s, h_dev=h_dev,
                            idx_host=outs[s])
    torch.cuda.synchronize()
    for s in range(5):
        ref = fs.sample(hs[s].cuda(), W, bias=bias, temperature=ts[s].cuda(), seed=wl.seed, step=s)
        assert torch.equal(ref.cpu(), outs[s]), s


@pytest.mark.parametrize("B", [1, 13, 16, 40])
def test_one_kernel_log_mass_and_shard_equal_stage2(B):
    # single group with logZ / log-prob (and a TP shard's summary): the last stage-1 CTA runs the
    # per-row reduce (B <= 16; larger B keep the stage-2 kernel) -- bit-identical to the stage-2 kernel
    wl = synth.make_workload("qwen25_7b", B, V=7001, D=256, seed_offset=5 * B)
    g = _gpu(wl)
    kw = dict(bias=g["bias"], temperature=g["temperature"], mask=g["mask"], seed=wl.seed, step=6)
    out = {}
    for fuse in (0, 1):
        fs.set_option("fuse_reduce", fuse)
        r = fs.sample(g["h"], g["W"], return_score=True, return_logprob=True, **kw)
        sh = fs.sample_shard(g["h"], g["W"][2000:5000].contiguous(), 2000, 7001, bias_shard=g["bias"][2000:5000],
                             temperature=g["temperature"], mask=g["mask"], seed=wl.seed, step=6)
        torch.cuda.synchronize()
        out[fuse] = list(r) + [sh.raw]
    for a, b in zip(out[0], out[1]):
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))


@pytest.mark.parametrize("opts", [{}, {"pair": 0}, {"pair": 1}, {"max_ctas": 37}, {"unit_rows": 64},
                                  {"force_simt": 1}])
@pytest.mark.parametrize("V,g,B", [(20011, 4096, 9), (9000, 128, 40), (5000, 640, 3), (7000, 1024, 100)])
def test_grouped_host_slot_ranges_equal_device_search(opts, V, g, B):
    # grouped stage 2 with host-computed group slot ranges (warp per (row, group); the last warp of a
    # row merges the groups in order) == the block-per-row kernel with a device binary search over the
    # ids stage 1 wrote (every slot layout: 1-CTA, CTA pair, capped grid, coarse units, CUDA-core).
    # Maxima / ids exact; log-masses are summed in another order (fp32 rounding only).
    wl = synth.make_workload("qwen25_7b", B, V=V, D=128, seed_offset=V % 97 + B)
    g_ = _gpu(wl)
    for k, v in opts.items():
        fs.set_option(k, v)
    out = {}
    for r in (0, 1):
        fs.set_option("grp_ranges", r)
        res = fs.sample_grouped(g_["h"], g_["W"], group_size=g, bias=g_["bias"], temperature=g_["temperature"],
                                mask=g_["mask"], seed=wl.seed, step=2, return_groups=True)
        torch.cuda.synchronize()
        out[r] = [res[0], res[1], res[2], res[3].raw]
    for k in ("grp_ranges", "force_simt", "unit_rows"):
        fs.set_option(k, {"grp_ranges": 1}.get(k, 0))
    assert torch.equal(out[0][0], out[1][0]) and torch.equal(out[0][1], out[1][1])
    torch.testing.assert_close(out[0][2], out[1][2], rtol=1e-6, atol=1e-6)
    g0, g1 = out[0][3], out[1][3]
    assert torch.equal(g0[..., :2], g1[..., :2])                       # max_score, idx
    torch.testing.assert_close(g0[..., 2].view(torch.float32), g1[..., 2].view(torch.float32), rtol=1e-6,
                               atol=1e-6)


@pytest.mark.parametrize("B", [8, 64])
def test_staged_grid_too_large_falls_back_to_copy_kernel(B):
    # in-kernel staging needs every CTA co-resident.  A persistent grid larger than the
    # device (max_ctas > #SMs) must be staged by the copy kernel instead -- same ids, counted.
    wl = synth.make_workload("llama3_8b", B, V=60000, D=256, seed_offset=3)
    W = wl.W.cuda()
    h_host = wl.h.pin_memory()
    h_dev = torch.empty(h_host.shape, dtype=h_host.dtype, device="cuda")
    out = torch.full((B,), -7, dtype=torch.int32).pin_memory()
    n_sms = int(fs.query("num_sms"))
    fs.set_option("max_ctas", 2 * n_sms + 2)
    before = fs.query("staged_fallbacks")
    fs.sample_from_host(h_host, W, seed=wl.seed, step=3, h_dev=h_dev, idx_host=out)
    torch.cuda.synchronize()
    assert fs.query("staged_fallbacks") == before + 1
    ref = fs.sample(wl.h.cuda(), W, seed=wl.seed, step=3)
    assert torch.equal(ref.cpu(), out)


def test_staging_barrier_timeout_is_recoverable():
    # Forced in-kernel staging with a grid that cannot be co-resident: the resident CTAs give up the
    # grid barrier after ~5 s instead of trapping; the call completes with every row undefined
    # (idx -1), the event is counted, and the context keeps working (no sticky CUDA error).
    B = 4
    wl = synth.make_workload("llama3_8b", B, V=80000, D=128, seed_offset=4)
    W = wl.W.cuda()
    h_host = wl.h.pin_memory()
    h_dev = torch.empty(h_host.shape, dtype=h_host.dtype, device="cuda")
    out = torch.full((B,), -7, dtype=torch.int32).pin_memory()
    n_sms = int(fs.query("num_sms"))
    fs.set_option("max_ctas", 3 * n_sms)
    fs.set_option("staging_check", 0)
    before = fs.query("staging_timeouts")
    fs.sample_from_host(h_host, W, seed=wl.seed, step=1, h_dev=h_dev, idx_host=out)
    torch.cuda.synchronize()
    assert fs.query("staging_timeouts") == before + 1
    assert bool((out == -1).all())
    fs.set_option("staging_check", 1)
    fs.set_option("max_ctas", 0)
    fs.sample_from_host(h_host, W, seed=wl.seed, step=1, h_dev=h_dev, idx_host=out)
    torch.cuda.synchronize()
    ref = fs.sample(wl.h.cuda(), W, seed=wl.seed, step=1)
    assert torch.equal(ref.cpu(), out)


def test_contexts_per_stream_sample_concurrently():
    # the binding keys contexts by (device, stream), so two streams sampling at once use
    # separate workspaces; results equal the serial calls bit for bit.
    wl = synth.make_workload("qwen25_7b", 48, V=30000, D=256, seed_offset=9)
    g = _gpu(wl)
    serial = [_sample(g, wl, s) for s in (1, 2)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    torch.cuda.synchronize()
    for rep in range(3):
        res = []
        for s, st in zip((1, 2), streams):
            with torch.cuda.stream(st):
                res.append(fs.sample(g["h"], g["W"], bias=g["bias"], temperature=g["temperature"], mask=g["mask"],
                                     seed=wl.seed, step=s, return_score=True))
        outs.append(res)
    torch.cuda.synchronize()
    for res in outs:
        for (i, sc), (ri, rs) in zip(res, serial):
            assert np.array_equal(i.cpu().numpy(), ri) and np.array_equal(sc.cpu().numpy(), rs)


@pytest.mark.parametrize("B", [1, 32, 300])
def test_host_step_sampler_done_flag_serving_loop(B):
    """HostStepSampler: the prepared fs_sample_staged call on a context of its own, completion by
    spinning on the pinned done flag the finalizing CTA sets (option "done_flag") instead of a stream
    sync.  A serving loop rewrites h_host between steps; every step's ids must equal the device path
    on that step's h, and be complete when wait() returns."""
    wl = synth.make_workload("llama3_8b", B, V=20011, D=256, seed_offset=B + 31)
    W = wl.W.cuda()
    h_host = torch.empty_like(wl.h).pin_memory()
    s = fs.HostStepSampler(h_host, W, seed=wl.seed)
    g = torch.Generator().manual_seed(B)
    for step in range(6):
        h_step = torch.randn(wl.h.shape, generator=g).to(torch.bfloat16)
        h_host.copy_(h_step)
        s(step)
        got = s.wait().clone()
        assert int(s.done[0]) == 1
        ref = fs.sample(h_step.cuda(), W, seed=wl.seed, step=step)
        torch.cuda.synchronize()
        assert torch.equal(got, ref.cpu()), step
