"""GPU test of the peer-memory TP exchange ("an equivalent reduction";
include/flashsample.h fs_comm_window_* / fs_sample_tp_push).

Only one GPU is available, so the ranks are separate processes on the SAME device: each maps the
others' exchange windows through CUDA IPC and the push/flag/ack protocol runs exactly as between
GPUs (the stores just do not cross NVLink).  Every rank must return the single-GPU fs_sample
result bit for bit (shards keyed by global ids, no split-K), over several consecutive steps so
both parity slots and the reader acknowledgements are exercised."""
import os
import socket

import numpy as np

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, B, V, D, steps, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        import synth
        import paper_2603_15854_b200 as fs
        from paper_2603_15854_b200 import tp
        wl = synth.make_workload(cfg, B, V=V, D=D, seed_offset=world)
        dev = torch.device("cuda", 0)
        h, W = wl.h.to(dev), wl.W.to(dev)
        bias = None if wl.bias is None else wl.bias.to(dev)
        tau = None if wl.temperature is None else wl.temperature.to(dev)
        mask = None if wl.mask is None else wl.mask.to(dev)
        lo, hi = tp.shard_bounds(V, world, rank)
        tp.PushExchange(B_max=B)
        from parity import check_flat, oracle_flat
        out = []
        for s in range(steps):
            idx, score, logZ = tp.sample_tp_push_step(
                h, W[lo:hi].contiguous(), lo, V, bias_shard=None if bias is None else bias[lo:hi].contiguous(),
                temperature=tau, mask=mask, seed=wl.seed, step=s, return_all=True)
            ref_idx, ref_score = fs.sample(h, W, bias=bias, temperature=tau, mask=mask, seed=wl.seed, step=s,
                                           return_score=True)
            oracle_ok = True
            if s in (0, steps - 1):          # the exchanged result against the fp64 oracle (every row)
                _, flat = oracle_flat(wl, s)
                check_flat(idx.cpu().numpy(), score.cpu().numpy(), flat)
                fin = np.isfinite(flat.logZ)
                oracle_ok = bool(np.all(np.abs(logZ.cpu().numpy()[fin] - flat.logZ[fin]) <= 1e-3))
            # idx-only step: the whole exchange fused into the shard kernel's finalizing CTA (one kernel)
            idx1 = tp.sample_tp_push_step(
                h, W[lo:hi].contiguous(), lo, V, bias_shard=None if bias is None else bias[lo:hi].contiguous(),
                temperature=tau, mask=mask, seed=wl.seed, step=s)
            out.append((torch.equal(idx, ref_idx) and torch.equal(idx1, ref_idx),
                        torch.equal(score.view(torch.int32), ref_score.view(torch.int32)), oracle_ok))
        timeouts = fs.query("comm_timeouts")
        dist.barrier()                       # peers stay mapped until everyone is done
        fs.comm_window_destroy()
        q.put((rank, out, timeouts, None))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, None, None, repr(e)))


# with logZ: B <= 16 the last stage-1 CTA pushes, 17..256 the stage-2 row reduce pushes, > 256 a separate push
# kernel; idx only (B <= 256): push, wait and combine all in the shard kernel's finalizing CTA
@pytest.mark.parametrize("world,cfg,B,V,D", [(2, "llama3_8b", 8, 20011, 256), (3, "qwen25_7b", 33, 9001, 128),
                                             (4, "llama3_8b", 1, 4096, 64), (2, "qwen25_7b", 300, 5003, 64)])
def test_push_exchange_matches_single_gpu(world, cfg, B, V, D):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, B, V, D, 5, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, out, timeouts, err in res:
        assert err is None, (rank, err)
        assert timeouts == 0
        assert all(a and b and c for a, b, c in out), (rank, out)


def test_nccl_sample_tp_world1_equals_single_gpu():
    """fs_comm_init + fs_sample_tp (library NCCL, §8(b)) on a one-rank communicator: the whole
    shard -> ncclAllGather -> combine sequence runs on the device and equals fs_sample / the oracle."""
    import paper_2603_15854_b200 as fs
    import synth
    from parity import check_flat, oracle_flat
    torch.cuda.set_device(0)
    fs.comm_init(fs.comm_unique_id(), 1, 0)
    wl = synth.make_workload("qwen25_7b", 40, V=7001, D=128)
    dev = {k: getattr(wl, k).cuda() for k in ("h", "W", "bias", "temperature", "mask")}
    for step in range(3):
        idx, score, logZ, ranks = fs.sample_tp(dev["h"], dev["W"], 0, wl.V, bias_shard=dev["bias"],
                                               temperature=dev["temperature"], mask=dev["mask"], seed=wl.seed,
                                               step=step, return_all=True, per_rank=True)
        ref_idx, ref_score = fs.sample(dev["h"], dev["W"], bias=dev["bias"], temperature=dev["temperature"],
                                       mask=dev["mask"], seed=wl.seed, step=step, return_score=True)
        torch.cuda.synchronize()
        assert torch.equal(idx, ref_idx)
        assert torch.equal(score.view(torch.int32), ref_score.view(torch.int32))
        assert torch.equal(ranks.idx[0], idx)
    _, flat = oracle_flat(wl, 2)
    check_flat(idx.cpu().numpy(), score.cpu().numpy(), flat)
    fs.comm_destroy()


def test_nccl_sample_tp_idx_only_skips_log_mass_and_matches():
    """fs_sample_tp without logZ / per-rank outputs runs the shard without the log-mass epilogue (one
    kernel, records written by the finalizing CTA): same idx as fs_sample on every step, for both
    stage-1 kernels (B = 1 single CTA, B = 40 / 300 CTA pairs; 300 = two batch chunks) and transforms."""
    import paper_2603_15854_b200 as fs
    import synth
    torch.cuda.set_device(0)
    fs.comm_init(fs.comm_unique_id(), 1, 0)
    for cfg, B, V, D in (("llama3_8b", 1, 20011, 256), ("qwen25_7b", 40, 7001, 128), ("llama3_8b", 300, 5003, 64)):
        wl = synth.make_workload(cfg, B, V=V, D=D)
        dev = {k: (getattr(wl, k).cuda() if getattr(wl, k) is not None else None)
               for k in ("h", "W", "bias", "temperature", "mask")}
        for step in range(3):
            idx = fs.sample_tp(dev["h"], dev["W"], 0, wl.V, bias_shard=dev["bias"], temperature=dev["temperature"],
                               mask=dev["mask"], seed=wl.seed, step=step)
            ref = fs.sample(dev["h"], dev["W"], bias=dev["bias"], temperature=dev["temperature"], mask=dev["mask"],
                            seed=wl.seed, step=step)
            torch.cuda.synchronize()
            assert torch.equal(idx, ref), (cfg, B, step)
    fs.comm_destroy()
