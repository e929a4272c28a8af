"""World-size-2 CPU test (gloo) of the tensor-parallel exchange plumbing (paper_2603_15854_b200.tp):
each rank computes its vocabulary shard's 12-byte summaries (here with the oracle, since there is
no GPU), all-gathers them through tp.gather_summaries, and runs the outer selection; every rank
must hold the flat single-device sample (Alg. A.4 P:820-836 with max reuse)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _pack(M, I, L):
    raw = np.zeros((len(M), 3), np.int32)
    raw[:, 0] = np.asarray(M, np.float32).view(np.int32)
    raw[:, 1] = np.asarray(I, np.int32)
    raw[:, 2] = np.asarray(L, np.float32).view(np.int32)
    return torch.from_numpy(raw)


def _worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    from oracle import sampler
    from paper_2603_15854_b200 import tp
    wl = synth.make_workload("llama3_8b", 6, V=3001, D=64, with_transforms=True)
    a = {k: synth.as_numpy_exact(getattr(wl, k)) for k in ("h", "W", "bias", "temperature", "mask")}
    lo, hi = tp.shard_bounds(wl.V, world, rank)
    assert (lo, hi) == sampler.shard_bounds(wl.V, world)[rank]
    sc = sampler.scores(a["h"], a["W"][lo:hi], seed=wl.seed, step=4, bias=a["bias"][lo:hi],
                        temperature=a["temperature"], mask=a["mask"], vocab_offset=lo)
    gr = sampler.group_summaries(sc, hi - lo)
    local = _pack(gr.M[:, 0], gr.I[:, 0], gr.L[:, 0])
    gathered = tp.gather_summaries(local).numpy()
    assert gathered.shape == (world, 6, 3)
    M = gathered[:, :, 0].view(np.float32)
    I = gathered[:, :, 1]
    L = gathered[:, :, 2].view(np.float32)
    idx, best, logZ = sampler.combine_shard_summaries(M, I, L)
    flat = sampler.flat_sample(sampler.scores(a["h"], a["W"], seed=wl.seed, step=4, bias=a["bias"],
                                              temperature=a["temperature"], mask=a["mask"]))
    # NcclComm's host plumbing: rank 0's NCCL unique id reaches every rank unchanged (fs_comm_init
    # itself needs a GPU per rank)
    uid = tp.broadcast_unique_id()
    result_q.put((rank, idx.tolist(), flat.idx.tolist(), float(np.max(np.abs(logZ - flat.logZ))), uid))
    dist.destroy_process_group()


def test_tp_exchange_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, idx, flat_idx, lz_err, uid in res:
        assert idx == flat_idx
        assert lz_err < 1e-5          # fp32-rounded summaries
        assert len(uid) == 128
    assert res[0][1] == res[1][1]
    assert res[0][4] == res[1][4]
