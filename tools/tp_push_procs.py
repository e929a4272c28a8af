"""Vocabulary-sharded step with the peer-memory push exchange (fs_sample_tp_push)
run by `world` processes that all sit on GPU 0 -- the only multi-process configuration a 1-GPU box
allows.  Each rank holds V/world rows of the 70B LM head, maps the others' exchange windows through
CUDA IPC, and times `steps` back-to-back idx-only steps (one kernel per rank: shard, push, wait,
combine).  The processes' kernels time-slice one GPU, so the step time here is NOT the multi-GPU
latency; it shows the protocol running end to end (every rank must agree with fs_sample, 0 timeouts).

    python tools/tp_push_procs.py [world] [steps] [B]    -> one JSON line
"""
import json
import os
import socket
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _worker(rank, world, port, B, steps, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import synth
        import paper_2603_15854_b200 as fs
        from paper_2603_15854_b200 import tp
        cfg = synth.CONFIGS["llama3_70b"]
        D, V = cfg["D"], cfg["V"]
        lo, hi = tp.shard_bounds(V, world, rank)
        dev = torch.device("cuda", 0)
        g = torch.Generator(device=dev)
        g.manual_seed(1234)
        h = torch.randn(B, D, device=dev, generator=g).to(torch.bfloat16)
        g.manual_seed(99 + rank)
        W = (torch.randn(hi - lo, D, device=dev, generator=g) * synth.W_STD).to(torch.bfloat16)
        tp.PushExchange(B_max=B)
        for s in range(3):
            fs.sample_tp_push(h, W, lo, V, seed=synth.SAMPLING_SEED, step=s)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for s in range(steps):
            idx = fs.sample_tp_push(h, W, lo, V, seed=synth.SAMPLING_SEED, step=100 + s)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        out = idx.cpu().tolist()
        timeouts = fs.query("comm_timeouts")
        dist.barrier()
        fs.comm_window_destroy()
        q.put((rank, wall, out, timeouts, None))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, None, None, None, repr(e)[:300]))


def main():
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    B = int(sys.argv[3]) if len(sys.argv) > 3 else 32
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    errs = [e for *_, e in res if e]
    line = {"world": world, "B": B, "steps": steps, "workload": "llama3_70b LM head, V/world rows per rank",
            "processes_on_one_gpu": True}
    if errs:
        line["error"] = errs[0]
    else:
        walls = [w for _, w, *_ in res]
        line["us_per_step_wall_max_over_ranks"] = round(1e6 * max(walls) / steps, 1)
        line["idx_identical_across_ranks"] = all(r[2] == res[0][2] for r in res)
        line["timeouts"] = sum(r[3] for r in res)
        line["note"] = ("ranks time-slice one GPU (no MPS): the step includes context switches between the "
                        "processes' kernels; not the NVLink latency")
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
