"""Vocabulary-sharded tensor-parallel FlashSampling (§4.2, Alg. A.4).

One process per GPU.  Rank k holds W rows [k V/n, (k+1) V/n) (Alg. A.4); every rank
runs the fused kernel on its shard (fs_sample_shard), the ranks exchange one 12-byte
summary (M, I, L) per row with a single all-gather over NCCL / NVLink ("all-gather
... or an equivalent reduction"), and every rank runs the outer selection
(fs_combine_summaries) so all ranks hold the identical global index.  Because the RNG is
keyed by global vocabulary ids and no logit's fp32 accumulation depends on the shard, the
result equals single-GPU fs_sample bit for bit.

The exchange is torch.distributed plumbing; all arithmetic runs in the library kernels.
transport="push" replaces the collective by the library's peer-memory
exchange: every rank stores its records into every peer's window (CUDA IPC; NVLink stores
between GPUs) and one kernel after stage 2 waits for the n records and combines them.  The
torch.distributed group is then used once, to all-gather the 64-byte window handles.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import Summaries, combine_summaries, comm_window_create, comm_window_open, sample_shard, sample_tp_push


def shard_bounds(V: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [k V/n, (k+1) V/n) of rank k (floor division; the last shard absorbs the rest)."""
    return rank * V // world, (rank + 1) * V // world


def gather_summaries(local: torch.Tensor, group=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather [B, 3] int32 summary records into [world, B, 3] (B*12 bytes per rank)."""
    world = dist.get_world_size(group)
    if out is None:
        out = torch.empty((world,) + tuple(local.shape), dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "gloo":
        dist.all_gather(list(out.unbind(0)), local.contiguous(), group=group)
    else:
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    return out


def sample_tp(h, W_shard, vocab_offset: int, V_total: int, *, group=None, bias_shard=None, temperature=None,
              mask=None, seed: int = 0, step: int = 0, return_all: bool = False, workspace=None):
    """Distributed FlashSampling step on this rank.  Returns idx [B] (identical on every rank),
    plus (score, logZ) if return_all.  `workspace` = (local Summaries, gathered tensor) to reuse."""
    local, gathered = workspace if workspace is not None else (None, None)
    local = sample_shard(h, W_shard, vocab_offset, V_total, bias_shard=bias_shard, temperature=temperature,
                         mask=mask, seed=seed, step=step, out=local)
    gathered = gather_summaries(local.raw, group=group, out=gathered)
    return combine_summaries(gathered, return_all=return_all)


class PushExchange:
    """Peer-memory exchange windows of a process group (one per rank, up to B_max rows).
    Creating it is collective: every rank all-gathers its window handle over `group`."""

    def __init__(self, B_max: int, group=None, device=None):
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        handle = comm_window_create(world, rank, B_max, device=device)
        handles = [None] * world
        dist.all_gather_object(handles, handle, group=group)
        comm_window_open(handles, device=device)
        self.world, self.rank, self.B_max = world, rank, B_max


def sample_tp_push_step(h, W_shard, vocab_offset: int, V_total: int, **kw):
    """One sharded step over an opened PushExchange (same arguments as sample_tp)."""
    return sample_tp_push(h, W_shard, vocab_offset, V_total, **kw)
