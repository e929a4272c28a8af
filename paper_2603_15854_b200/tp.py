"""Vocabulary-sharded tensor-parallel FlashSampling (§4.2, Alg. A.4).

One process per GPU.  Rank k holds W rows [k V/n, (k+1) V/n) (Alg. A.4); every rank
runs the fused kernel on its shard (fs_sample_shard), the ranks exchange one 12-byte
summary (M, I, L) per row with a single all-gather over NCCL / NVLink ("all-gather
... or an equivalent reduction"), and every rank runs the outer selection
(fs_combine_summaries) so all ranks hold the identical global index.  Because the RNG is
keyed by global vocabulary ids and no logit's fp32 accumulation depends on the shard, the
result equals single-GPU fs_sample bit for bit.

Three transports, all with the arithmetic in the library kernels:
  * "nccl"  (default on an NCCL process group): the library's own NCCL communicator
            (fs_comm_init, created once by NcclComm) and fs_sample_tp -- shard kernel, ncclAllGather
            of the B x 12-byte records and the combine, all enqueued by the library on the caller's
            stream.  torch.distributed only broadcasts the 128-byte NCCL unique id, once.
  * "torch" (default on gloo): fs_sample_shard, torch.distributed all-gather, fs_combine_summaries.
  * push    (PushExchange + sample_tp_push_step): the library's peer-memory exchange
            -- the shard kernel stores its records straight into every peer's window (CUDA IPC;
            NVLink stores between GPUs).  Idx only: the same kernel's finalizing CTA then waits for
            the n records and combines (one kernel per rank and step); with logZ one small
            PDL-chained kernel waits and combines.  The group is used once, to all-gather the 64-byte
            window handles.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import (Summaries, combine_summaries, comm_init, comm_unique_id, comm_window_create, comm_window_open,
               sample_shard, sample_tp_push)
from . import sample_tp as _sample_tp_lib


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


class NcclComm:
    """The library's NCCL communicator over the ranks of `group` (collective to create): rank 0
    draws the NCCL unique id, torch.distributed broadcasts the 128 bytes, every rank calls
    fs_comm_init on its device's context.  Afterwards sample_tp(transport="nccl") runs the whole
    exchange inside the library."""

    def __init__(self, group=None, device=None):
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.unique_id = broadcast_unique_id(group)
        comm_init(self.unique_id, self.world, self.rank, device=device)


def broadcast_unique_id(group=None) -> bytes:
    """Rank 0 of `group` draws an NCCL unique id (fs_comm_unique_id); every rank returns the same
    128 bytes (host plumbing of NcclComm, testable without a GPU)."""
    obj = [comm_unique_id() if dist.get_rank(group) == 0 else None]
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


def sample_tp(h, W_shard, vocab_offset: int, V_total: int, *, group=None, bias_shard=None, temperature=None,
              mask=None, seed: int = 0, step: int = 0, return_all: bool = False, workspace=None,
              transport: str | None = None, out=None):
    """Distributed FlashSampling step on this rank.  Returns idx [B] (identical on every rank),
    plus (score, logZ) if return_all.  transport "nccl" (needs an NcclComm on this device's
    context; default for an NCCL group) or "torch" (default otherwise).  `workspace` =
    (local Summaries, gathered tensor) to reuse on the "torch" transport."""
    if transport is None:
        transport = "nccl" if dist.get_backend(group) == "nccl" else "torch"
    if transport == "nccl":
        return _sample_tp_lib(h, W_shard, vocab_offset, V_total, bias_shard=bias_shard, temperature=temperature,
                              mask=mask, seed=seed, step=step, return_all=return_all, out=out)
    if transport != "torch":
        raise ValueError(f"unknown transport {transport!r}")
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
