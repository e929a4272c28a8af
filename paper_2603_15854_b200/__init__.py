"""FlashSampling on B200: fused LM-head projection + exact Gumbel-max sampling (arXiv 2603.15854).

Thin Python binding over the C ABI (include/flashsample.h, libflashsample.so).  Every step
of the sampling path runs in the library's sm_100a kernels; this module only validates
tensors, passes pointers and the current CUDA stream, and allocates outputs.

    import paper_2603_15854_b200 as fs
    idx = fs.sample(h, W, seed=..., step=...)                       # Alg. 2
    idx, logZ, groups = fs.sample_grouped(h, W, group_size=4096)    # §4.1, App. E
    summ = fs.sample_shard(h, W_shard, vocab_offset, V_total)       # Alg. A.4 rank-local half
    idx = fs.combine_summaries(gathered)                            # Alg. A.4 outer selection
"""
from __future__ import annotations

import ctypes
import dataclasses
import threading
import time

import torch

from . import _lib
from ._lib import FS_BF16, FS_F32, FlashSampleError

__all__ = ["sample", "sample_grouped", "sample_logits", "sample_shard", "combine_summaries", "merge_summaries",
           "random_bits", "gumbel_from_bits", "Summaries", "context", "set_option", "query",
           "FlashSampleError", "version", "sample_from_host", "comm_window_create", "comm_window_open",
           "comm_window_destroy", "sample_tp_push", "comm_unique_id", "comm_init", "comm_destroy", "sample_tp",
           "HostStepSampler"]

_ctx = {}            # (device, CUDA stream handle) -> fs_ctx handle
_opts = {}           # device -> {option: value}, applied to every context of that device
_ctx_lock = threading.Lock()


def version() -> str:
    return _lib.lib().fs_version().decode()


def _device_index(device) -> int:
    if device is None:
        return torch.cuda.current_device()
    if isinstance(device, torch.device):
        return device.index if device.index is not None else torch.cuda.current_device()
    return int(device)


def context(device: int | torch.device | None = None, stream=None) -> ctypes.c_void_p:
    """The library context (ctypes handle) for (device, stream), created on first use.
    A context owns one device workspace, so calls on it must be stream-ordered
    (include/flashsample.h): keying contexts by stream lets several streams -- or host threads
    on their own streams -- sample concurrently.  `stream` defaults to the device's current
    stream.  Options set through set_option() apply to every context of the device."""
    dev = _device_index(device)
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    key = (dev, int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream))
    with _ctx_lock:
        if key not in _ctx:
            h = ctypes.c_void_p()
            _lib.check(_lib.lib().fs_ctx_create(dev, ctypes.byref(h)), "fs_ctx_create")
            for name, value in _opts.get(dev, {}).items():
                _lib.check(_lib.lib().fs_ctx_set_option(h, name.encode(), int(value)), "fs_ctx_set_option")
            _ctx[key] = h
        return _ctx[key]


def set_option(name: str, value: int, device=None) -> None:
    """Set a library option (fs_ctx_set_option) on every context of the device, present and future."""
    dev = _device_index(device)
    context(dev)                         # make sure the current stream's context exists
    with _ctx_lock:
        _opts.setdefault(dev, {})[name] = int(value)
        handles = [h for (d, _), h in _ctx.items() if d == dev]
    for h in handles:
        _lib.check(_lib.lib().fs_ctx_set_option(h, name.encode(), int(value)), "fs_ctx_set_option")


def query(name: str, device=None) -> float:
    """fs_ctx_query on the context of the device's current stream."""
    out = ctypes.c_double()
    _lib.check(_lib.lib().fs_ctx_query(context(device), name.encode(), ctypes.byref(out)), "fs_ctx_query")
    return out.value


def _stream(t: torch.Tensor):
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _dtype_code(h: torch.Tensor, W: torch.Tensor) -> int:
    if h.dtype != W.dtype:
        raise TypeError("h and W must have the same dtype")
    if h.dtype == torch.bfloat16:
        return FS_BF16
    if h.dtype == torch.float32:
        return FS_F32
    raise TypeError(f"unsupported dtype {h.dtype} (bf16 or fp32)")


def _check_inputs(h, W, bias, temperature, mask, V_total=None):
    for name, t in (("h", h), ("W", W)):
        if not t.is_cuda or not t.is_contiguous() or t.dim() != 2:
            raise ValueError(f"{name} must be a contiguous 2-D CUDA tensor")
    B, D = h.shape
    V, D2 = W.shape
    if D != D2:
        raise ValueError("h and W disagree on D")
    V_total = V if V_total is None else V_total
    if bias is not None and (bias.dtype != torch.float32 or bias.numel() != V or not bias.is_contiguous()):
        raise ValueError("bias must be a contiguous fp32 [V] tensor")
    if temperature is not None and (temperature.dtype != torch.float32 or temperature.numel() != B
                                    or not temperature.is_contiguous()):
        raise ValueError("temperature must be a contiguous fp32 [B] tensor")
    if mask is not None and (mask.dtype != torch.int32 or tuple(mask.shape) != (B, (V_total + 31) // 32)
                             or not mask.is_contiguous()):
        raise ValueError("mask must be a contiguous int32 [B, ceil(V/32)] bit tensor")
    return B, D, V


def _u64(t, B, name, dev):
    if t is None:
        return None
    if t.dtype not in (torch.int64, torch.uint64) or t.numel() != B or not t.is_contiguous() or t.device != dev:
        raise ValueError(f"{name} must be a contiguous int64/uint64 [B] tensor on the sampling device")
    return t


def sample(h, W, *, bias=None, temperature=None, mask=None, seed: int = 0, step: int = 0,
           seeds=None, steps=None, top_k: int = 0, top_p: float = 1.0, return_score: bool = False,
           return_logprob: bool = False, out=None):
    """Fused LM-head + exact Gumbel-max sample per row.  Returns int32 [B]; with return_score
    also the winning perturbed scores; with return_logprob also (logZ, log p(idx)).
    seeds / steps: optional [B] int64 per-request streams (batch-position invariant, reading R18);
    temperature[b] == 0 samples row b greedily.  top_k (1..1024) / top_p: exact top-k then
    nucleus sampling through the LM head (reading R19; logZ / log-prob are those of the kept set)."""
    B, D, V = _check_inputs(h, W, bias, temperature, mask)
    idx = out if out is not None else torch.empty(B, dtype=torch.int32, device=h.device)
    score = torch.empty(B, dtype=torch.float32, device=h.device) if return_score else None
    seeds = _u64(seeds, B, "seeds", h.device)
    steps = _u64(steps, B, "steps", h.device)
    if seeds is None and steps is None and not return_logprob and not top_k and top_p >= 1.0:
        _lib.check(_lib.lib().fs_sample(context(h.device), _dtype_code(h, W), _ptr(h), _ptr(W), _ptr(bias),
                                        _ptr(temperature), _ptr(mask), seed & (2**64 - 1), step & (2**64 - 1),
                                        B, D, V, _ptr(idx), _ptr(score), _stream(h)), "fs_sample")
        return (idx, score) if return_score else idx
    logZ = torch.empty(B, dtype=torch.float32, device=h.device) if return_logprob else None
    logprob = torch.empty(B, dtype=torch.float32, device=h.device) if return_logprob else None
    args = _lib.SampleArgs(_ptr(bias), _ptr(temperature), _ptr(mask), seed & (2**64 - 1), step & (2**64 - 1),
                           _ptr(seeds), _ptr(steps), 0, _ptr(idx), _ptr(score), _ptr(logZ), _ptr(logprob), None,
                           int(top_k), float(top_p))
    _lib.check(_lib.lib().fs_sample_ex(context(h.device), _dtype_code(h, W), _ptr(h), _ptr(W), B, D, V,
                                       ctypes.byref(args), _stream(h)), "fs_sample_ex")
    res = (idx,) + ((score,) if return_score else ()) + ((logZ, logprob) if return_logprob else ())
    return res if len(res) > 1 else idx


def comm_window_create(world: int, rank: int, B_max: int, device=None) -> bytes:
    """Allocate this rank's peer-exchange window; returns its 64-byte IPC handle,
    to be all-gathered by the caller (any host transport) and passed to comm_window_open."""
    hd = _lib.IpcHandle()
    _lib.check(_lib.lib().fs_comm_window_create(context(device), int(world), int(rank), int(B_max), ctypes.byref(hd)),
               "fs_comm_window_create")
    return bytes(hd.bytes)


def comm_window_open(handles, device=None) -> None:
    """Map the peers' windows from the gathered handles (list of `world` 64-byte strings)."""
    arr = (_lib.IpcHandle * len(handles))()
    for i, hb in enumerate(handles):
        ctypes.memmove(arr[i].bytes, bytes(hb), 64)
    _lib.check(_lib.lib().fs_comm_window_open(context(device), arr), "fs_comm_window_open")


def comm_window_destroy(device=None) -> None:
    _lib.check(_lib.lib().fs_comm_window_destroy(context(device)), "fs_comm_window_destroy")


def sample_tp_push(h, W_shard, vocab_offset: int, V_total: int, *, bias_shard=None, temperature=None, mask=None,
                   seed: int = 0, step: int = 0, return_all: bool = False):
    """Vocabulary-sharded step with the peer-memory exchange (fs_sample_tp_push): shard summary,
    push to every peer window, wait, outer selection.  idx [B] identical on all ranks."""
    B, D, V_local = _check_inputs(h, W_shard, bias_shard, temperature, mask, V_total=V_total)
    idx = torch.empty(B, dtype=torch.int32, device=h.device)
    score = torch.empty(B, dtype=torch.float32, device=h.device) if return_all else None
    logZ = torch.empty(B, dtype=torch.float32, device=h.device) if return_all else None
    _lib.check(_lib.lib().fs_sample_tp_push(
        context(h.device), _dtype_code(h, W_shard), _ptr(h), _ptr(W_shard), _ptr(bias_shard), _ptr(temperature),
        _ptr(mask), seed & (2**64 - 1), step & (2**64 - 1), B, D, V_local, int(vocab_offset), int(V_total),
        _ptr(idx), _ptr(score), _ptr(logZ), _stream(h)), "fs_sample_tp_push")
    return (idx, score, logZ) if return_all else idx


def comm_unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) for fs_comm_init; create it on one rank and broadcast it."""
    buf = ctypes.create_string_buffer(128)
    _lib.check(_lib.lib().fs_comm_unique_id(buf), "fs_comm_unique_id")
    return buf.raw


def comm_init(unique_id: bytes, world: int, rank: int, device=None) -> None:
    """Create the library's NCCL communicator on this rank's context (collective; fs_comm_init)."""
    if len(unique_id) != 128:
        raise ValueError("unique_id must be the 128 bytes of comm_unique_id()")
    buf = ctypes.create_string_buffer(bytes(unique_id), 128)
    _lib.check(_lib.lib().fs_comm_init(context(device), buf, int(world), int(rank)), "fs_comm_init")


def comm_destroy(device=None) -> None:
    _lib.check(_lib.lib().fs_comm_destroy(context(device)), "fs_comm_destroy")


def sample_tp(h, W_shard, vocab_offset: int, V_total: int, *, bias_shard=None, temperature=None, mask=None,
              seed: int = 0, step: int = 0, return_all: bool = False, per_rank: bool = False, out=None):
    """One vocabulary-sharded step through the library's NCCL path (fs_sample_tp): shard summaries,
    ncclAllGather of B x 12 bytes, outer selection.  idx [B] identical on every rank.
    Returns idx, or (idx, score, logZ[, per-rank Summaries [world, B]]) with return_all."""
    B, D, V_local = _check_inputs(h, W_shard, bias_shard, temperature, mask, V_total=V_total)
    idx = out if out is not None else torch.empty(B, dtype=torch.int32, device=h.device)
    score = torch.empty(B, dtype=torch.float32, device=h.device) if return_all else None
    logZ = torch.empty(B, dtype=torch.float32, device=h.device) if return_all else None
    ranks = None
    if per_rank:
        ranks = Summaries.empty(int(query("nccl_world", h.device)), B, device=h.device)
    _lib.check(_lib.lib().fs_sample_tp(
        context(h.device), _dtype_code(h, W_shard), _ptr(h), _ptr(W_shard), _ptr(bias_shard), _ptr(temperature),
        _ptr(mask), seed & (2**64 - 1), step & (2**64 - 1), B, D, V_local, int(vocab_offset), int(V_total),
        _ptr(idx), _ptr(score), _ptr(logZ), _ptr(ranks.raw) if ranks is not None else None, _stream(h)),
        "fs_sample_tp")
    if not return_all:
        return idx
    return (idx, score, logZ) + ((ranks,) if per_rank else ())


@dataclasses.dataclass
class Summaries:
    """fs_summary records {max_score f32, idx i32, log_mass f32} stored as int32 [..., 3]."""
    raw: torch.Tensor

    @property
    def max_score(self):
        return self.raw[..., 0].view(torch.float32)

    @property
    def idx(self):
        return self.raw[..., 1]

    @property
    def log_mass(self):
        return self.raw[..., 2].view(torch.float32)

    @staticmethod
    def empty(*shape, device):
        return Summaries(torch.empty(*shape, 3, dtype=torch.int32, device=device))


def sample_grouped(h, W, *, group_size: int, bias=None, temperature=None, mask=None, seed: int = 0,
                   step: int = 0, return_groups: bool = True, return_logprob: bool = False):
    """Grouped FlashSampling (fs_sample_grouped).  Returns (idx [B] int32, score [B] fp32,
    logZ [B] fp32, Summaries [B, ceil(V/g)] or None) [+ logprob [B] fp32 if return_logprob]."""
    B, D, V = _check_inputs(h, W, bias, temperature, mask)
    n_groups = (V + group_size - 1) // group_size
    idx = torch.empty(B, dtype=torch.int32, device=h.device)
    score = torch.empty(B, dtype=torch.float32, device=h.device)
    logZ = torch.empty(B, dtype=torch.float32, device=h.device)
    logprob = torch.empty(B, dtype=torch.float32, device=h.device) if return_logprob else None
    groups = Summaries.empty(B, n_groups, device=h.device) if return_groups else None
    _lib.check(_lib.lib().fs_sample_grouped(
        context(h.device), _dtype_code(h, W), _ptr(h), _ptr(W), _ptr(bias), _ptr(temperature), _ptr(mask),
        seed & (2**64 - 1), step & (2**64 - 1), B, D, V, group_size, _ptr(idx), _ptr(score), _ptr(logZ),
        _ptr(logprob), _ptr(groups.raw) if groups else None, _stream(h)), "fs_sample_grouped")
    if return_logprob:
        return idx, score, logZ, groups, logprob
    return idx, score, logZ, groups


def sample_logits(logits, *, bias=None, temperature=None, mask=None, seed: int = 0, step: int = 0,
                  seeds=None, steps=None, top_k: int = 0, top_p: float = 1.0, return_all: bool = False,
                  return_score: bool = False):
    """Standalone Gumbel-max over materialised logits [B, V] (bf16 or fp32, row stride may exceed V)
    (fs_sample_logits[_ex]).  top_k (1..1024) / top_p: exact top-k then nucleus sampling (R19).
    Returns idx [B]; (idx, score) if return_score; (idx, score, logZ, logprob) if return_all."""
    if not logits.is_cuda or logits.dim() != 2 or logits.stride(1) != 1:
        raise ValueError("logits must be a 2-D CUDA tensor with unit column stride")
    B, V = logits.shape
    if bias is not None and (bias.dtype != torch.float32 or bias.numel() != V):
        raise ValueError("bias must be fp32 [V]")
    if temperature is not None and (temperature.dtype != torch.float32 or temperature.numel() != B):
        raise ValueError("temperature must be fp32 [B]")
    if mask is not None and (mask.dtype != torch.int32 or tuple(mask.shape) != (B, (V + 31) // 32)):
        raise ValueError("mask must be int32 [B, ceil(V/32)]")
    code = FS_BF16 if logits.dtype == torch.bfloat16 else FS_F32 if logits.dtype == torch.float32 else None
    if code is None:
        raise TypeError("logits must be bf16 or fp32")
    dev = logits.device
    seeds = _u64(seeds, B, "seeds", dev)
    steps = _u64(steps, B, "steps", dev)
    idx = torch.empty(B, dtype=torch.int32, device=dev)
    score = torch.empty(B, dtype=torch.float32, device=dev) if (return_all or return_score) else None
    logZ = torch.empty(B, dtype=torch.float32, device=dev) if return_all else None
    logprob = torch.empty(B, dtype=torch.float32, device=dev) if return_all else None
    args = _lib.SampleArgs(_ptr(bias), _ptr(temperature), _ptr(mask), seed & (2**64 - 1), step & (2**64 - 1),
                           _ptr(seeds), _ptr(steps), 0, _ptr(idx), _ptr(score), _ptr(logZ), _ptr(logprob), None,
                           int(top_k), float(top_p))
    _lib.check(_lib.lib().fs_sample_logits_ex(context(dev), code, _ptr(logits), logits.stride(0), B, V,
                                              ctypes.byref(args), _stream(logits)), "fs_sample_logits_ex")
    if return_all:
        return idx, score, logZ, logprob
    return (idx, score) if return_score else idx


def sample_shard(h, W_shard, vocab_offset: int, V_total: int, *, bias_shard=None, temperature=None,
                 mask=None, seed: int = 0, step: int = 0, out: Summaries | None = None) -> Summaries:
    """Rank-local half of distributed FlashSampling (fs_sample_shard): this shard's (M, I, L)."""
    B, D, V = _check_inputs(h, W_shard, bias_shard, temperature, mask, V_total=V_total)
    summ = out if out is not None else Summaries.empty(B, device=h.device)
    _lib.check(_lib.lib().fs_sample_shard(
        context(h.device), _dtype_code(h, W_shard), _ptr(h), _ptr(W_shard), _ptr(bias_shard), _ptr(temperature),
        _ptr(mask), seed & (2**64 - 1), step & (2**64 - 1), B, D, V, int(vocab_offset), int(V_total),
        _ptr(summ.raw), _stream(h)), "fs_sample_shard")
    return summ


def combine_summaries(gathered: Summaries | torch.Tensor, *, return_all: bool = False):
    """Outer selection over gathered summaries [n, B] (fs_combine_summaries)."""
    raw = gathered.raw if isinstance(gathered, Summaries) else gathered
    n, B = raw.shape[0], raw.shape[1]
    raw = raw.contiguous()
    idx = torch.empty(B, dtype=torch.int32, device=raw.device)
    score = torch.empty(B, dtype=torch.float32, device=raw.device)
    logZ = torch.empty(B, dtype=torch.float32, device=raw.device)
    _lib.check(_lib.lib().fs_combine_summaries(_ptr(raw), n, B, _ptr(idx), _ptr(score), _ptr(logZ),
                                               _stream(raw)), "fs_combine_summaries")
    return (idx, score, logZ) if return_all else idx


def merge_summaries(a: Summaries, b: Summaries) -> Summaries:
    """Online binary merge of two summary arrays of disjoint vocabularies (fs_merge_summaries)."""
    out = Summaries(torch.empty_like(a.raw))
    _lib.check(_lib.lib().fs_merge_summaries(_ptr(a.raw.contiguous()), _ptr(b.raw.contiguous()), _ptr(out.raw),
                                             a.raw.numel() // 3, _stream(a.raw)), "fs_merge_summaries")
    return out


def random_bits(seed: int, step: int, b: torch.Tensor, v: torch.Tensor, tag: int = 0) -> torch.Tensor:
    """Device Philox draws r for positions (b[i], v[i]) (diagnostic, fs_random_bits)."""
    b = b.to(torch.int32).contiguous()
    v = v.to(torch.int64).contiguous()
    r = torch.empty(b.numel(), dtype=torch.int32, device=b.device)
    _lib.check(_lib.lib().fs_random_bits(seed & (2**64 - 1), step & (2**64 - 1), tag, _ptr(b), _ptr(v), _ptr(r),
                                         b.numel(), _stream(b)), "fs_random_bits")
    return r


def read_probe(buf: torch.Tensor, sink: torch.Tensor, grid: int = 0) -> None:
    """Read-only HBM roofline probe (fs_read_probe): stream the bytes of the device tensor `buf` once;
    XOR of the first 8 bytes of every 16 KB chunk of each CTA slice into sink (int64 [1])."""
    if not buf.is_cuda or not buf.is_contiguous() or sink.dtype != torch.int64 or not sink.is_cuda:
        raise ValueError("buf: contiguous CUDA tensor; sink: CUDA int64 tensor")
    _lib.check(_lib.lib().fs_read_probe(_ptr(buf), buf.numel() * buf.element_size(), _ptr(sink), int(grid),
                                        _stream(buf)), "fs_read_probe")


def gumbel_from_bits(r: torch.Tensor) -> torch.Tensor:
    """Device fp32 G32(r) (diagnostic, fs_gumbel_from_bits).  r: int32 tensor of bit patterns."""
    r = r.contiguous()
    g = torch.empty(r.shape, dtype=torch.float32, device=r.device)
    _lib.check(_lib.lib().fs_gumbel_from_bits(_ptr(r), _ptr(g), r.numel(), _stream(r)), "fs_gumbel_from_bits")
    return g


def copy_async(dst, src):
    """fs_copy_async: kernel copy of `src` (pinned host or device tensor) into the device tensor
    `dst` on the current stream (PDL-chained with fs_sample when option pdl_w is set)."""
    if not dst.is_cuda or not dst.is_contiguous() or not src.is_contiguous():
        raise ValueError("copy_async: dst must be a contiguous device tensor, src contiguous")
    if src.device.type == "cpu" and not src.is_pinned():
        raise ValueError("copy_async: a host src must be pinned")
    nbytes = src.numel() * src.element_size()
    if dst.numel() * dst.element_size() != nbytes:
        raise ValueError("copy_async: size mismatch")
    _lib.check(_lib.lib().fs_copy_async(context(dst.device), _ptr(dst), _ptr(src), nbytes,
                                        _stream(dst)), "fs_copy_async")


def sample_from_host(h_host, W, *, temperature_host=None, mask_host=None, bias=None, seed=0, step=0,
                     h_dev=None, t_dev=None, m_dev=None, idx_dev=None, idx_host=None):
    """End-to-end call a serving loop makes: copy this step's inputs from (pinned) host memory,
    sample on the device, copy the sampled ids back.  Device staging buffers may be passed in
    to avoid allocation.  Returns the host int32 [B] tensor.
    With pinned host tensors the inputs are staged by fs_copy_async (a kernel, PDL-chained with
    the sampling kernel) and the ids are written by the sampling kernel straight into the pinned
    idx_host (no copy-engine round trips); otherwise torch copies are used."""
    dev = W.device
    pinned = h_host.is_pinned() and (temperature_host is None or temperature_host.is_pinned()) and \
        (mask_host is None or mask_host.is_pinned()) and (idx_host is None or idx_host.is_pinned())
    if pinned and mask_host is None and h_host.dtype == torch.bfloat16:
        # fs_sample_staged: the sampling kernel stages h itself (one kernel per step); the tiny
        # temperature vector is read by the kernel straight from pinned host memory
        h_dev = h_dev if h_dev is not None else torch.empty_like(h_host, device=dev)
        idx_host = idx_host if idx_host is not None else torch.empty(h_host.shape[0], dtype=torch.int32,
                                                                     pin_memory=True)
        B, D = h_host.shape
        V = W.shape[0]
        if temperature_host is not None and (temperature_host.dtype != torch.float32 or temperature_host.numel() != B):
            raise ValueError("temperature must be fp32 [B]")
        if bias is not None and (bias.dtype != torch.float32 or bias.numel() != V or not bias.is_cuda):
            raise ValueError("bias must be a device fp32 [V] tensor")
        _lib.check(_lib.lib().fs_sample_staged(context(dev), FS_BF16, _ptr(h_host), _ptr(h_dev), _ptr(W), _ptr(bias),
                                               _ptr(temperature_host), None, seed & (2**64 - 1), step & (2**64 - 1),
                                               B, D, V, _ptr(idx_host), None, _stream(W)), "fs_sample_staged")
        return idx_host
    if pinned:
        h_dev = h_dev if h_dev is not None else torch.empty_like(h_host, device=dev)
        copy_async(h_dev, h_host)
        if temperature_host is not None:
            t_dev = t_dev if t_dev is not None else torch.empty_like(temperature_host, device=dev)
            copy_async(t_dev, temperature_host)
        if mask_host is not None:
            m_dev = m_dev if m_dev is not None else torch.empty_like(mask_host, device=dev)
            copy_async(m_dev, mask_host)
        idx_host = idx_host if idx_host is not None else torch.empty(h_host.shape[0], dtype=torch.int32,
                                                                     pin_memory=True)
        sample(h_dev, W, bias=bias, temperature=t_dev if temperature_host is not None else None,
               mask=m_dev if mask_host is not None else None, seed=seed, step=step, out=idx_host)
        return idx_host
    h_dev = h_dev if h_dev is not None else torch.empty_like(h_host, device=dev)
    h_dev.copy_(h_host, non_blocking=True)
    if temperature_host is not None:
        t_dev = t_dev if t_dev is not None else torch.empty_like(temperature_host, device=dev)
        t_dev.copy_(temperature_host, non_blocking=True)
    if mask_host is not None:
        m_dev = m_dev if m_dev is not None else torch.empty_like(mask_host, device=dev)
        m_dev.copy_(mask_host, non_blocking=True)
    idx_dev = sample(h_dev, W, bias=bias, temperature=t_dev if temperature_host is not None else None,
                     mask=m_dev if mask_host is not None else None, seed=seed, step=step, out=idx_dev)
    idx_host = idx_host if idx_host is not None else torch.empty(idx_dev.shape, dtype=torch.int32, pin_memory=True)
    idx_host.copy_(idx_dev, non_blocking=True)
    return idx_host


class HostStepSampler:
    """A serving loop's per-step call, prepared once: the end-to-end step of `sample_from_host`
    (fs_sample_staged: the sampling kernel stages this step's h from the pinned host buffer itself
    and stores the ids into the pinned host idx buffer) with every argument validated and marshalled
    at construction, so a step costs one ctypes call.  The caller rewrites `h_host` (pinned, bf16
    [B, D]) in place between steps and reads `idx_host` after `wait()`.
        s = HostStepSampler(h_host, W, seed=...)
        for t in ...: s(step=t); s.wait(); tok = s.idx_host
    """
    def __init__(self, h_host, W, *, bias=None, temperature_host=None, seed: int = 0, h_dev=None, idx_host=None):
        if h_host.dtype != torch.bfloat16 or h_host.dim() != 2 or not h_host.is_pinned() or not h_host.is_contiguous():
            raise ValueError("h_host must be a contiguous pinned bf16 [B, D] tensor")
        if W.dtype != torch.bfloat16 or not W.is_cuda or not W.is_contiguous() or W.shape[1] != h_host.shape[1]:
            raise ValueError("W must be a contiguous bf16 [V, D] CUDA tensor with D = h_host.shape[1]")
        B, D = h_host.shape
        V = W.shape[0]
        if temperature_host is not None and (temperature_host.dtype != torch.float32 or temperature_host.numel() != B
                                             or not temperature_host.is_pinned()):
            raise ValueError("temperature_host must be a pinned fp32 [B] tensor")
        if bias is not None and (bias.dtype != torch.float32 or bias.numel() != V or not bias.is_cuda):
            raise ValueError("bias must be a device fp32 [V] tensor")
        self.h_host, self.W, self.bias, self.temperature_host = h_host, W, bias, temperature_host
        self.h_dev = h_dev if h_dev is not None else torch.empty_like(h_host, device=W.device)
        self.idx_host = idx_host if idx_host is not None else torch.empty(B, dtype=torch.int32, pin_memory=True)
        self.stream = torch.cuda.current_stream(W.device)
        self._fn = _lib.lib().fs_sample_staged
        # a context of its own: its completion flag (option "done_flag") is set only by this loop's calls
        self._ctx = ctypes.c_void_p()
        _lib.check(_lib.lib().fs_ctx_create(_device_index(W.device), ctypes.byref(self._ctx)), "fs_ctx_create")
        with _ctx_lock:
            opts = dict(_opts.get(_device_index(W.device), {}))
        for name, value in opts.items():
            _lib.check(_lib.lib().fs_ctx_set_option(self._ctx, name.encode(), int(value)), "fs_ctx_set_option")
        self.done = torch.zeros(1, dtype=torch.int64, pin_memory=True)
        self._done_np = self.done.numpy()
        _lib.check(_lib.lib().fs_ctx_set_option(self._ctx, b"done_flag", self.done.data_ptr()), "fs_ctx_set_option")
        self._head = (self._ctx, FS_BF16, _ptr(h_host), _ptr(self.h_dev), _ptr(W), _ptr(bias),
                      _ptr(temperature_host), None)
        self._seed = seed & (2**64 - 1)
        self._tail = (B, D, V, _ptr(self.idx_host), None, ctypes.c_void_p(self.stream.cuda_stream))

    def set_option(self, name: str, value: int) -> None:
        """fs_ctx_set_option on this sampler's own context."""
        _lib.check(_lib.lib().fs_ctx_set_option(self._ctx, name.encode(), int(value)), "fs_ctx_set_option")

    def __call__(self, step: int):
        self._done_np[0] = 0
        st = self._fn(*self._head, self._seed, step & (2**64 - 1), *self._tail)
        if st:
            _lib.check(st, "fs_sample_staged")
        return self.idx_host

    def wait(self, timeout_s: float = 10.0):
        """Spin on the pinned completion flag the finalizing CTA sets after the ids (no stream sync);
        falls back to synchronising the stream after `timeout_s`."""
        f = self._done_np
        if f[0]:
            return self.idx_host
        t_end = None
        n = 0
        while not f[0]:
            n += 1
            if n & 0xFFFF == 0:
                t_end = t_end or time.perf_counter() + timeout_s
                if time.perf_counter() > t_end:
                    self.stream.synchronize()
                    if not f[0]:
                        raise FlashSampleError(_lib.FS_ERR_CUDA, "HostStepSampler.wait", "completion flag never set")
        return self.idx_host

    def __del__(self):
        try:
            if getattr(self, "_ctx", None):
                self.stream.synchronize()
                _lib.lib().fs_ctx_destroy(self._ctx)
                self._ctx = None
        except Exception:
            pass
