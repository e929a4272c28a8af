"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no GEMM, no transform, no RNG of the
sampler, no Gumbel, no argmax).  It only draws the *inputs* of a sampling step --
hidden states h, LM-head weights W, optional bias / temperature / vocabulary mask --
with the shapes and value distributions of the paper's workloads (DESIGN.md
"Input recipe").  Both sides (oracle/ and the CUDA product) consume
the same arrays: the oracle reads the exact bf16 bit patterns, the product receives
the same tensors on the device.

Workload shapes (BASELINE.json `configs`):
  tiny        B=4,   D=64,   V=1000    fp32   (oracle check)
  llama3_8b   D=4096, V=128256  bf16  (headline; §5.1 decode regime)
  qwen25_7b   D=3584, V=152064  bf16  tau=0.7 + bias + 25% mask
  gemma3_27b  D=5376, V=262208  bf16  grouped variant (g=4096, 65 groups)
  llama3_70b  D=8192, V=128256  bf16  vocab-sharded TP
  paper_d4096 D=4096, V=151936  bf16  the paper's Table 3 workload (context for its ratios)
"""
from __future__ import annotations

import dataclasses
import numpy as np
import torch

CONFIGS = {
    "tiny": dict(D=64, V=1000, dtype="f32", config_id=0),
    "llama3_8b": dict(D=4096, V=128256, dtype="bf16", config_id=1),
    "qwen25_7b": dict(D=3584, V=152064, dtype="bf16", config_id=2,
                      temperature=0.7, bias_std=0.5, mask_ban_frac=0.25),
    "gemma3_27b": dict(D=5376, V=262208, dtype="bf16", config_id=3, group_size=4096),
    "llama3_70b": dict(D=8192, V=128256, dtype="bf16", config_id=4),
    # the paper's own B200 workload (§5.1, Table 3): Qwen3-8B-like LM head
    "paper_d4096": dict(D=4096, V=151936, dtype="bf16", config_id=5),
}

# Sampling seed used by every default workload.
SAMPLING_SEED = 0x243F6A8885A308D3
W_STD = 0.02          # typical LLM init scale for the LM head
INPUT_SEED_BASE = 0x5EED


@dataclasses.dataclass
class Workload:
    """One sampling step's inputs.  Tensors live on `device` (CPU by default)."""
    name: str
    B: int
    D: int
    V: int
    dtype: str                      # "bf16" or "f32": storage/arithmetic type of h and W
    h: torch.Tensor                 # [B, D]
    W: torch.Tensor                 # [V, D] row-major (nn.Linear weight layout)
    bias: torch.Tensor | None       # [V] fp32
    temperature: torch.Tensor | None  # [B] fp32
    mask: torch.Tensor | None       # [B, ceil(V/32)] int32 words; bit v%32 of word v/32: 1 = allowed
    seed: int = SAMPLING_SEED
    group_size: int | None = None

    @property
    def mask_words(self) -> int:
        return (self.V + 31) // 32


def _gen(seed: int, device="cpu") -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def make_workload(name: str, B: int, *, device="cpu", seed_offset: int = 0,
                  pattern: str = "default", V: int | None = None, D: int | None = None,
                  with_transforms: bool | None = None) -> Workload:
    """Draw the seeded synthetic inputs of configuration `name` at batch size B.

    pattern (parity-only variants):
      default    h~N(0,1), W~N(0,0.02^2) (fp32 tiny: W~N(0,1/D) so logits ~ N(0,1))
      peaked     W std 0.2 (logit std ~13: low-entropy rows)
      duplicate  W rows come in identical pairs (2j, 2j+1)
      edge       row 0 fully masked, row 1 has a single allowed token, per-row tau~U(0.5,1.5)
    """
    cfg = dict(CONFIGS[name])
    D = D or cfg["D"]
    V = V or cfg["V"]
    seed = INPUT_SEED_BASE + cfg["config_id"] + 7919 * seed_offset
    g = _gen(seed, device)
    kw = dict(device=device, generator=g)
    if cfg["dtype"] == "f32":
        h = torch.randn(B, D, dtype=torch.float32, **kw)
        W = torch.randn(V, D, dtype=torch.float32, **kw) * (1.0 / np.sqrt(D))
    else:
        h = torch.randn(B, D, dtype=torch.float32, **kw).to(torch.bfloat16)
        std = 0.2 if pattern == "peaked" else W_STD
        W = torch.empty(V, D, dtype=torch.bfloat16, device=device)
        # fill in row chunks to bound the fp32 temporary
        step = max(1, (1 << 26) // D)
        for r0 in range(0, V, step):
            r1 = min(V, r0 + step)
            W[r0:r1] = (torch.randn(r1 - r0, D, dtype=torch.float32, **kw) * std).to(torch.bfloat16)
    if pattern == "duplicate":
        W[1::2] = W[0:(V // 2) * 2:2][: W[1::2].shape[0]]

    transforms = with_transforms if with_transforms is not None else ("temperature" in cfg)
    bias = temperature = mask = None
    nw = (V + 31) // 32
    if transforms:
        bias = torch.randn(V, dtype=torch.float32, **kw) * cfg.get("bias_std", 0.5)
        temperature = torch.full((B,), cfg.get("temperature", 0.7), dtype=torch.float32, device=device)
        ban = torch.rand(B, V, **kw) < cfg.get("mask_ban_frac", 0.25)
        mask = pack_allowed_bits(~ban)
    if pattern == "edge":
        if temperature is None:
            temperature = torch.ones(B, dtype=torch.float32, device=device)
        temperature = 0.5 + torch.rand(B, **kw)
        allowed = unpack_allowed_bits(mask, V) if mask is not None else torch.ones(B, V, dtype=torch.bool, device=device)
        allowed[0, :] = False                      # row with no finite logit -> idx -1
        if B > 1:
            allowed[1, :] = False
            allowed[1, (V * 5) // 7] = True        # row with a single allowed token
        mask = pack_allowed_bits(allowed)
    return Workload(name=name, B=B, D=D, V=V, dtype=cfg["dtype"], h=h, W=W, bias=bias,
                    temperature=temperature, mask=mask, group_size=cfg.get("group_size"))


def pack_allowed_bits(allowed: torch.Tensor) -> torch.Tensor:
    """[B, V] bool -> [B, ceil(V/32)] int32 words, bit v%32 of word v/32 set iff allowed."""
    B, V = allowed.shape
    nw = (V + 31) // 32
    pad = torch.zeros(B, nw * 32, dtype=torch.int64, device=allowed.device)
    pad[:, :V] = allowed.to(torch.int64)
    bits = pad.view(B, nw, 32) << torch.arange(32, device=allowed.device, dtype=torch.int64)
    words = bits.sum(dim=2)                       # < 2^32
    words = torch.where(words >= 2**31, words - 2**32, words)
    return words.to(torch.int32)


def unpack_allowed_bits(words: torch.Tensor, V: int) -> torch.Tensor:
    B, nw = words.shape
    w = words.to(torch.int64) & 0xFFFFFFFF
    bits = (w.unsqueeze(2) >> torch.arange(32, device=words.device, dtype=torch.int64)) & 1
    return bits.view(B, nw * 32)[:, :V].bool()


def bf16_bits(t: torch.Tensor) -> np.ndarray:
    """Exact bf16 bit patterns (uint16) of a bf16 tensor, as numpy (for the oracle)."""
    assert t.dtype == torch.bfloat16
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def as_numpy_exact(t: torch.Tensor | None):
    """Host numpy view carrying the exact stored values: uint16 bf16 bits, or fp32, or uint32 words."""
    if t is None:
        return None
    if t.dtype == torch.bfloat16:
        return bf16_bits(t)
    if t.dtype == torch.int32:
        return t.detach().cpu().numpy().view(np.uint32)
    return t.detach().cpu().numpy()
