"""§4.7 cost model, test infrastructure only.

  I_mat(B)   = B V D / (V D + B D + 2 B V)     FLOP/byte, BF16 materialised lower bound
  I_fused(B) = B V / (V + B)                   FLOP/byte, fused
  extra      = 4 B V / (2 V D) = 2 B / D       logits write+reread vs W read
  round trip = 4 B V bytes
"""
from __future__ import annotations


def intensity_materialized(B, V, D) -> float:
    return B * V * D / (V * D + B * D + 2 * B * V)


def intensity_fused(B, V, D=None) -> float:
    return B * V / (V + B)


def extra_traffic_fraction(B, D) -> float:
    return 2.0 * B / D


def logits_round_trip_bytes(B, V) -> int:
    return 4 * B * V


def seconds_at(bytes_, bandwidth_Bps) -> float:
    return bytes_ / bandwidth_Bps


def ops_per_byte(peak_flops, bandwidth_Bps) -> float:
    """Table 2 ops:byte = peak dense FLOP/s / HBM bytes/s."""
    return peak_flops / bandwidth_Bps
