"""Pins of oracle.costmodel against the worked numbers PAPER.md prints (§4.7, Table 2)."""
import json
import os

import pytest

from oracle import costmodel

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "costmodel_paper.json")))


def test_extra_traffic_fraction_p437():
    for row in GOLD["extra_fraction_2B_over_D"]:
        got = 100 * costmodel.extra_traffic_fraction(row["B"], row["D"])
        assert round(got, 3) == pytest.approx(row["percent"], abs=1e-3)


def test_round_trip_p441():
    r = GOLD["round_trip"]
    b = costmodel.logits_round_trip_bytes(r["B"], r["V"])
    assert b == r["bytes"]
    assert round(b / 1e6, 3) == r["MB"]
    assert 1e3 * costmodel.seconds_at(b, 8e12) == pytest.approx(r["ms_at_8TBps"], rel=5e-3)


def test_ops_per_byte_table2():
    for row in GOLD["ops_per_byte"]:
        got = costmodel.ops_per_byte(row["tflops"] * 1e12, row["tbps"] * 1e12)
        assert round(got) == row["ratio"]


def test_intensity_forms():
    # fused intensity exceeds the materialised bound, and both ~ B at B << V, D
    for B in (1, 8, 64, 256):
        im = costmodel.intensity_materialized(B, 151936, 4096)
        fu = costmodel.intensity_fused(B, 151936, 4096)
        assert fu > im
        assert fu == pytest.approx(B, rel=B / 151936 * 1.01 + 1e-12)
