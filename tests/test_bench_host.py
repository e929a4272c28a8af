"""Host-side arithmetic of bench.py (no GPU): the algorithmic bytes / flops the roofline divides by
(SURVEY §8(d) table), the choice of the binding roofline (HBM copy peak vs SUSTAINED bf16 tensor
peak), and the workload description both arms print."""
import bench


def test_algorithmic_bytes_match_survey_table():
    # Llama-3-8B 2VD + 2BD (+ 4B idx) = 1050.94 MB at B = 32; W alone 1,050,673,152 B
    assert bench.stage1_bytes(32, 4096, 128256) == 2 * 128256 * 4096 + 2 * 32 * 4096
    assert 2 * 128256 * 4096 == 1_050_673_152
    assert bench.algorithmic_bytes(32, 4096, 128256) == 1_050_935_296 + 4 * 32
    # Qwen2.5-7B with transforms: bias 4V, tau 4B, mask 4B*ceil(V/32)
    b = bench.stage1_bytes(32, 3584, 152064, transforms=True)
    assert b == 2 * 152064 * 3584 + 2 * 32 * 3584 + 4 * 152064 + 4 * 32 + 4 * 32 * 4752
    # grouped summaries 12 B per (row, group); TP exchange 12 B per (row, rank)
    assert bench.algorithmic_bytes(4, 5376, 262208, n_groups=65) - bench.algorithmic_bytes(4, 5376, 262208) == 12 * 4 * 65
    assert bench.algorithmic_bytes(8, 8192, 128256, tp_world=8) - bench.algorithmic_bytes(8, 8192, 128256) == 12 * 8 * 8


def test_roofline_bound_uses_sustained_tensor_peak():
    pk = dict(hbm_gbs=6553.6, bf16_tflops=1650.5, bf16_tflops_sustained=1403.4, source="test")
    # B = 32: HBM-bound; achieved = bytes / time against the copy peak
    r = bench.roofline("llama3_8b", 32, 4096, 128256, 0.1618, pk, False)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert abs(r["achieved"] - bench.stage1_bytes(32, 4096, 128256) / 0.1618e-3 / 1e9) < 0.1
    assert abs(r["frac"] - r["achieved"] / 6553.6) < 1e-3
    # B = 256: 2BVD / sustained (191.7 us) > bytes / HBM (160.5 us) -> tensor-bound at the sustained peak
    r = bench.roofline("llama3_8b", 256, 4096, 128256, 0.2443, pk, False)
    assert r["bound"] == "tensor" and r["peak"] == 1403.4 and r["peak_kind"] == "bf16_tflops_sustained"
    assert abs(r["t_tc_sustained_us"] - 2 * 256 * 128256 * 4096 / 1403.4e12 * 1e6) < 0.05
    assert abs(r["frac_of_floor"] - r["t_tc_sustained_us"] / 244.3) < 1e-3
    # B = 128: HBM-bound at either tensor peak
    r = bench.roofline("llama3_8b", 128, 4096, 128256, 0.1833, pk, False)
    assert r["bound"] == "hbm" and r["frac_of_floor"] == r["frac"]


def test_config_dict_is_shared_by_both_arms():
    a = bench.config_dict("llama3_8b", 32)
    assert a == bench.config_dict("llama3_8b", 32)
    assert a["B"] == 32 and a["D"] == 4096 and a["V"] == 128256 and a["parallelism"] == "single GPU"
    t = bench.config_dict("llama3_8b", 32, world=4)
    assert t["parallelism"] == "tp4 (vocab)" and "per rank" in t["l2"]
    g = bench.config_dict("gemma3_27b", 4)
    assert "65 groups" in g["workload"]
