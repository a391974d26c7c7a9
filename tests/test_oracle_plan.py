"""Pins of oracle/plan.py: SPEC.md's worked predictor values (derived from the paper's Eq. 1,
2, 5 by hand), the paper's printed model sizes and hand-off size
(PAPER.md:355), and the exact stage byte counts of SURVEY Appendix A."""
import pytest

import hsgen
from oracle.plan import eq1_ttft, eq2_tpot, eq5_ttft, plan, select_servers, stage_param_bytes


def test_eq1_spec_values():
    assert eq1_ttft(10, 100, 4, 0, [16] * 4, [128] * 4, 0.5, 0.01) == pytest.approx(13.7978125, abs=1e-12)
    assert eq1_ttft(10, 100, 4, 4, [16] * 4, [128] * 4, 0.5, 0.01) == pytest.approx(12.2978125, abs=1e-12)
    assert eq1_ttft(10, 100, 1, 1, [16], [128], 0.5, 0.01) == pytest.approx(17.54125, abs=1e-12)


def test_eq2_spec_values():
    assert eq2_tpot(0.05, 4, 0, 0.01) == pytest.approx(0.24)
    assert eq2_tpot(0.05, 4, 4, 0.01) == pytest.approx(0.09)
    assert eq2_tpot(0.05, 1, 1, 0.01) == pytest.approx(0.06)


def test_eq5_spec_values():
    assert eq5_ttft(4, 2, 6, 100, 4, 0, [16] * 4, [128] * 4, 0.5, 0.01) == pytest.approx(14.04)
    assert eq5_ttft(0, 0, 0, 400, 4, 0, [16] * 4, [1000] * 4, 0, 0) == pytest.approx(6.25)
    assert eq5_ttft(0, 0, 0, 100, 4, 0, [16] * 4, [128] * 4, 0, 0) == pytest.approx(1.5625)


def test_select_servers_spec():
    full = [("A", 0.0234), ("B", 0.039)]
    low = [("C", 0.0703), ("D", 0.078)]
    assert select_servers(full, low, 3, 1) == ["A", "B", "C"]
    assert select_servers(full, low, 2, 0) == ["A", "B"]
    eq = [("b", 1.0), ("a", 1.0)]
    assert select_servers(eq, [], 2, 0) == ["a", "b"]


def test_paper_model_sizes():
    """Llama2-7B 12.5GB, Llama2-13B 24.2GB (GiB, truncated)."""
    for name, paper_gib in (("llama2-7b", 12.5), ("llama2-13b", 24.2)):
        total = sum(stage_param_bytes(hsgen.CONFIGS[name], 1))
        assert int(total / 2**30 * 10) / 10 == paper_gib
    assert sum(stage_param_bytes(hsgen.CONFIGS["llama2-7b"], 1)) == 13_476_831_232
    assert sum(stage_param_bytes(hsgen.CONFIGS["llama2-13b"], 1)) == 26_031_728_640
    # 8 KB of inter-layer results per token for Llama2-7B
    assert hsgen.CONFIGS["llama2-7b"]["hidden"] * 2 == 8 * 1024


def test_stage_bytes_appendix_a():
    c7, c13 = hsgen.CONFIGS["llama2-7b"], hsgen.CONFIGS["llama2-13b"]
    assert stage_param_bytes(c7, 2) == [6_738_411_520, 6_738_419_712]
    s = stage_param_bytes(c7, 4)
    assert (s[0], s[1], s[3]) == (3_500_277_760, 3_238_133_760, 3_500_285_952)
    s = stage_param_bytes(c7, 8)
    assert (s[0], s[1], s[7]) == (1_881_210_880, 1_619_066_880, 1_881_219_072)
    s = stage_param_bytes(c13, 4)
    assert (s[0], s[1], s[3]) == (6_671_769_600, 6_344_089_600, 6_671_779_840)
    assert stage_param_bytes(hsgen.CONFIGS["tiny"], 2) == [3_934_208, 3_934_720]


def test_plan_full_memory_and_prediction():
    cfg = hsgen.CONFIGS["llama2-7b"]
    gpus = [dict(device=i, h2d_gbps=55.0 - i * 0.1, link_group=i // 2, free_bytes=180 * 10**9) for i in range(4)]
    p = plan(cfg, gpus, 4, 1)
    assert p["device"] == [0, 1, 2, 3] and p["full_memory"] == [1, 0, 0, 0]
    assert p["ranges"] == [(0, 8), (8, 16), (16, 24), (24, 32)]
    # TTFT_pred(s) = max_k bytes_k / p_k (+ t_p (s-w+w/s) + s t_n): slowest stage dominates
    assert p["pred_ttft_s"] == pytest.approx(max(b / (g * 1e9) for b, g in zip(p["stage_bytes"], [55.0, 54.9, 54.8, 54.7])))
