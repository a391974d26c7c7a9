"""SLO-driven choice of s (Algorithm 1) and contention-aware
admission of simultaneous cold starts on shared host links (Eq. 3/4).  The library (host
code, CPU) against SPEC.md's worked values and the oracle's exhaustive/literal versions."""
import numpy as np
import pytest

import hsgen
from oracle import plan as oplan
from paper_2502_15524_b200 import hs

CFG = hsgen.CONFIGS["llama2-7b"]
MODEL = sum(oplan.stage_param_bytes(CFG, 1))


def test_admit_settle_spec_examples():
    # SPEC.md:213-215 (Gbit units; any consistent unit works)
    L = hs.Links([16.0])
    assert L.admit(0, 50, 10, 0) == (True, 1)
    assert L.admit(0, 25, 5, 0)[0]                       # shares 8: 50 <= 80 and 25 <= 40
    L2 = hs.Links([16.0])
    L2.admit(0, 50, 5, 0)
    assert not L2.admit(0, 1, 100, 0)[0]                 # 50 <= 8 * 5 = 40 is false
    assert hs.Links([16.0]).admit(0, 100, 100, 0)[0]     # empty server
    # S=100, B=16, N=2, 5 s -> 60; 15 s -> removed
    L3 = hs.Links([16.0])
    _, a = L3.admit(0, 100, 1000, 0)
    _, b = L3.admit(0, 100, 1000, 0)
    L3.settle(0, 5.0)
    assert L3.pending(0) == {a: pytest.approx(60.0), b: pytest.approx(60.0)}
    L3.settle(0, 15.0)
    assert L3.pending(0) == {}


def test_contention_randomized_vs_oracle():
    rng = np.random.default_rng(0)
    for trial in range(200):
        B = float(rng.uniform(10, 100))
        lib, ora = hs.Links([B]), oplan.ContentionRegistry(B)
        now, live = 0.0, []
        for _ in range(30):
            now += float(rng.exponential(1.0))
            if live and rng.random() < 0.3:
                wid = live.pop(int(rng.integers(len(live))))
                lib.complete(0, wid, now)
                ora.complete(wid, now)
            else:
                S, D = float(rng.uniform(1, 200)), now + float(rng.uniform(0.5, 20))
                r1, r2 = lib.admit(0, S, D, now), ora.admit(S, D, now)
                assert r1 == r2, (trial, r1, r2)
                if r1[0]:
                    live.append(r1[1])
            pend = lib.pending(0)
            assert set(pend) == set(ora.ws)
            for k, v in pend.items():
                assert v == pytest.approx(ora.ws[k][0], rel=1e-9, abs=1e-9)


def gpus_box(n=8, workers=None, free=None):
    return [dict(device=i, h2d_gbps=55.6, link_group=i, free_bytes=(free or {}).get(i, 180 * 10**9),
                 n_workers=(workers or {}).get(i, 0)) for i in range(n)]


@pytest.mark.parametrize("case", range(60))
def test_alg1_matches_exhaustive_oracle(case):
    rng = np.random.default_rng(case)
    workers = {i: int(rng.integers(0, 3)) for i in range(8)}
    free = {i: int(rng.choice([20, 60, 180])) * 10**9 for i in range(8)}
    g = gpus_box(8, workers, free)
    t_p, t_d, t_n = float(rng.uniform(0.004, 0.03)), float(rng.uniform(0.002, 0.01)), float(rng.uniform(1e-5, 1e-3))
    slo_ttft, slo_tpot = float(rng.uniform(0.03, 0.4)), float(rng.uniform(0.003, 0.05))
    p, share, ok = hs.plan_auto(CFG, g, t_p, t_d, t_n, slo_ttft, slo_tpot, max_pp=8)
    rp, rshare, rok = oplan.alg1(CFG, g, t_p, t_d, t_n, slo_ttft, slo_tpot, max_pp=8)
    d = p.as_dict()
    assert ok == rok and share == rshare
    assert d["device"] == rp["device"] and d["ranges"] == rp["ranges"] and d["full_memory"] == rp["full_memory"]
    if ok:  # soundness
        assert d["pred_ttft_s"] <= slo_ttft + 1e-12
        assert oplan.eq2_tpot(t_d, d["pp"], sum(d["full_memory"]), t_n) <= slo_tpot + 1e-12


def test_alg1_prefers_free_gpus_and_falls_back():
    # GPUs 0-3 busy, 4-7 idle: the chosen plan uses idle GPUs only
    g = gpus_box(8, workers={0: 1, 1: 1, 2: 1, 3: 1})
    p, share, ok = hs.plan_auto(CFG, g, 0.01, 0.005, 1e-5, 1.0, 1.0, max_pp=4)
    assert ok and share == 0 and all(d >= 4 for d in p.as_dict()["device"])
    # an impossible TTFT SLO -> (1, 1, (i_1)) fallback
    p, share, ok = hs.plan_auto(CFG, gpus_box(8), 0.01, 0.005, 1e-5, 1e-4, 1.0, max_pp=4)
    assert not ok and p.pp == 1 and p.full_memory[0] == 1
    # a tight TTFT SLO forces s > 1 (7B: 242 ms over one link, 63 ms at s = 4)
    p, share, ok = hs.plan_auto(CFG, gpus_box(8), 0.005, 0.005, 1e-5, 0.1, 1.0, max_pp=8)
    assert ok and p.pp >= 3


@pytest.mark.parametrize("case", range(40))
def test_place_cold_start_matches_oracle(case):
    """hs_place_cold_start (library) == oracle.plan.place_cold_start (Alg. 1 + Eq. 3/4, reading
    R20) over a random burst of mixed 7B / 13B cold starts on 4 or 8 GPUs with per-GPU or shared
    link groups: same GPUs, stage ranges, prediction, admission, and the same registries after."""
    rng = np.random.default_rng(100 + case)
    n = int(rng.choice([4, 8]))
    shared = bool(rng.integers(0, 2))
    groups = [i // 2 if shared else i for i in range(n)]
    ng = max(groups) + 1
    B = [float(rng.uniform(40, 120)) * 1e9 for _ in range(ng)]
    gpus = [dict(device=i, h2d_gbps=float(rng.uniform(40, 60)), link_group=groups[i], free_bytes=180 * 10**9)
            for i in range(n)]
    links = hs.Links(B)
    regs = {g: oplan.ContentionRegistry(B[g]) for g in range(ng)}
    now = 0.0
    for j in range(10):
        now += float(rng.gamma(1 / 64, 64 / 8.0))
        cfg = hsgen.CONFIGS["llama2-7b" if rng.random() < 0.5 else "llama2-13b"]
        slo = float(rng.uniform(0.05, 0.6))
        p, pred, ok, ids = links.place(cfg, gpus, now, slo, max_pp=4)
        rp, rpred, rok, rids = oplan.place_cold_start(cfg, gpus, regs, now, slo, max_pp=4)
        d = p.as_dict()
        assert d["device"] == rp["device"] and d["ranges"] == rp["ranges"], (case, j)
        assert ok == rok and pred == pytest.approx(rpred, rel=1e-12) and len(set(ids)) == len(ids) == p.pp
        for g in range(ng):  # same workers (pending bytes, deadlines) on every link group
            pend = sorted(links.pending(g).values())
            ref = sorted(S for S, _ in regs[g].ws.values())
            assert len(pend) == len(ref)
            for a, b in zip(pend, ref):
                assert a == pytest.approx(b, rel=1e-9, abs=1e-3)


def test_place_cold_start_spreads_a_burst():
    """Four simultaneous 7B cold starts on 4 GPUs with independent links: the first takes all 4
    GPUs (s = 4 is the fastest), later ones see the links busy and the predictions grow; each
    prediction accounts for the equal-credit share of every load in flight."""
    gpus = [dict(device=i, h2d_gbps=55.0, link_group=i, free_bytes=180 * 10**9) for i in range(4)]
    links = hs.Links([55e9] * 4)
    preds = []
    for j in range(4):
        p, pred, ok, ids = links.place(CFG, gpus, 0.0, 10.0, max_pp=4)
        preds.append(pred)
        assert len(ids) == p.pp
    assert preds[0] == pytest.approx(max(oplan.stage_param_bytes(CFG, 4)) / 55e9, rel=1e-9)
    assert preds == sorted(preds)
