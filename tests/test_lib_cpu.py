"""CPU-side checks of the C-ABI library (no GPU needed): it loads, exports every symbol the
headers declare, its image layout agrees with the input generator's, and its host-only
planner / predictors agree with the oracle (integers bit-exact, predictions to 1e-12)."""
import os
import re

import pytest

import hsgen
from oracle import plan as oplan
from paper_2502_15524_b200 import hs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = []
    for h in ("hs.h", "hs_kernels.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        names += re.findall(r"^\s*(?:hs_status|double|int32_t|const char\*)\s+(hs_\w+)\s*\(", src, re.M)
    return names


def test_library_exports_every_declared_symbol():
    L = hs.lib()
    decl = declared_symbols()
    assert len(decl) >= 25
    missing = [n for n in decl if not hasattr(L, n)]
    assert not missing, missing
    assert set(decl) == set(hs.SYMBOLS)


def test_probes_live_outside_the_product_library():
    """Test-only hardware probes (include/hs_probes.h) are exported by libhs_probe.so and absent
    from libhs.so."""
    src = open(os.path.join(ROOT, "include", "hs_probes.h")).read()
    probes = re.findall(r"^\s*hs_status\s+(hs_\w+)\s*\(", src, re.M)
    assert probes
    P = hs.probe_lib()
    for n in probes:
        assert hasattr(P, n)
        assert not hasattr(hs.lib(), n), n


@pytest.mark.parametrize("name", ["tiny", "llama2-7b", "llama2-13b"])
def test_image_layout_matches_generator(name):
    a = hs.image_layout(hsgen.CONFIGS[name])
    b = hsgen.image_header(hsgen.CONFIGS[name])
    assert bytes(a) == bytes(b)
    assert a.param_bytes == sum(oplan.stage_param_bytes(hsgen.CONFIGS[name], 1))


@pytest.mark.parametrize("name,pp", [("tiny", 1), ("tiny", 2), ("tiny", 3), ("tiny", 4), ("llama2-7b", 1),
                                     ("llama2-7b", 2), ("llama2-7b", 4), ("llama2-7b", 8), ("llama2-13b", 4),
                                     ("llama2-13b", 8), ("llama2-13b", 3)])
def test_plan_matches_oracle(name, pp):
    cfg = hsgen.CONFIGS[name]
    gpus = [dict(device=i, h2d_gbps=55.6 - 0.01 * ((i * 5) % 8), link_group=i // 2, free_bytes=183 * 2**30)
            for i in range(8)]
    if name != "tiny":  # only two GPUs can hold the whole model: w=1 goes to the fastest of them
        for g in gpus[2:]:
            g["free_bytes"] = 20 * 2**30 if name == "llama2-7b" else 9 * 2**30
    ours = hs.plan_stages(cfg, gpus, pp, 1, t_prefill_s=0.01, t_hop_s=1e-5).as_dict()
    ref = oplan.plan(cfg, gpus, pp, 1, t_prefill_s=0.01, t_hop_s=1e-5)
    assert ours["device"] == ref["device"]
    assert ours["ranges"] == ref["ranges"]
    assert ours["stage_bytes"] == ref["stage_bytes"]
    assert ours["full_memory"] == ref["full_memory"]
    assert ours["pred_ttft_s"] == pytest.approx(ref["pred_ttft_s"], rel=1e-12)
    # slices are contiguous, cover [embed, end) and each holds at least the stage's bytes
    h = hs.image_layout(cfg)
    sl = ours["slices"]
    assert sl[0][0] == h.embed_off and sl[-1][1] == h.total_bytes
    assert all(sl[k][1] == sl[k + 1][0] for k in range(pp - 1))
    assert all(e - b >= nb for (b, e), nb in zip(sl, ours["stage_bytes"]))


def test_plan_errors():
    cfg = hsgen.CONFIGS["llama2-7b"]
    gpus = [dict(device=0, h2d_gbps=55.0, free_bytes=183 * 2**30)]
    with pytest.raises(hs.HsError) as e:
        hs.plan_stages(cfg, gpus, 2, 1)
    assert e.value.code == 4  # HS_E_INFEASIBLE
    with pytest.raises(hs.HsError) as e:
        hs.plan_stages(cfg, gpus, 0, 1)
    assert e.value.code == 1  # pp = 0 (SLO-driven choice) is not implemented yet
    small = [dict(device=i, h2d_gbps=55.0, free_bytes=1 * 2**30) for i in range(8)]
    with pytest.raises(hs.HsError):
        hs.plan_stages(cfg, small, 8, 1)  # 1.9 GB stages do not fit 1 GiB


def test_predictors_spec_values():
    assert hs.predict_ttft_eq1(10, 100, 4, 0, [16] * 4, [128] * 4, 0.5, 0.01) == pytest.approx(13.7978125, abs=1e-12)
    assert hs.predict_ttft_eq1(10, 100, 4, 4, [16] * 4, [128] * 4, 0.5, 0.01) == pytest.approx(12.2978125, abs=1e-12)
    assert hs.predict_tpot_eq2(0.05, 4, 0, 0.01) == pytest.approx(0.24)
    assert hs.predict_tpot_eq2(0.05, 4, 4, 0.01) == pytest.approx(0.09)
    assert hs.predict_ttft_eq5(4, 2, 6, 100, 4, 0, [16] * 4, [128] * 4, 0.5, 0.01) == pytest.approx(14.04)
    for args in [(3, 1, 2, 50, 2, 1, [10, 20], [30, 5], 0.2, 0.01), (0, 0, 0, 400, 4, 0, [16] * 4, [1000] * 4, 0, 0)]:
        assert hs.predict_ttft_eq5(*args) == pytest.approx(oplan.eq5_ttft(*args), rel=1e-12)


def test_prefetcher_fills_region_and_publishes_watermark(tmp_path):
    """Model prefetcher on the host only: the region equals the file bytes,
    the 8-byte watermark ends at the fetched end (image offsets), the throttle holds, and a short
    file is reported with the watermark left at the last complete chunk."""
    import time

    import numpy as np
    data = np.random.default_rng(0).integers(0, 256, 3 << 20, dtype=np.uint8)
    path = tmp_path / "model.img"
    data.tofile(path)
    off = 1 << 20
    dst = np.zeros(2 << 20, dtype=np.uint8)
    wm = np.zeros(1, dtype=np.uint64)
    t0 = time.perf_counter()
    p = hs.Prefetch(str(path), off, dst.ctypes.data, dst.nbytes, wm.ctypes.data, chunk_bytes=256 << 10, max_gbps=0.02)
    seen = []
    while True:
        v = int(wm[0])
        seen.append(v)
        if v >= off + dst.nbytes:
            break
        time.sleep(0.002)
    n, secs = p.wait()
    assert n == dst.nbytes and np.array_equal(dst, data[off:off + dst.nbytes])
    assert seen == sorted(seen) and seen[-1] == off + dst.nbytes and any(off < v < off + dst.nbytes for v in seen)
    assert secs >= 0.9 * dst.nbytes / 0.02e9 and time.perf_counter() - t0 >= 0.09
    p.destroy()
    short = np.zeros(4 << 20, dtype=np.uint8)
    p = hs.Prefetch(str(path), off, short.ctypes.data, short.nbytes, wm.ctypes.data, chunk_bytes=1 << 20)
    with pytest.raises(hs.HsError):
        p.wait()
    assert int(wm[0]) == off + (2 << 20)
    p.destroy()


def test_image_weights_are_tiled_blocks_of_the_draws():
    """The host image's weight matrices are the generator's draws in the tiled weight layout of
    include/hs.h ([M/128][K/64][128][64], w_qkv = q, k, v rows stacked, w_gu = gate/up rows
    interleaved by 16), the embedding table row-major; a partial fill writes exactly the
    requested bytes."""
    import numpy as np
    cfg = hsgen.CONFIGS["tiny"]
    h = hsgen.image_header(cfg)
    img = np.zeros(h.total_bytes, dtype=np.uint8)
    hsgen.image_fill(h, hsgen.WEIGHT_SEED, img.ctypes.data, 0, h.total_bytes)
    H, F = cfg["hidden"], cfg["ffn"]

    def untile(off, M, K):
        t = img[off:off + 2 * M * K].view(np.uint16).reshape(M // 128, K // 64, 128, 64)
        return t.transpose(0, 2, 1, 3).reshape(M, K)

    draw = lambda tid: hsgen.tensor_bf16(cfg, hsgen.WEIGHT_SEED, tid)  # noqa: E731
    l = 2
    L0 = h.layer_off[l]
    qkv = np.concatenate([draw(hsgen.layer_tensor(l, k)) for k in (hsgen.WQ, hsgen.WK, hsgen.WV)])
    assert np.array_equal(untile(L0 + h.t_wqkv, 3 * H, H), qkv)
    assert np.array_equal(untile(L0 + h.t_wo, H, H), draw(hsgen.layer_tensor(l, hsgen.WO)))
    g, u = draw(hsgen.layer_tensor(l, hsgen.WG)), draw(hsgen.layer_tensor(l, hsgen.WU))
    gu = np.stack([g.reshape(-1, 16, H), u.reshape(-1, 16, H)], axis=1).reshape(2 * F, H)
    assert np.array_equal(untile(L0 + h.t_wgu, 2 * F, H), gu)
    assert np.array_equal(untile(L0 + h.t_wd, H, F), draw(hsgen.layer_tensor(l, hsgen.WD)))
    assert np.array_equal(untile(h.final_off + h.t_lm_head, cfg["vocab"], H), draw(hsgen.LM_HEAD))
    emb = img[h.embed_off:h.embed_off + 2 * cfg["vocab"] * H].view(np.uint16).reshape(cfg["vocab"], H)
    assert np.array_equal(emb, draw(hsgen.EMBED))
    part = np.zeros(h.layer_bytes + 77, dtype=np.uint8)  # an unaligned slice across a layer
    b = int(L0) - 33
    hsgen.image_fill(h, hsgen.WEIGHT_SEED, part.ctypes.data, b, b + part.size)
    assert np.array_equal(part, img[b:b + part.size])
