"""Full-size (Llama-2-7B shape, BASELINE configs 2/3) checks on the GPU, in the kernels and
launch configuration bench.py times (512-token prefill -> tensor-core prefill GEMMs and
flash attention; decode -> stream-K GEMMs with fused epilogues, split-KV attention):

  * properties that hold at any size, bitwise: PP=2 == PP=1 (logits, KV), consolidated KV ==
    pre-consolidation KV, consolidated weights == the host image, decode after consolidation
    == unpartitioned decode;
  * the oracle at full size on sampled outputs: final logits of a 128-token prompt and 3
    teacher-forced decode steps vs the fp64 oracle, tolerance max(2e-2, 1.5 x the oracle's own
    fp32-accumulation floor on the same inputs).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

import hsgen  # noqa: E402

if torch.cuda.is_available():
    from paper_2502_15524_b200 import hs  # noqa: E402

CFG = dict(hsgen.CONFIGS["llama2-7b"])


@pytest.fixture(scope="module")
def image():
    h = hs.image_layout(CFG)
    img = hs.HostImage(h, 0, h.total_bytes)
    hsgen.image_fill(hsgen.image_header(CFG), hsgen.WEIGHT_SEED, img.ptr, 0, h.total_bytes)
    return img


def group(image, pp):
    gpus = [dict(device=d, h2d_gbps=55.0, free_bytes=180 << 30) for d in range(pp)]
    plan = hs.plan_stages(CFG, gpus, pp, 1)
    for k in range(pp):
        plan.device[k] = 0
    g = hs.Group(CFG, plan, image, num_blocks=160, max_seqs=2, max_tokens=512)
    g.load_stage_async(-1)
    return g


def test_7b_pp_invariance_and_consolidation_bitwise(image):
    prompt = hsgen.prompts(1, 512, CFG["vocab"])
    g1, g2 = group(image, 1), group(image, 2)
    t1, l1 = g1.prefill([0], prompt, want_logits=True)
    t2, l2 = g2.prefill([0], prompt, want_logits=True)
    assert np.array_equal(t1, t2) and np.array_equal(l1, l2)
    for _ in range(8):
        a, b = g1.decode_step([0], want_logits=True), g2.decode_step([0], want_logits=True)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    layers = [0, 15, 16, 31]
    kv = {l: g2.read_kv(0, l, 0, 520) for l in layers}
    for l in layers:
        assert np.array_equal(kv[l], g1.read_kv(0, l, 0, 520))
    st = g2.consolidate(0)
    assert st.weight_bytes == 6_738_419_712  # the last stage's slice
    assert st.kv_bytes == 33 * 16 * 2 * 4096 * 2 * 16  # 33 blocks x 16 moved layers
    for l in layers:
        assert np.array_equal(g2.read_kv(0, l, 0, 520), kv[l])
    h = hs.image_layout(CFG)
    w = g2.read_weights(0, h.embed_off, h.total_bytes - h.embed_off)
    assert np.array_equal(w, image.buf.numpy()[h.embed_off:])
    for _ in range(4):
        a, b = g1.decode_step([0], want_logits=True), g2.decode_step([0], want_logits=True)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    g1.destroy()
    g2.destroy()


def test_7b_logits_vs_oracle_sampled(image):
    from oracle.decoder import Group as OGroup, Weights
    prompt = hsgen.prompts(1, 128, CFG["vocab"])
    W = Weights(CFG, cache=True)
    og = OGroup(CFG, W, pp=1, num_blocks=16)
    fg = OGroup(CFG, W, pp=1, num_blocks=16, acc=np.float32)
    rt, rl = og.prefill([0], prompt)
    _, fl = fg.prefill([0], prompt)
    hist, floor = [(rt, rl)], [np.abs(rl - fl).max()]
    for _ in range(3):
        t_in = hist[-1][0]
        t, l = og.decode([0], t_in)
        _, f = fg.decode([0], t_in)
        hist.append((t, l))
        floor.append(np.abs(l - f).max())
    tol = max(2e-2, 1.5 * max(floor))
    g = group(image, 2)
    toks, logits = g.prefill([0], prompt, want_logits=True)
    errs = [np.abs(logits - rl).max()]
    assert toks[0] == rt[0]
    for step in range(1, 4):
        toks, logits = g.decode_step([0], hist[step - 1][0], want_logits=True)
        errs.append(np.abs(logits - hist[step][1]).max())
        assert toks[0] == hist[step][0][0]
    print("7B max|dlogit| per step", errs, "floor", floor, "tol", tol)
    assert max(errs) <= tol, (errs, floor)
    g.destroy()


def test_7b_pp8_equals_pp1_then_consolidates(image):
    """PP = 8 (the scaling run's largest degree; 4 layers per stage, 8 stages on one GPU here):
    prefill and decode bitwise equal to PP = 1, consolidation into stage 0, decode continues
    bitwise equal."""
    prompt = hsgen.prompts(1, 512, CFG["vocab"])
    g1, g8 = group(image, 1), group(image, 8)
    t1, l1 = g1.prefill([0], prompt, want_logits=True)
    t8, l8 = g8.prefill([0], prompt, want_logits=True)
    assert np.array_equal(t1, t8) and np.array_equal(l1, l8)
    for _ in range(4):
        a, b = g1.decode_step([0], want_logits=True), g8.decode_step([0], want_logits=True)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    g8.consolidate(0)
    for _ in range(2):
        a, b = g1.decode_step([0], want_logits=True), g8.decode_step([0], want_logits=True)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    g1.destroy()
    g8.destroy()
