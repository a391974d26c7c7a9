"""Full-size checks on the GPU in the kernels and launch configuration bench.py times
(Llama-2-7B shape: BASELINE configs 2/3; Llama-2-13B shape: config 4):

  * properties that hold at any size, bitwise: PP=s == PP=1 (logits, KV), consolidated KV ==
    pre-consolidation KV, consolidated weights == the host image, decode after consolidation
    == unpartitioned decode;
  * the oracle, layer by layer (tests/layerwise.py): every half-layer of every
    layer fed the GPU's own input, within one bf16 ulp at the row's scale; logits from the GPU's
    final hidden state within 2e-2 of the oracle's head; greedy tokens = the oracle's argmax of
    the same state.  7B: 512-token prefill + 64 decode steps, all 32 layers.  13B config 4: 16 x
    512 prefill (4 micro-batches) + 64 decode steps at B=16 (decode stack, H=5120), consolidation
    into stage 0 (all 16 sequences' KV compared byte for byte), 64 more steps; the oracle follows
    2 of the 16 sequences on 8 layers (every stage's first and last).
The measured errors are written to gpurun_out/parity_*.json (copied to profiles/).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

import hsgen  # noqa: E402
import layerwise as LW  # noqa: E402
from oracle.decoder import Weights  # noqa: E402

if torch.cuda.is_available():
    from paper_2502_15524_b200 import hs  # noqa: E402

CFG = dict(hsgen.CONFIGS["llama2-7b"])


def make_image(cfg):
    h = hs.image_layout(cfg)
    img = hs.HostImage(h, 0, h.total_bytes)
    hsgen.image_fill(hsgen.image_header(cfg), hsgen.WEIGHT_SEED, img.ptr, 0, h.total_bytes)
    return img


@pytest.fixture(scope="module")
def image():
    return make_image(CFG)


def group(image, pp, cfg=CFG, num_blocks=160, max_seqs=2, max_tokens=512):
    gpus = [dict(device=d, h2d_gbps=55.0, free_bytes=180 << 30) for d in range(pp)]
    plan = hs.plan_stages(cfg, gpus, pp, 1)
    for k in range(pp):
        plan.device[k] = 0
    g = hs.Group(cfg, plan, image, num_blocks=num_blocks, max_seqs=max_seqs, max_tokens=max_tokens)
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


@pytest.mark.parametrize("pp", [1, 2])
def test_7b_layerwise_512_prefill_64_decode(image, pp):
    """Config 2 (PP=1) / config 3 shape (PP=2): 512-token prefill + 64 greedy decode steps
    (device feedback, the decode stack), every half-layer of all 32 layers against the oracle."""
    prompt = hsgen.prompts(1, 512, CFG["vocab"])
    g = group(image, pp)
    g.capture(True)
    rec = LW.Recorder(CFG)
    toks, logits = g.prefill([0], prompt, want_logits=True)
    rec.record(g, [0], [512], logits, toks)
    for _ in range(64):
        toks, logits = g.decode_step([0], want_logits=True)
        rec.record(g, [0], [1], logits, toks)
    W = Weights(CFG, cache=True)
    res = {}
    LW.check_heads(CFG, W, rec, res)
    LW.check_layers(CFG, W, rec, g, range(CFG["n_layers"]), [("prefill", {0: (0, 1)}), ("decode", {0: (1, None)})],
                    res, evict=True)
    res["summary"] = LW.summary(res)
    LW.save(res, f"7b_pp{pp}")
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


def test_13b_config4_layerwise_and_consolidation():
    """BASELINE config 4 on one GPU (4 stages): 13B, 16 x 512 prompts (4 prefill micro-batches),
    64 decode steps at B = 16 through the decode stack (H = 5120), consolidation into stage 0
    after step 64 (ctx 576; every live sequence's KV of the 30 moved layers compared byte for
    byte; weights against the host image), 64 more steps.  The oracle follows sequences 0 and 15
    on the first and last layer of every stage (prefill, decode before and after consolidation)."""
    cfg = dict(hsgen.CONFIGS["llama2-13b"])
    img = make_image(cfg)
    n, plen = 16, 512
    prompts = hsgen.prompts(n, plen, cfg["vocab"])
    ids = list(range(n))
    nb = n * ((plen + 128 + 15) // 16 + 1) + 8
    g = group(img, 4, cfg, num_blocks=nb, max_seqs=n, max_tokens=n * plen)
    g.capture(True)
    follow = [0, 15]
    L = cfg["n_layers"]
    layers = [0, 9, 10, 19, 20, 29, 30, 39]
    rec = LW.Recorder(cfg, points=sorted({p for l in layers for p in (2 * l, 2 * l + 1, 2 * l + 2)} | {2 * L}))
    toks, logits = g.prefill(ids, prompts, want_logits=True)
    rec.record(g, ids, [plen] * n, logits, toks, want=follow)
    for _ in range(64):
        toks, logits = g.decode_step(ids, want_logits=True)
        rec.record(g, ids, [1] * n, logits, toks, want=follow)
    moved = range(10, L)
    kv_before = {(s, l): g.read_kv(s, l, 0, plen + 64) for s in ids for l in moved}
    st = g.consolidate(0)
    assert st.kv_bytes == 5_662_310_400  # 16 seqs x 36 blocks x 320 KiB x 30 layers
    assert st.weight_bytes == 19_359_959_040
    for (s, l), v in kv_before.items():
        assert np.array_equal(g.read_kv(s, l, 0, plen + 64), v), (s, l)
    del kv_before
    h = hs.image_layout(cfg)
    assert np.array_equal(g.read_weights(0, h.embed_off, h.total_bytes - h.embed_off), img.buf.numpy()[h.embed_off:])
    for _ in range(64):
        toks, logits = g.decode_step(ids, want_logits=True)
        rec.record(g, ids, [1] * n, logits, toks, want=follow)
    W = Weights(cfg, cache=True)
    res = {"consolidation": dict(weight_bytes=st.weight_bytes, kv_bytes=st.kv_bytes, seconds=st.seconds,
                                 pause_seconds=st.pause_seconds)}
    LW.check_heads(cfg, W, rec, res)
    phases = [("prefill", {s: (0, 1) for s in follow}), ("decode_pp4", {s: (1, 65) for s in follow}),
              ("decode_consolidated", {s: (65, None) for s in follow})]
    LW.check_layers(cfg, W, rec, g, layers, phases, res, evict=True)
    res["summary"] = LW.summary(res)
    LW.save(res, "13b_config4")
    g.destroy()
