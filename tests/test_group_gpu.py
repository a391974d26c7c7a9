"""End-to-end parity of the pipeline-parallel group (C ABI hs_* calls) against the oracle on
BASELINE config 1 (tiny decoder, one 32-token prompt, PP=2, 8 greedy decode steps, then
consolidation to one stage, continued to 64 steps), plus the GPU-side invariants:
PP=s == PP=1 bitwise (partition-invariant kernels), consolidated KV / weights bit-exact,
readiness gating (poisoned weights + streamed load), multi-sequence varlen prefill.

Acceptance (BASELINE north star): max |logit - oracle| <= TOL and
greedy tokens equal for >= 64 steps (teacher-forced; a mismatch only counts as a tie when
the oracle's top-2 margin is below 2x the observed logit error).  TOL = max(2e-2, 1.5 x F)
where F is the floor measured on the same workload between the oracle and the oracle with
fp32 accumulation (tests/test_oracle_floor.py: F ~ 2.2-2.6e-2 on config 1, i.e. the north
star's 2e-2 sits at the bf16 noise floor of any fp32-accumulating implementation)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import hsgen  # noqa: E402
from oracle.decoder import Group as OGroup, Weights  # noqa: E402

if torch.cuda.is_available():
    from paper_2502_15524_b200 import hs  # noqa: E402

CFG = hsgen.CONFIGS["tiny"]
TOL = 2e-2
ERRS = []


@pytest.fixture(scope="module")
def image():
    h = hs.image_layout(CFG)
    img = hs.HostImage(h, 0, h.total_bytes)
    hsgen.image_fill(hsgen.image_header(CFG), hsgen.WEIGHT_SEED, img.ptr, 0, h.total_bytes)
    return img


@pytest.fixture(scope="module")
def oracle_run():
    """Oracle: prefill + 72 greedy steps of two prompts (teacher-forcing reference), and the
    fp32-accumulation floor F on the same teacher-forced run."""
    global TOL
    W = Weights(CFG)
    g = OGroup(CFG, W, pp=1, num_blocks=64)
    f = OGroup(CFG, W, pp=1, num_blocks=64, acc=np.float32)
    prompts = hsgen.prompts(2, 32, CFG["vocab"])
    toks, logits = g.prefill([0, 1], prompts)
    _, lf = f.prefill([0, 1], prompts)
    floor = [np.abs(logits - lf).max()]
    hist = [(np.array(toks), logits)]
    for _ in range(72):
        t_in = toks
        toks, logits = g.decode([0, 1], t_in)
        _, lf = f.decode([0, 1], t_in)
        floor.append(np.abs(logits - lf).max())
        hist.append((np.array(toks), logits))
    TOL = max(2e-2, 1.5 * max(floor))
    return prompts, hist, g


def make_group(image, pp, devices=None, num_blocks=64):
    n = torch.cuda.device_count()
    devices = devices or [0] * pp
    gpus = [dict(device=d, h2d_gbps=50.0, free_bytes=8 << 30) for d in range(max(n, pp))]
    plan = hs.plan_stages(CFG, gpus, pp, 1)
    for k in range(pp):  # fake PP: several stages on one GPU
        plan.device[k] = devices[k]
    return hs.Group(CFG, plan, image, num_blocks=num_blocks, max_seqs=8, max_tokens=256)


def compare(step, gpu_tok, gpu_logits, ref_tok, ref_logits, ties):
    err = np.abs(gpu_logits.astype(np.float64) - ref_logits).max()
    ERRS.append(err)
    assert err <= TOL, f"step {step}: max |dlogit| {err}"
    for i in range(len(ref_tok)):
        if gpu_tok[i] != ref_tok[i]:
            top2 = np.sort(ref_logits[i])[-2:]
            assert top2[1] - top2[0] < 2 * err, f"step {step} seq {i}: token mismatch without a tie"
            ties.append((step, i))
    return err


@pytest.mark.parametrize("pp", [1, 2])
def test_tiny_teacher_forced_64_steps(image, oracle_run, pp):
    prompts, hist, _ = oracle_run
    g = make_group(image, pp)
    g.load_stage_async(-1)
    ties, errs = [], []
    toks, logits = g.prefill([0, 1], prompts, want_logits=True)
    errs.append(compare(0, toks, logits, hist[0][0], hist[0][1], ties))
    for step in range(1, 65):
        toks, logits = g.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        errs.append(compare(step, toks, logits, hist[step][0], hist[step][1], ties))
    assert len(ties) <= 1, ties
    g.destroy()


def test_tiny_free_running_greedy_matches_oracle(image, oracle_run):
    """Device-side token feedback (in_tokens = NULL): 64 greedy steps equal the oracle's."""
    prompts, hist, _ = oracle_run
    g = make_group(image, 2)
    g.load_stage_async(-1)
    toks, _ = g.prefill([0, 1], prompts)
    seq = [toks.copy()]
    for _ in range(64):
        toks, _ = g.decode_step([0, 1])
        seq.append(toks.copy())
    ref = [h[0] for h in hist[:65]]
    # equal until the first oracle near-tie (margin < 2*TOL); afterwards sequences may fork
    for step, (a, b) in enumerate(zip(seq, ref)):
        if not np.array_equal(a, b):
            top2 = np.sort(hist[step][1], axis=1)[:, -2:]
            assert (top2[:, 1] - top2[:, 0]).min() < 2 * TOL, f"fork at step {step} without a tie"
            break
    else:
        return
    assert step >= 16, step
    g.destroy()


def test_pp_split_equals_unsplit_bitwise_on_gpu(image, oracle_run):
    prompts, hist, _ = oracle_run
    runs = []
    for pp in (1, 2, 4):
        g = make_group(image, pp)
        g.load_stage_async(-1)
        out = [g.prefill([0, 1], prompts, want_logits=True)]
        for step in range(1, 9):
            out.append(g.decode_step([0, 1], hist[step - 1][0], want_logits=True))
        kv = [g.read_kv(s, l, 0, 40) for s in (0, 1) for l in range(CFG["n_layers"])]
        runs.append((out, kv))
        g.destroy()
    for out, kv in runs[1:]:
        for (t0, l0), (t1, l1) in zip(runs[0][0], out):
            assert np.array_equal(t0, t1) and np.array_equal(l0, l1)
        for a, b in zip(runs[0][1], kv):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("pp,target", [(2, 0), (4, 0)])
def test_consolidation_bit_exact_then_decode(image, oracle_run, pp, target):
    """Config 1: PP=2, 8 greedy steps, consolidate to stage 0, continue to 64 steps."""
    prompts, hist, _ = oracle_run
    g1 = make_group(image, 1)
    g1.load_stage_async(-1)
    g = make_group(image, pp)
    g.load_stage_async(-1)
    ref_out = [g1.prefill([0, 1], prompts, want_logits=True)]
    out = [g.prefill([0, 1], prompts, want_logits=True)]
    for step in range(1, 9):
        ref_out.append(g1.decode_step([0, 1], hist[step - 1][0], want_logits=True))
        out.append(g.decode_step([0, 1], hist[step - 1][0], want_logits=True))
    kv_before = {(s, l): g.read_kv(s, l, 0, 40) for s in (0, 1) for l in range(CFG["n_layers"])}
    st = g.consolidate(target)
    assert g.info()[0] == 1
    # P8 byte counts: weights = model - target slice; KV = blocks of live seqs x moved layers
    stage_bytes = hs.plan_stages(CFG, [dict(device=d, h2d_gbps=50.0, free_bytes=8 << 30) for d in range(pp)], pp, 1).as_dict()["stage_bytes"]
    assert st.weight_bytes == sum(stage_bytes) - stage_bytes[target]
    moved = CFG["n_layers"] - CFG["n_layers"] // pp
    assert st.kv_bytes == 2 * 3 * moved * 16 * 2 * CFG["hidden"] * 2
    # KV bit-exact (gathered blocks placed at their layers)
    for k, v in kv_before.items():
        assert np.array_equal(g.read_kv(k[0], k[1], 0, 40), v)
    # weights bit-exact against the host image
    h = hs.image_layout(CFG)
    w = g.read_weights(target, h.embed_off, h.total_bytes - h.embed_off)
    assert np.array_equal(w, image.buf.numpy()[h.embed_off:])
    # continue decoding alone == unpartitioned run (bitwise), up to 64 steps in total
    for step in range(9, 65):
        a = g.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        b = g1.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), step
        assert np.abs(a[1] - hist[step][1]).max() <= TOL
    g.destroy()
    g1.destroy()


def test_readiness_gating_with_poisoned_weights(image, oracle_run):
    """Weights poisoned with bf16 NaN, load issued with tiny chunks, prefill enqueued at once:
    any missing per-layer wait would read NaN weights."""
    prompts, hist, _ = oracle_run
    g = make_group(image, 2)
    for k in range(2):
        g.poison(k)
    g.load_stage_async(-1, chunk_bytes=64 << 10)
    toks, logits = g.prefill([0, 1], prompts, want_logits=True)
    assert np.isfinite(logits).all()
    assert np.abs(logits - hist[0][1]).max() <= TOL
    s = g.load_stats(0)
    assert s.done == 1 and s.layers_ready == 2
    g.destroy()


def test_varlen_multi_sequence_prefill(image):
    W = Weights(CFG)
    prompts = [hsgen.tokens(100 + i, n, CFG["vocab"]) for i, n in enumerate((5, 17, 33, 1))]
    og = OGroup(CFG, W, pp=1, num_blocks=64)
    rt, rl = og.prefill([0, 1, 2, 3], prompts)
    g = make_group(image, 2)
    g.load_stage_async(-1)
    toks, logits = g.prefill([10, 11, 12, 13], prompts, want_logits=True)
    assert np.abs(logits - rl).max() <= TOL
    assert list(toks) == list(rt)
    for sid in (10, 11, 12, 13):
        g.release_seq(sid)
    with pytest.raises(hs.HsError):
        g.decode_step([10])
    g.destroy()


def test_errors_are_returned(image):
    g = make_group(image, 2)
    with pytest.raises(hs.HsError) as e:  # prefill before any load was issued
        g.prefill([0], [hsgen.tokens(1, 4, CFG["vocab"])])
    assert e.value.code == 5
    g.load_stage_async(-1)
    with pytest.raises(hs.HsError) as e:
        g.prefill([0], [np.array([CFG["vocab"]], np.int32)])
    assert e.value.code == 1
    with pytest.raises(hs.HsError):
        g.consolidate(1)  # stage 1 is a low-memory worker
    g.destroy()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_two_gpu_pipeline_and_consolidation(image, oracle_run):
    prompts, hist, _ = oracle_run
    g = make_group(image, 2, devices=[0, 1])
    g.load_stage_async(-1)
    toks, logits = g.prefill([0, 1], prompts, want_logits=True)
    assert np.abs(logits - hist[0][1]).max() <= TOL
    for step in range(1, 9):
        toks, logits = g.decode_step([0, 1], None if step > 1 else toks, want_logits=True)
        assert np.abs(logits - hist[step][1]).max() <= TOL
    g.consolidate(0)
    for step in range(9, 20):
        toks, logits = g.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        assert np.abs(logits - hist[step][1]).max() <= TOL
    g.destroy()


@pytest.mark.parametrize("pp", [2, 4])
def test_background_host_load_then_kv_only_consolidation(image, oracle_run, pp):
    """the target loads the other stages' layers over its own host link in
    the background while the group decodes pipelined; consolidation then moves only KV."""
    prompts, hist, _ = oracle_run
    g = make_group(image, pp)
    g.load_stage_async(-1)
    g.prefill([0, 1], prompts)
    g.load_background_async(0)
    for step in range(1, 9):
        toks, logits = g.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        assert np.abs(logits - hist[step][1]).max() <= TOL
    kv_before = {(s, l): g.read_kv(s, l, 0, 40) for s in (0, 1) for l in range(CFG["n_layers"])}
    st = g.consolidate(0)
    sb = hs.plan_stages(CFG, [dict(device=d, h2d_gbps=50.0, free_bytes=8 << 30) for d in range(pp)], pp, 1).as_dict()["stage_bytes"]
    assert st.weight_bytes == 0 and st.weight_bytes_host == sum(sb) - sb[0] and st.kv_bytes > 0
    for k, v in kv_before.items():
        assert np.array_equal(g.read_kv(k[0], k[1], 0, 40), v)
    h = hs.image_layout(CFG)
    assert np.array_equal(g.read_weights(0, h.embed_off, h.total_bytes - h.embed_off), image.buf.numpy()[h.embed_off:])
    for step in range(9, 20):
        toks, logits = g.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        assert np.abs(logits - hist[step][1]).max() <= TOL
    g.destroy()


def test_scale_up_every_stage_becomes_an_endpoint(image, oracle_run):
    """PP=2 with both stages full-memory; after 8 steps
    every stage becomes a standalone endpoint holding the whole model and the KV of the
    sequences assigned to it; each endpoint then decodes its sequence alone == PP=1 run."""
    prompts, hist, _ = oracle_run
    n = torch.cuda.device_count()
    gpus = [dict(device=d, h2d_gbps=50.0, free_bytes=8 << 30) for d in range(max(n, 2))]
    plan = hs.plan_stages(CFG, gpus, 2, 2)
    plan.device[0] = plan.device[1] = 0
    g = hs.Group(CFG, plan, image, num_blocks=64, max_seqs=8, max_tokens=256)
    g.load_stage_async(-1)
    g1 = make_group(image, 1)
    g1.load_stage_async(-1)
    g.prefill([0, 1], prompts)
    g1.prefill([0, 1], prompts)
    for step in range(1, 9):
        g.decode_step([0, 1], hist[step - 1][0])
        g1.decode_step([0, 1], hist[step - 1][0])
    kv_before = {(s_, l): g.read_kv(s_, l, 0, 40) for s_ in (0, 1) for l in range(CFG["n_layers"])}
    eps, st = g.scale_up([0, 1])  # seq 0 -> endpoint 0, seq 1 -> endpoint 1
    assert len(eps) == 2 and st.kv_bytes > 0
    h = hs.image_layout(CFG)
    for k, e in enumerate(eps):
        assert e.info()[0] == 1
        assert np.array_equal(e.read_weights(0, h.embed_off, h.total_bytes - h.embed_off), image.buf.numpy()[h.embed_off:])
        for l in range(CFG["n_layers"]):
            assert np.array_equal(e.read_kv(k, l, 0, 40), kv_before[(k, l)])
    for step in range(9, 20):
        ref = g1.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        for k, e in enumerate(eps):
            t, lg = e.decode_step([k], [hist[step - 1][0][k]], want_logits=True)
            assert t[0] == ref[0][k] and np.array_equal(lg[0], ref[1][k])
    for e in eps:
        e.destroy()
    g.destroy()
    g1.destroy()


@pytest.mark.parametrize("n_seqs,long_ctx", [(1, 1000), (12, 0), (24, 0), (40, 0), (70, 0)])
def test_decode_stack_batches_and_long_context(image, oracle_run, n_seqs, long_ctx):
    """The decode-stack kernel (every layer of the stage in one launch) against the oracle,
    teacher-forced: one sequence whose context crosses several attention splits (merged in
    split order), 12-, 24- and 40-sequence batches (tile widths 16, 32, 64),
    varied prompt lengths; PP = 2 on one GPU so the stage boundary is crossed too.  70 sequences
    exceed the decode stack's 64-token tile: the per-kernel decode path runs instead."""
    W = Weights(CFG)
    lens = [long_ctx] if long_ctx else [1 + (7 * i) % 60 for i in range(n_seqs)]
    prompts = [hsgen.tokens(300 + i, n, CFG["vocab"]) for i, n in enumerate(lens)]
    ids = list(range(n_seqs))
    nb = sum((n + 8 + 15) // 16 for n in lens) + 8
    og = OGroup(CFG, W, pp=1, num_blocks=nb)
    rt, rl = og.prefill(ids, prompts)
    gpus = [dict(device=0, h2d_gbps=50.0, free_bytes=8 << 30)]
    plan = hs.plan_stages(CFG, gpus * 2, 2, 1)
    plan.device[0] = plan.device[1] = 0
    g = hs.Group(CFG, plan, image, num_blocks=nb, max_seqs=max(8, n_seqs), max_tokens=max(256, sum(lens)))
    g.load_stage_async(-1)
    ties = []
    toks, logits = g.prefill(ids, prompts, want_logits=True)
    compare(0, toks, logits, rt, rl, ties)
    for step in range(1, 7):
        t_in = np.asarray(rt)
        rt, rl = og.decode(ids, t_in)
        toks, logits = g.decode_step(ids, t_in, want_logits=True)
        compare(step, toks, logits, rt, rl, ties)
    # every mismatch is an oracle near-tie (checked in compare); bound how many, per sequence
    assert len(ties) <= max(1, n_seqs // 8), ties
    g.destroy()


def test_feedback_after_consolidating_into_a_later_stage(image, oracle_run):
    """Device token feedback survives consolidation into a full-memory stage that is not the
    first one (every full-memory stage receives the sampled tokens in local mode)."""
    prompts, hist, _ = oracle_run
    n = torch.cuda.device_count()
    gpus = [dict(device=d, h2d_gbps=50.0, free_bytes=8 << 30) for d in range(max(n, 2))]
    plan = hs.plan_stages(CFG, gpus, 2, 2)
    plan.device[0] = plan.device[1] = 0
    g = hs.Group(CFG, plan, image, num_blocks=64, max_seqs=8, max_tokens=256)
    g.load_stage_async(-1)
    toks, _ = g.prefill([0, 1], prompts)
    for step in range(1, 5):
        toks, _ = g.decode_step([0, 1])
    g.consolidate(1)
    toks, logits = g.decode_step([0, 1], want_logits=True)   # no in_tokens: device feedback
    assert np.array_equal(toks, hist[5][0]) or np.diff(np.sort(hist[5][1], axis=1)[:, -2:], axis=1).min() < 2 * TOL
    g.destroy()
