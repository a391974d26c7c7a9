"""End-to-end parity of the pipeline-parallel group (C ABI hs_* calls) against the oracle on
BASELINE config 1 (tiny decoder, 32-token prompts, PP=2, greedy decode, consolidation to one
stage, continued to 64 steps), plus the GPU-side invariants: PP=s == PP=1 bitwise
(partition-invariant kernels), consolidated KV / weights bit-exact, readiness gating (poisoned
weights + streamed load), multi-sequence varlen prefill, micro-batched (chunked) prefill,
scale-up against the oracle's scale-up.

Acceptance (BASELINE north star): layer-level teacher forcing (tests/layerwise.py):
every half-layer of every layer, fed the GPU's own input, within one bf16 ulp at the row's scale
of the oracle; the GPU's K/V likewise; logits from the GPU's final hidden state within 2e-2 of the
oracle's head on the same state; greedy tokens equal to the oracle's for >= 64 steps (a fork only
at an oracle near-tie).  The measured errors are written to gpurun_out/parity_*.json."""
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import hsgen  # noqa: E402
import layerwise as LW  # noqa: E402
from oracle.decoder import Group as OGroup, Weights  # noqa: E402

if torch.cuda.is_available():
    from paper_2502_15524_b200 import hs  # noqa: E402

CFG = hsgen.CONFIGS["tiny"]
L = CFG["n_layers"]
ALL = range(L)


@pytest.fixture(scope="module")
def image():
    h = hs.image_layout(CFG)
    img = hs.HostImage(h, 0, h.total_bytes)
    hsgen.image_fill(hsgen.image_header(CFG), hsgen.WEIGHT_SEED, img.ptr, 0, h.total_bytes)
    return img


@pytest.fixture(scope="module")
def W():
    return Weights(CFG)


@pytest.fixture(scope="module")
def oracle_run(W):
    """Oracle: prefill + 72 free-running greedy steps of two 32-token prompts."""
    g = OGroup(CFG, W, pp=1, num_blocks=64)
    prompts = hsgen.prompts(2, 32, CFG["vocab"])
    toks, logits = g.prefill([0, 1], prompts)
    hist = [(np.array(toks), logits)]
    for _ in range(72):
        toks, logits = g.decode([0, 1], toks)
        hist.append((np.array(toks), logits))
    return prompts, hist, g


def make_group(image, pp, devices=None, num_blocks=64, full_memory=1, max_seqs=8, max_tokens=256):
    n = torch.cuda.device_count()
    devices = devices or [0] * pp
    gpus = [dict(device=d, h2d_gbps=50.0, free_bytes=8 << 30) for d in range(max(n, pp))]
    plan = hs.plan_stages(CFG, gpus, pp, full_memory)
    for k in range(pp):  # fake PP: several stages on one GPU
        plan.device[k] = devices[k]
    return hs.Group(CFG, plan, image, num_blocks=num_blocks, max_seqs=max_seqs, max_tokens=max_tokens)


def greedy_matches(seq, hist, what):
    """Free-running GPU tokens == the oracle's greedy tokens, until a fork at an oracle near-tie."""
    for step, a in enumerate(seq):
        if not np.array_equal(a, hist[step][0]):
            top2 = np.sort(hist[step][1], axis=1)[:, -2:]
            assert (top2[:, 1] - top2[:, 0]).min() < 2 * LW.LOGIT_TOL, f"{what}: fork at step {step} without a tie"
            return step
    return len(seq)


@pytest.mark.parametrize("pp", [1, 2])
def test_tiny_layerwise_parity_64_steps(image, W, oracle_run, pp):
    """Config 1: prefill 2 x 32 tokens + 64 greedy decode steps (device token feedback); every
    half-layer of every call against the oracle, logits from the GPU's final hidden state, greedy
    tokens against the oracle's free-running run."""
    prompts, hist, _ = oracle_run
    g = make_group(image, pp)
    g.capture(True)
    g.load_stage_async(-1)
    rec = LW.Recorder(CFG)
    toks, logits = g.prefill([0, 1], prompts, want_logits=True)
    rec.record(g, [0, 1], [32, 32], logits, toks)
    seq = [toks.copy()]
    for _ in range(64):
        toks, logits = g.decode_step([0, 1], want_logits=True)
        rec.record(g, [0, 1], [1, 1], logits, toks)
        seq.append(toks.copy())
    res = {}
    phases = [("prefill", {0: (0, 1), 1: (0, 1)}), ("decode", {0: (1, None), 1: (1, None)})]
    LW.check_layers(CFG, W, rec, g, ALL, phases, res)
    LW.check_heads(CFG, W, rec, res)
    res["greedy_steps_equal"] = greedy_matches(seq, hist, f"pp{pp}")
    res["summary"] = LW.summary(res)
    LW.save(res, f"tiny_pp{pp}")
    assert res["greedy_steps_equal"] >= 16
    g.destroy()


def test_tiny_free_running_greedy_matches_oracle(image, oracle_run):
    """Device-side token feedback (in_tokens = NULL) over 64 greedy steps at PP=2 equals the
    oracle's greedy run (a fork is only accepted at an oracle near-tie)."""
    prompts, hist, _ = oracle_run
    g = make_group(image, 2)
    g.load_stage_async(-1)
    toks, _ = g.prefill([0, 1], prompts)
    seq = [toks.copy()]
    for _ in range(64):
        toks, _ = g.decode_step([0, 1])
        seq.append(toks.copy())
    assert greedy_matches(seq, hist, "free-running") >= 16
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
        kv = [g.read_kv(s, l, 0, 40) for s in (0, 1) for l in range(L)]
        runs.append((out, kv))
        g.destroy()
    for out, kv in runs[1:]:
        for (t0, l0), (t1, l1) in zip(runs[0][0], out):
            assert np.array_equal(t0, t1) and np.array_equal(l0, l1)
        for a, b in zip(runs[0][1], kv):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("pp,target", [(2, 0), (4, 0)])
def test_consolidation_bit_exact_then_decode(image, W, oracle_run, pp, target):
    """Config 1: PP=2, 8 greedy steps, consolidate to stage 0 (weights + KV bit-exact, byte counts
    = the oracle's), continue to 64 steps bitwise equal to PP=1 and layer-level equal to the
    oracle."""
    prompts, hist, _ = oracle_run
    g1 = make_group(image, 1)
    g1.load_stage_async(-1)
    g = make_group(image, pp)
    g.load_stage_async(-1)
    g1.prefill([0, 1], prompts, want_logits=True)
    g.prefill([0, 1], prompts, want_logits=True)
    for step in range(1, 9):
        g1.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        g.decode_step([0, 1], hist[step - 1][0], want_logits=True)
    kv_before = {(s, l): g.read_kv(s, l, 0, 40) for s in (0, 1) for l in range(L)}
    st = g.consolidate(target)
    assert g.info()[0] == 1
    # byte counts equal the oracle's consolidation of the same state (P8)
    og = OGroup(CFG, W, pp=pp, num_blocks=64)
    og.prefill([0, 1], prompts)
    for step in range(1, 9):
        og.decode([0, 1], hist[step - 1][0])
    wb, kvb = og.consolidate(target)
    assert st.weight_bytes == wb and st.kv_bytes == kvb
    # KV bit-exact (gathered blocks placed at their layers)
    for k, v in kv_before.items():
        assert np.array_equal(g.read_kv(k[0], k[1], 0, 40), v)
    # weights bit-exact against the host image
    h = hs.image_layout(CFG)
    w = g.read_weights(target, h.embed_off, h.total_bytes - h.embed_off)
    assert np.array_equal(w, image.buf.numpy()[h.embed_off:])
    # continue decoding alone == unpartitioned run (bitwise), up to 64 steps in total; layer
    # level against the oracle on the consolidated endpoint
    g.capture(True)
    rec = LW.Recorder(CFG)
    for step in range(9, 65):
        a = g.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        b = g1.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), step
        if step < 17:
            rec.record(g, [0, 1], [1, 1], a[1], a[0])
    for sid in (0, 1):  # the recorder's positions start at the consolidated context
        rec.rows[sid] = [(pos + 40, pts) for pos, pts in rec.rows[sid]]
    res = {}
    LW.check_layers(CFG, W, rec, g, ALL, [("after_consolidation", {0: (0, None), 1: (0, None)})], res)
    LW.check_heads(CFG, W, rec, res)
    LW.save(res, f"tiny_consolidate_pp{pp}")
    g.destroy()
    g1.destroy()


def test_readiness_gating_with_poisoned_weights(image, oracle_run):
    """Weights poisoned with bf16 NaN, load issued with tiny chunks, prefill enqueued at once:
    any missing per-layer wait would read NaN weights.  The result is bitwise the result of a
    group whose weights were resident before the call."""
    prompts, hist, _ = oracle_run
    ref = make_group(image, 2)
    ref.load_stage_async(-1)
    ref.load_stats(0)
    ref.load_stats(1)
    rt, rl = ref.prefill([0, 1], prompts, want_logits=True)
    g = make_group(image, 2)
    for k in range(2):
        g.poison(k)
    g.load_stage_async(-1, chunk_bytes=64 << 10)
    toks, logits = g.prefill([0, 1], prompts, want_logits=True)
    assert np.isfinite(logits).all()
    assert np.array_equal(toks, rt) and np.array_equal(logits, rl)
    s = g.load_stats(0)
    assert s.done == 1 and s.layers_ready == 2
    g.destroy()
    ref.destroy()


def test_varlen_multi_sequence_prefill(image, W):
    """Packed prefill of 4 prompts of lengths 5, 17, 33, 1 (ragged, one single-token prompt):
    layer-level parity of every sequence, then release."""
    prompts = [hsgen.tokens(100 + i, n, CFG["vocab"]) for i, n in enumerate((5, 17, 33, 1))]
    g = make_group(image, 2)
    g.capture(True)
    g.load_stage_async(-1)
    ids = [10, 11, 12, 13]
    toks, logits = g.prefill(ids, prompts, want_logits=True)
    rec = LW.Recorder(CFG)
    rec.record(g, ids, [len(p) for p in prompts], logits, toks)
    res = {}
    LW.check_layers(CFG, W, rec, g, ALL, [("prefill", {i: (0, 1) for i in ids})], res)
    LW.check_heads(CFG, W, rec, res)
    LW.save(res, "tiny_varlen")
    for sid in ids:
        g.release_seq(sid)
    with pytest.raises(hs.HsError):
        g.decode_step([10])
    g.destroy()


_CHUNKED_REF = {}


@pytest.mark.parametrize("resident", [True, False])
def test_chunked_prefill_layerwise(image, W, resident):
    """Micro-batched prefill (prefill half): 4 sequences of 96-160 tokens cut
    into 4 chunks (chunk c attends to the cached KV of chunks < c), through PP=2.  resident=False:
    the stages' weights are still streaming in (64 KiB chunks after a poison), so the first stage
    runs layer-major; resident=True: chunk-major.  Both layer-level equal to the oracle and
    bitwise equal to each other; the unchunked call (max_chunks = 1) also passes the oracle check
    and gives the same tokens."""
    lens = (96, 160, 128, 112)
    prompts = [hsgen.tokens(500 + i, n, CFG["vocab"]) for i, n in enumerate(lens)]
    ids = [0, 1, 2, 3]
    outs = {}
    for mode in ("chunked", "unchunked"):
        g = make_group(image, 2, num_blocks=128, max_tokens=512)
        if mode == "chunked":
            g.set_prefill_chunking(min_chunk_tokens=64, max_chunks=4)
        else:
            g.set_prefill_chunking(max_chunks=1)
        g.capture(True)
        if not resident:
            g.poison(0)
            g.poison(1)
            g.load_stage_async(-1, chunk_bytes=64 << 10)
        else:
            g.load_stage_async(-1)
            g.load_stats(0)
            g.load_stats(1)
        toks, logits = g.prefill(ids, prompts, want_logits=True)
        rec = LW.Recorder(CFG)
        rec.record(g, ids, list(lens), logits, toks)
        res = {}
        LW.check_layers(CFG, W, rec, g, ALL, [("prefill", {i: (0, 1) for i in ids})], res)
        LW.check_heads(CFG, W, rec, res)
        LW.save(res, f"tiny_{mode}_prefill_{'resident' if resident else 'streaming'}")
        kv = [g.read_kv(s, l, 0, lens[s]) for s in ids for l in range(L)]
        outs[mode] = (toks, logits, kv)
        g.destroy()
    assert np.array_equal(outs["chunked"][0], outs["unchunked"][0])
    if resident:
        _CHUNKED_REF["resident"] = outs["chunked"]
    elif "resident" in _CHUNKED_REF:  # layer-major == chunk-major, bit for bit
        a, b = _CHUNKED_REF["resident"], outs["chunked"]
        assert np.array_equal(a[1], b[1]) and all(np.array_equal(x, y) for x, y in zip(a[2], b[2]))


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
    with pytest.raises(hs.HsError) as e:
        g.read_hidden(0, 0, 1)  # capture off
    assert e.value.code == 5
    g.destroy()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_two_gpu_pipeline_and_consolidation(image, oracle_run):
    """Stages on two GPUs (NVLink hand-off): bitwise equal to PP=1 on one GPU, before and after
    consolidation."""
    prompts, hist, _ = oracle_run
    g1 = make_group(image, 1)
    g1.load_stage_async(-1)
    g = make_group(image, 2, devices=[0, 1])
    g.load_stage_async(-1)
    a, b = g.prefill([0, 1], prompts, want_logits=True), g1.prefill([0, 1], prompts, want_logits=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    for step in range(1, 9):
        a = g.decode_step([0, 1], None, want_logits=True)
        b = g1.decode_step([0, 1], None, want_logits=True)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    g.consolidate(0)
    for step in range(9, 20):
        a = g.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        b = g1.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    g.destroy()
    g1.destroy()


@pytest.mark.parametrize("pp", [2, 4])
def test_background_host_load_then_kv_only_consolidation(image, oracle_run, pp):
    """the target loads the other stages' layers over its own host link in
    the background while the group decodes pipelined; consolidation then moves only KV.  Every
    step bitwise equal to PP=1."""
    prompts, hist, _ = oracle_run
    g1 = make_group(image, 1)
    g1.load_stage_async(-1)
    g = make_group(image, pp)
    g.load_stage_async(-1)
    g.prefill([0, 1], prompts)
    g1.prefill([0, 1], prompts)
    g.load_background_async(0)
    for step in range(1, 9):
        a = g.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        b = g1.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    kv_before = {(s, l): g.read_kv(s, l, 0, 40) for s in (0, 1) for l in range(L)}
    st = g.consolidate(0)
    sb = hs.plan_stages(CFG, [dict(device=d, h2d_gbps=50.0, free_bytes=8 << 30) for d in range(pp)], pp, 1).as_dict()["stage_bytes"]
    assert st.weight_bytes == 0 and st.weight_bytes_host == sum(sb) - sb[0] and st.kv_bytes > 0
    for k, v in kv_before.items():
        assert np.array_equal(g.read_kv(k[0], k[1], 0, 40), v)
    h = hs.image_layout(CFG)
    assert np.array_equal(g.read_weights(0, h.embed_off, h.total_bytes - h.embed_off), image.buf.numpy()[h.embed_off:])
    for step in range(9, 20):
        a = g.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        b = g1.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    g.destroy()
    g1.destroy()


@pytest.mark.parametrize("pp", [2, 4])
def test_scale_up_against_the_oracle(image, W, pp):
    """PP=pp with every stage full-memory; after 8 steps
    every stage becomes a standalone endpoint holding the whole model and the KV of the sequences
    assigned to it.  Against the oracle's scale-up of the same state: migrated byte counts equal,
    each endpoint's KV equal to the pre-scale-up KV bit for bit, then 12 steps on each endpoint
    layer-level equal to the oracle's endpoint, greedy tokens equal (teacher-forced on the
    oracle endpoints' tokens, a mismatch only at a near-tie)."""
    prompts = hsgen.prompts(3, 32, CFG["vocab"])
    ids = [0, 1, 2]
    owner = [0, pp - 1, 1]
    g = make_group(image, pp, full_memory=pp)
    g.load_stage_async(-1)
    og = OGroup(CFG, W, pp=pp, num_blocks=64)
    g.prefill(ids, prompts)
    ot, _ = og.prefill(ids, prompts)
    for step in range(8):
        g.decode_step(ids, ot)
        ot, _ = og.decode(ids, ot)
    kv_before = {(s, l): g.read_kv(s, l, 0, 40) for s in ids for l in range(L)}
    eps, st = g.scale_up(owner)
    oeps, wb, kvb = og.scale_up(dict(zip(ids, owner)))
    assert len(eps) == pp and st.weight_bytes == wb and st.kv_bytes == kvb
    h = hs.image_layout(CFG)
    for e in eps:
        assert e.info()[0] == 1
        assert np.array_equal(e.read_weights(0, h.embed_off, h.total_bytes - h.embed_off), image.buf.numpy()[h.embed_off:])
    for s in ids:
        for l in range(L):
            assert np.array_equal(eps[owner[s]].read_kv(s, l, 0, 40), kv_before[(s, l)])
    res = {}
    for k, e in enumerate(eps):
        mine = [s for s in ids if owner[s] == k]
        if not mine:
            continue
        e.capture(True)
        rec = LW.Recorder(CFG)
        tin = [ot[s] for s in mine]
        for step in range(12):
            t, lg = e.decode_step(mine, tin, want_logits=True)
            rec.record(e, mine, [1] * len(mine), lg, t)
            tin, _ = oeps[k].decode(mine, tin)
            for i in range(len(mine)):  # same greedy token as the oracle endpoint, or a near-tie
                if t[i] != tin[i]:
                    top2 = np.sort(lg[i])[-2:]
                    assert top2[1] - top2[0] < 2 * LW.LOGIT_TOL
        for s in mine:
            rec.rows[s] = [(pos + 40, pts) for pos, pts in rec.rows[s]]
        LW.check_layers(CFG, W, rec, e, ALL, [("endpoint", {s: (0, None) for s in mine})], res, tag=f"ep{k}.")
        LW.check_heads(CFG, W, rec, res, tag=f"ep{k}.")
    LW.save(res, f"tiny_scale_up_pp{pp}")
    for e in eps:
        e.destroy()
    g.destroy()


@pytest.mark.parametrize("n_seqs,long_ctx", [(1, 1000), (12, 0), (24, 0), (40, 0), (70, 0)])
def test_decode_stack_batches_and_long_context(image, W, n_seqs, long_ctx):
    """The decode-stack kernel (every layer of the stage in one launch), layer-level against the
    oracle: one sequence whose context crosses several attention splits (merged in split order),
    12-, 24- and 40-sequence batches (tile widths 16, 32, 64), varied prompt lengths; PP = 2 on
    one GPU so the stage boundary is crossed too.  70 sequences exceed the decode stack's
    64-token tile: the per-kernel decode path runs instead."""
    lens = [long_ctx] if long_ctx else [1 + (7 * i) % 60 for i in range(n_seqs)]
    prompts = [hsgen.tokens(300 + i, n, CFG["vocab"]) for i, n in enumerate(lens)]
    ids = list(range(n_seqs))
    nb = sum((n + 8 + 15) // 16 for n in lens) + 8
    gpus = [dict(device=0, h2d_gbps=50.0, free_bytes=8 << 30)]
    plan = hs.plan_stages(CFG, gpus * 2, 2, 1)
    plan.device[0] = plan.device[1] = 0
    g = hs.Group(CFG, plan, image, num_blocks=nb, max_seqs=max(8, n_seqs), max_tokens=max(256, sum(lens)))
    g.load_stage_async(-1)
    g.prefill(ids, prompts)
    g.capture(True)
    rec = LW.Recorder(CFG)
    for step in range(6):
        toks, logits = g.decode_step(ids, None, want_logits=True)
        rec.record(g, ids, [1] * n_seqs, logits, toks)
    for s, n in zip(ids, lens):
        rec.rows[s] = [(pos + n, pts) for pos, pts in rec.rows[s]]
    res = {}
    LW.check_layers(CFG, W, rec, g, ALL, [("decode", {s: (0, None) for s in ids})], res)
    LW.check_heads(CFG, W, rec, res)
    LW.save(res, f"tiny_decode_b{n_seqs}_ctx{long_ctx}")
    g.destroy()


def test_feedback_after_consolidating_into_a_later_stage(image, oracle_run):
    """Device token feedback survives consolidation into a full-memory stage that is not the
    first one (every full-memory stage receives the sampled tokens in local mode): bitwise equal
    to the same run on PP=1."""
    prompts, hist, _ = oracle_run
    g1 = make_group(image, 1)
    g1.load_stage_async(-1)
    g = make_group(image, 2, full_memory=2)
    g.load_stage_async(-1)
    g.prefill([0, 1], prompts)
    g1.prefill([0, 1], prompts)
    for step in range(1, 5):
        g.decode_step([0, 1])
        g1.decode_step([0, 1])
    g.consolidate(1)
    a = g.decode_step([0, 1], want_logits=True)   # no in_tokens: device feedback
    b = g1.decode_step([0, 1], want_logits=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    g.destroy()
    g1.destroy()


def test_prefetch_watermark_gates_load_and_prefill(image, oracle_run, tmp_path):
    """the model file is streamed into pinned memory by
    the prefetcher at a throttled rate (256 KiB pieces, 50 MB/s) while the loader, issued at once,
    gates every H2D chunk on the 8-byte fetched-end watermark (cuStreamWaitValue64 on the copy
    stream) and the prefill gates its host-image embedding reads the same way.  Unfetched bytes
    are bf16 NaN (0xFF) and the device weights are poisoned: any chunk copied or row read before
    its fetch would show up.  The result equals the resident-image run bit for bit, and the first
    token cannot arrive before the prefetcher has fetched what the prefill needs."""
    prompts, hist, _ = oracle_run
    h = hs.image_layout(CFG)
    path = tmp_path / "tiny.hsimg"
    image.buf.numpy().tofile(path)  # the model file: the host image's bytes, header first
    ref = make_group(image, 2)
    ref.load_stage_async(-1)
    ref.load_stats(0)
    ref.load_stats(1)
    rt, rl = ref.prefill([0, 1], prompts, want_logits=True)
    img = hs.HostImage(h, 0, h.total_bytes)
    img.buf.fill_(0xFF)
    pf = img.prefetch_from(str(path), chunk_bytes=256 << 10, max_gbps=0.05)
    t0 = time.perf_counter()
    g = make_group(img, 2)
    g.poison(0)
    g.poison(1)
    g.load_stage_async(-1, chunk_bytes=64 << 10)
    toks, logits = g.prefill([0, 1], prompts, want_logits=True)
    t1 = time.perf_counter()
    n, secs = pf.wait()
    assert n == h.total_bytes
    assert np.array_equal(toks, rt) and np.array_equal(logits, rl)
    # the last stage's slice ends the file: its last chunk cannot be copied before the fetch ends
    assert t1 - t0 >= 0.8 * secs, (t1 - t0, secs)
    s1 = g.load_stats(1)
    assert s1.done == 1 and s1.load_ms >= 0.5 * 1e3 * secs * (h.total_bytes - g.plan.as_dict()["slices"][1][0]) / h.total_bytes
    g.destroy()
    ref.destroy()
    pf.destroy()


@pytest.mark.parametrize("pp,n,m", [(1, 8, 2), (2, 8, 2), (4, 16, 4), (2, 6, 2)])
def test_decode_steps_micro_batched_equals_stepwise(image, pp, n, m):
    """SURVEY §8(f) row 4 (decode half): hs_decode_steps runs the batch as m micro-batches
    ("virtual engines") through the stages with device feedback.  Per sequence it is bitwise
    equal to n stepwise hs_decode_step calls (tokens of every step, the KV of every layer and
    position), and device feedback continues across the two APIs."""
    lens = [5 + 3 * i for i in range(n)]
    prompts = [hsgen.tokens(700 + i, k, CFG["vocab"]) for i, k in enumerate(lens)]
    ids = list(range(n))
    ga = make_group(image, pp, num_blocks=96, max_seqs=n, max_tokens=512)
    gb = make_group(image, pp, num_blocks=96, max_seqs=n, max_tokens=512)
    for g in (ga, gb):
        g.load_stage_async(-1)
        g.prefill(ids, prompts)
    toks = ga.decode_steps(ids, 8, n_micro=m)
    ref = np.stack([gb.decode_step(ids)[0] for _ in range(8)])
    assert np.array_equal(toks, ref)
    for s, k in zip(ids, lens):
        for l in range(L):
            assert np.array_equal(ga.read_kv(s, l, 0, k + 8), gb.read_kv(s, l, 0, k + 8))
    a, b = ga.decode_step(ids, want_logits=True), gb.decode_step(ids, want_logits=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    toks2 = ga.decode_steps(ids, 3, n_micro=m, in_tokens=a[0])
    ref2 = np.stack([gb.decode_step(ids, a[0] if i == 0 else None)[0] for i in range(3)])
    assert np.array_equal(toks2, ref2)
    ga.destroy()
    gb.destroy()


@pytest.mark.parametrize("pp", [2, 4])
def test_background_nvlink_pull_then_kv_only_consolidation(image, oracle_run, pp):
    """PAPER.md:602 with the other stages' HBM as the source: the full-memory target pulls every
    other stage's weight slice over NVLink (copy engines, low-priority stream) while the group
    decodes pipelined (bitwise equal to PP=1 throughout); consolidation then moves only KV and
    the target's weights equal the host image."""
    prompts, hist, _ = oracle_run
    g1 = make_group(image, 1)
    g1.load_stage_async(-1)
    g = make_group(image, pp)
    g.load_stage_async(-1)
    with pytest.raises(hs.HsError) as e:  # before any call: the sources may still be loading
        g.pull_background_async(0)
    assert e.value.code == 5
    g.prefill([0, 1], prompts)
    g1.prefill([0, 1], prompts)
    g.pull_background_async(0, chunk_bytes=256 << 10)
    for step in range(1, 9):
        a = g.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        b = g1.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    kv_before = {(s_, l): g.read_kv(s_, l, 0, 40) for s_ in (0, 1) for l in range(L)}
    st = g.consolidate(0)
    sb = hs.plan_stages(CFG, [dict(device=d, h2d_gbps=50.0, free_bytes=8 << 30) for d in range(pp)], pp, 1).as_dict()["stage_bytes"]
    assert st.weight_bytes == 0 and st.weight_bytes_background == sum(sb) - sb[0] and st.kv_bytes > 0
    for k, v in kv_before.items():
        assert np.array_equal(g.read_kv(k[0], k[1], 0, 40), v)
    h = hs.image_layout(CFG)
    assert np.array_equal(g.read_weights(0, h.embed_off, h.total_bytes - h.embed_off), image.buf.numpy()[h.embed_off:])
    for step in range(9, 20):
        a = g.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        b = g1.decode_step([0, 1], hist[step - 1][0], want_logits=True)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    g.destroy()
    g1.destroy()


@pytest.mark.parametrize("pp", [1, 2])
def test_decode_stack_state_zeroed_in_stream_order(image, pp):
    """Regression (run 42, DESIGN.md §7.1 "Intermittent decode traps"): the decode stack's state
    is created at a group's first decode step and its counters must be zeroed in the order of
    the stage's stream.  Here the legacy default stream is kept busy (torch.cuda._sleep) across
    the first decode steps, so a legacy-stream memset would land behind the sleep, after the
    first launches had counted, and trap a later step.  Every step must equal a reference
    group's, and the steps must outlast the sleep (else the window was not covered)."""
    prompts = hsgen.prompts(2, 32, CFG["vocab"])
    n_max = 600
    ref = make_group(image, pp, num_blocks=128)
    ref.load_stage_async(-1)
    ref.prefill([0, 1], prompts)
    want = [ref.decode_step([0, 1])[0] for _ in range(n_max)]
    ref.destroy()
    g = make_group(image, pp, num_blocks=128)
    g.load_stage_async(-1)
    g.prefill([0, 1], prompts)
    torch.cuda.synchronize()
    sleep_s = 0.03
    t0 = time.time()
    torch.cuda._sleep(int(sleep_s * 2.0e9))  # ~30 ms of SM cycles on the legacy default stream
    got = []
    while len(got) < n_max and (len(got) < 50 or time.time() - t0 < 4 * sleep_s):
        got.append(g.decode_step([0, 1])[0])
    covered = time.time() - t0
    torch.cuda.synchronize()
    g.destroy()
    assert covered > 2 * sleep_s, f"decode steps ended after {covered:.3f} s, inside the sleep window"
    for i, a in enumerate(got):
        assert np.array_equal(a, want[i]), f"step {i}"
