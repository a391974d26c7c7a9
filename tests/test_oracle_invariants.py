"""Invariants the paper fixes, checked on the oracle in its bf16 mode (SURVEY §8(c) pins):
  P3  PP-split == unsplit, bitwise
  P4  consolidated KV == single-worker KV, bitwise; later decode identical
  P5  cached decode == full recompute
  P6  brute-force dense model (no paging, no packing, recompute per step) agrees
  P8  migration byte counts = sum_seq ceil(ctx/16)*16 * kv_bytes/token * |moved layers| and
      weight bytes = model - target slice (SPEC.md:321 formula, exact counts)
"""
import numpy as np
import pytest

import hsgen
from oracle.decoder import (BLOCK, Group, Weights, embed_param_bytes, final_param_bytes,
                            layer_param_bytes)
from oracle.numerics import (bf16, linear, rmsnorm, rope, rope_cos_sin, silu)


@pytest.fixture(scope="module")
def W(tiny_cfg):
    return Weights(tiny_cfg)


def run(cfg, W, pp, prompts, steps, ranges=None):
    g = Group(cfg, W, pp=pp, ranges=ranges, num_blocks=64)
    ids = list(range(len(prompts)))
    toks, logits = g.prefill(ids, prompts)
    hist = [(list(toks), logits)]
    for _ in range(steps):
        toks, logits = g.decode(ids, toks)
        hist.append((list(toks), logits))
    return g, hist


def test_pp_split_equals_unsplit_bitwise(tiny_cfg, W):
    prompts = hsgen.prompts(2, 32, tiny_cfg["vocab"])
    g1, h1 = run(tiny_cfg, W, 1, prompts, 4)
    for pp, ranges in ((2, None), (4, None), (3, [(0, 1), (1, 3), (3, 4)])):
        g, h = run(tiny_cfg, W, pp, prompts, 4, ranges)
        for (t1, l1), (t, l) in zip(h1, h):
            assert t1 == t and np.array_equal(l1, l)
        for seq in (0, 1):
            for layer in range(tiny_cfg["n_layers"]):
                assert np.array_equal(g.read_kv(seq, layer, 0, 37), g1.read_kv(seq, layer, 0, 37))
    # hand-off bytes: 2H per token per boundary ("8 KB ... per token" for H=4096)
    g2, _ = run(tiny_cfg, W, 2, prompts, 0)
    assert g2.handoff_bytes == 64 * tiny_cfg["hidden"] * 2


def test_packed_varlen_equals_separate(tiny_cfg, W):
    prompts = [hsgen.tokens(5, 19, tiny_cfg["vocab"]), hsgen.tokens(6, 33, tiny_cfg["vocab"])]
    g = Group(tiny_cfg, W, pp=2, num_blocks=64)
    toks, logits = g.prefill([10, 11], prompts)
    for i, p in enumerate(prompts):
        gi = Group(tiny_cfg, W, pp=1, num_blocks=64)
        ti, li = gi.prefill([0], [p])
        assert ti[0] == toks[i] and np.array_equal(li[0], logits[i])


def test_cached_decode_equals_recompute(tiny_cfg, W):
    prompt = list(hsgen.tokens(8, 21, tiny_cfg["vocab"]))
    g = Group(tiny_cfg, W, pp=2, num_blocks=64)
    toks, _ = g.prefill([0], [prompt])
    seq = prompt + [toks[0]]
    for _ in range(5):
        toks, logits = g.decode([0], toks)
        fresh = Group(tiny_cfg, W, pp=1, num_blocks=64)
        t2, l2 = fresh.prefill([0], [seq])
        assert t2[0] == toks[0]
        assert np.array_equal(l2[0], logits[0])
        seq.append(toks[0])


def brute_force_logits(cfg, W, seq):
    """Independent dense implementation: whole sequence recomputed, no cache, no paging,
    no packing; same rounding points (DESIGN.md numerics contract)."""
    T, H, nh, d = len(seq), cfg["hidden"], cfg["n_heads"], cfg["head_dim"]
    x = W.embed_rows(seq)
    c, s = rope_cos_sin(np.arange(T), d, cfg["rope_theta"])
    for l in range(cfg["n_layers"]):
        w = W.layer(l)
        # RMSNorm feeding a linear layer: operand bf16(x * w), row scale r after the product (R10b)
        r = 1.0 / np.sqrt(np.mean(x * x, axis=1, keepdims=True) + cfg["rms_eps"])
        n = bf16(x * w["attn_norm"])
        q = rope(bf16(r * linear(n, w["wq"])).reshape(T, nh, d), c, s)
        k = rope(bf16(r * linear(n, w["wk"])).reshape(T, nh, d), c, s)
        v = bf16(r * linear(n, w["wv"])).reshape(T, nh, d)
        o = np.zeros((T, nh, d))
        for hh in range(nh):
            S = q[:, hh] @ k[:, hh].T / np.sqrt(d)
            S[np.triu_indices(T, 1)] = -np.inf
            P = np.exp(S - S.max(axis=1, keepdims=True))
            o[:, hh] = bf16((P @ v[:, hh]) / P.sum(axis=1, keepdims=True))
        h = bf16(x + linear(o.reshape(T, H), w["wo"]))
        r2 = 1.0 / np.sqrt(np.mean(h * h, axis=1, keepdims=True) + cfg["rms_eps"])
        n2 = bf16(h * w["ffn_norm"])
        x = bf16(h + linear(bf16(silu(r2 * linear(n2, w["wg"])) * (r2 * linear(n2, w["wu"]))), w["wd"]))
    nf = rmsnorm(x[-1:], W.final_norm(), cfg["rms_eps"])
    return linear(nf, W.lm_head())[0]


def test_brute_force_dense(tiny_cfg, W):
    prompt = list(hsgen.tokens(3, 17, tiny_cfg["vocab"]))
    g = Group(tiny_cfg, W, pp=2, num_blocks=64)
    toks, logits = g.prefill([0], [prompt])
    seq = prompt
    for step in range(4):
        ref = brute_force_logits(tiny_cfg, W, seq)
        assert np.allclose(logits[0], ref, rtol=0, atol=1e-9)
        assert toks[0] == int(np.argmax(ref))
        seq = seq + [toks[0]]
        toks, logits = g.decode([0], toks)


@pytest.mark.parametrize("pp,target", [(2, 0), (4, 0), (4, 2)])
def test_consolidation_bitwise_and_bytes(tiny_cfg, W, pp, target):
    cfg = tiny_cfg
    prompts = hsgen.prompts(3, 32, cfg["vocab"])
    g1, h1 = run(cfg, W, 1, prompts, 12)
    g = Group(cfg, W, pp=pp, num_blocks=64)
    ids = [0, 1, 2]
    toks, _ = g.prefill(ids, prompts)
    for _ in range(8):
        toks, _ = g.decode(ids, toks)
    tgt_layers = set(g.workers[target].layers)
    wb, kvb = g.consolidate(target)
    moved = cfg["n_layers"] - len(tgt_layers)
    ctx = 32 + 8
    assert kvb == 3 * ((ctx + BLOCK - 1) // BLOCK) * BLOCK * (2 * cfg["hidden"] * 2) * moved
    expect_w = moved * layer_param_bytes(cfg) + (embed_param_bytes(cfg) if target != 0 else 0) \
        + (final_param_bytes(cfg) if target != pp - 1 else 0)
    assert wb == expect_w
    assert len(g.workers) == 1 and g.workers[0].layers == list(range(cfg["n_layers"]))
    for seq in ids:
        for layer in range(cfg["n_layers"]):
            assert np.array_equal(g.read_kv(seq, layer, 0, ctx), g1.read_kv(seq, layer, 0, ctx))
    for step in range(4):  # continue decoding alone == unpartitioned decode
        toks, logits = g.decode(ids, toks)
        t1, l1 = h1[9 + step]
        assert toks == t1 and np.array_equal(logits, l1)


def test_config4_kv_bytes_formula():
    """13B PP4 -> stage 0, 16 seqs at ctx 576 -> 5,662,310,400 B."""
    cfg = hsgen.CONFIGS["llama2-13b"]
    kv_per_block = BLOCK * 2 * cfg["hidden"] * 2
    assert 16 * (576 // BLOCK) * kv_per_block * 30 == 5_662_310_400


@pytest.mark.parametrize("pp", [2, 4])
def test_scale_up_endpoints_bitwise_and_bytes(tiny_cfg, W, pp):
    """Scale-up: after 8 pipelined steps every worker becomes an endpoint;
    each sequence then decodes on its endpoint bitwise equal to the unpartitioned run (its KV of
    every layer is the single-worker KV); bytes: each endpoint receives the
    model minus its own slice ((s-1) x model in total) and, for every layer it lacked, the used
    blocks of its own sequences."""
    cfg = tiny_cfg
    prompts = hsgen.prompts(3, 32, cfg["vocab"])
    g1, h1 = run(cfg, W, 1, prompts, 12)
    g = Group(cfg, W, pp=pp, num_blocks=64)
    ids = [0, 1, 2]
    toks, _ = g.prefill(ids, prompts)
    for _ in range(8):
        toks, _ = g.decode(ids, toks)
    layers_of = [list(wk.layers) for wk in g.workers]
    owner = {0: 0, 1: pp - 1, 2: 1}
    eps, wb, kvb = g.scale_up(owner)
    model = cfg["n_layers"] * layer_param_bytes(cfg) + embed_param_bytes(cfg) + final_param_bytes(cfg)
    assert wb == (pp - 1) * model
    ctx = 32 + 8
    blocks = (ctx + BLOCK - 1) // BLOCK
    assert kvb == sum(blocks * BLOCK * 2 * cfg["hidden"] * 2 * (cfg["n_layers"] - len(layers_of[owner[s]])) for s in ids)
    assert len(eps) == pp
    for s in ids:
        e = eps[owner[s]]
        assert sorted(e.bm.tables) == sorted(x for x in ids if owner[x] == owner[s])
        for layer in range(cfg["n_layers"]):
            assert np.array_equal(e.read_kv(s, layer, 0, ctx), g1.read_kv(s, layer, 0, ctx))
    for step in range(4):  # each endpoint continues its sequences == the unpartitioned run
        t1, l1 = h1[9 + step]
        for s in ids:
            e = eps[owner[s]]
            t, lg = e.decode([s], [toks[s]])
            assert t[0] == t1[s] and np.array_equal(lg[0], l1[s])
        toks = list(t1)
