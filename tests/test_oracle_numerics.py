"""Pins of oracle/numerics.py against things other than itself: known bit patterns, torch's
own bf16 cast, torch fp64 library routines, and closed forms (SURVEY §8(c) pins P6, P7)."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle.numerics import (attention_one, bf16, bf16_bits, bf16_value, exact, linear, rmsnorm, rmsnorm_split, rope,
                             rope_cos_sin, silu)


def test_bf16_known_patterns():
    vals = np.array([1.0, 1 + 2**-8, 1 + 3 * 2**-8, -0.0, np.inf, -np.inf, 2**-133, 65504.0, 3.0e38])
    want = [0x3F80, 0x3F80, 0x3F82, 0x8000, 0x7F80, 0xFF80, 0x0001, 0x4780, 0x7F62]
    assert [int(b) for b in bf16_bits(vals)] == want
    assert np.isnan(bf16_value(bf16_bits(np.nan)))


def test_bf16_matches_torch_cast():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(100000) * 10.0 ** rng.integers(-30, 30, 100000),
                        rng.standard_normal(1000)]).astype(np.float32)
    t = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(bf16_bits(x), t)


def test_rmsnorm_vs_torch_and_closed_form():
    rng = np.random.default_rng(1)
    x, w = rng.standard_normal((7, 64)), 1 + 0.1 * rng.standard_normal(64)
    ref = F.rms_norm(torch.from_numpy(x), (64,), torch.from_numpy(w), eps=1e-5).numpy()
    assert np.allclose(rmsnorm(x, w, 1e-5, exact), ref, rtol=1e-13, atol=1e-13)
    # RMSNorm(c * 1) = sign(c) * w when c^2 >> eps (rounded once)
    for c in (3.0, -250.0):
        y = rmsnorm(np.full((1, 64), c), w, 1e-5)
        assert np.array_equal(y[0], bf16(np.sign(c) * w * (abs(c) / np.sqrt(c * c + 1e-5))))
        assert np.allclose(y[0], np.sign(c) * bf16(w), rtol=2**-7)


def test_rmsnorm_split_vs_torch_norm_then_linear():
    """R10b: the RMSNorm feeding a linear layer as r * ((x * w) W^T).  Exact mode equals torch's
    rms_norm followed by the matmul (an independent library path); bf16 mode rounds only the
    operand x * w; constant rows give r = 1/sqrt(c^2 + eps) in closed form."""
    rng = np.random.default_rng(11)
    x, w, W = rng.standard_normal((5, 64)), 1 + 0.1 * rng.standard_normal(64), rng.standard_normal((24, 64))
    a, r = rmsnorm_split(x, w, 1e-5, exact)
    ref = F.rms_norm(torch.from_numpy(x), (64,), torch.from_numpy(w), eps=1e-5) @ torch.from_numpy(W).T
    assert np.allclose(r * linear(a, W), ref.numpy(), rtol=1e-12, atol=1e-12)
    xb, wb = bf16(x), bf16(w)
    a, r = rmsnorm_split(xb, wb, 1e-5)
    assert np.array_equal(a, bf16(xb * wb))
    assert np.array_equal(r[:, 0], 1.0 / np.sqrt(np.mean(xb * xb, axis=1) + 1e-5))
    for c in (3.0, -250.0):
        _, r = rmsnorm_split(np.full((1, 64), c), w, 1e-5)
        assert r[0, 0] == 1.0 / np.sqrt(c * c + 1e-5)


def test_rope_identity_norm_and_complex_form():
    rng = np.random.default_rng(2)
    d, T = 64, 9
    x = rng.standard_normal((T, 3, d))
    pos = np.arange(T) * 37
    c, s = rope_cos_sin(pos, d, 1e4, table_f32=False)
    y = rope(x, c, s, exact)
    # position 0 is the identity
    assert np.allclose(y[0], x[0], atol=0)
    # each (i, i + d/2) pair keeps its norm
    h = d // 2
    assert np.allclose(x[..., :h] ** 2 + x[..., h:] ** 2, y[..., :h] ** 2 + y[..., h:] ** 2, rtol=1e-12)
    # complex form: (x_i + j x_{i+d/2}) * exp(j p theta^(-2i/d))
    z = (x[..., :h] + 1j * x[..., h:]) * np.exp(1j * pos[:, None, None] * 1e4 ** (-2 * np.arange(h) / d))
    assert np.allclose(y[..., :h], z.real, atol=1e-12) and np.allclose(y[..., h:], z.imag, atol=1e-12)
    # relative-position property: <rope(q,p), rope(k,p')> depends on p - p' only
    q, k = rng.standard_normal((1, 1, d)), rng.standard_normal((1, 1, d))
    def dot(p, pp):
        c1, s1 = rope_cos_sin(np.array([p]), d, 1e4, False)
        c2, s2 = rope_cos_sin(np.array([pp]), d, 1e4, False)
        return float((rope(q, c1, s1, exact) * rope(k, c2, s2, exact)).sum())
    assert abs(dot(10, 3) - dot(107, 100)) < 1e-9


def test_attention_closed_forms_and_sdpa():
    rng = np.random.default_rng(3)
    nh, d = 2, 16
    q = rng.standard_normal((nh, d))
    v = rng.standard_normal((1, nh, d))
    # one key -> exactly v (rounded)
    assert np.array_equal(attention_one(q, rng.standard_normal((1, nh, d)), v), bf16(v[0]))
    # identical keys -> mean of v
    K = np.repeat(rng.standard_normal((1, nh, d)), 5, axis=0)
    V = rng.standard_normal((5, nh, d))
    assert np.allclose(attention_one(q, K, V, exact), V.mean(axis=0), rtol=1e-12)
    # shift invariance of softmax: adding a constant to all scores (via q . k shift) is neutral
    # and a causal sequence matches torch fp64 SDPA
    T = 11
    Q, Kk, Vv = (rng.standard_normal((T, nh, d)) for _ in range(3))
    ours = np.stack([attention_one(Q[t], Kk[: t + 1], Vv[: t + 1], exact) for t in range(T)])
    ref = F.scaled_dot_product_attention(torch.from_numpy(Q).transpose(0, 1), torch.from_numpy(Kk).transpose(0, 1),
                                         torch.from_numpy(Vv).transpose(0, 1), is_causal=True)
    assert np.allclose(ours, ref.transpose(0, 1).numpy(), rtol=1e-11, atol=1e-12)


def test_silu():
    g = np.linspace(-20, 20, 401)
    assert silu(np.array([0.0]))[0] == 0.0
    assert np.allclose(silu(g), F.silu(torch.from_numpy(g)).numpy(), rtol=1e-14, atol=1e-300)


def test_argmax_lowest_tie_semantics():
    """Greedy ties go to the lowest token id (R11, torch.argmax semantics)."""
    from oracle.numerics import argmax_lowest
    assert argmax_lowest(np.array([0.5, 2.0, 2.0, -1.0])) == 1
    assert argmax_lowest(np.array([3.0, 3.0, 3.0])) == 0
    assert argmax_lowest(np.array([-np.inf, -1.0, -1.0])) == 1
    v = np.zeros(1024)
    v[[7, 300, 1023]] = 5.0
    assert argmax_lowest(v) == 7


def test_decoder_paged_attention_equals_attention_one():
    """The decoder's bf16 paged attention (rows read back through a non-contiguous block table,
    causal over a packed 2-sequence batch) equals oracle.numerics.attention_one (pinned against
    torch SDPA in this file) applied query by query to the same k', v."""
    import hsgen
    from oracle.decoder import BLOCK, Weights, Worker
    from oracle.numerics import attention_one
    cfg = hsgen.CONFIGS["tiny"]
    W = Weights(cfg)
    wk = Worker(cfg, W, 1, 2, num_blocks=16)
    rng = np.random.default_rng(3)
    x = bf16(rng.standard_normal((40 + 23, cfg["hidden"])))
    tabs = [[9, 2, 14], [5, 0]]
    batch = []
    for sid, (n, tab) in enumerate(((40, tabs[0]), (23, tabs[1]))):
        pos = np.arange(n)
        batch.append((sid, pos, [(tab[p // BLOCK], p % BLOCK) for p in pos], tab))
    tr = {}
    wk.attention_half(1, x, batch, tr)
    t0 = 0
    worst = 0
    for (_, pos, _, _) in batch:
        for i, p in enumerate(pos):
            K = tr["k"][t0:t0 + p + 1]
            V = tr["v"][t0:t0 + p + 1]
            ref = attention_one(tr["q"][t0 + i], K, V)
            diff = np.abs(tr["o"][t0 + i] - ref)
            ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(ref), 2.0 ** -126))) - 7)
            worst = max(worst, float((diff / ulp).max()))
        t0 += len(pos)
    assert worst <= 1.0, worst
