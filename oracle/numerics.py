"""Oracle numerics: the per-op definitions of a Llama-2 decoder layer, in float64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Rounding contract: activations are
stored in bf16; every expression is evaluated in float64 and rounded to bf16 exactly once
where a tensor is materialised.  ``rnd`` is the rounding function; passing ``exact`` (the
identity) gives the unrounded float64 model used to pin the architecture against an
independent library implementation (tests/test_oracle_arch.py).
"""
from __future__ import annotations

import numpy as np


# ---------------------------------------------------------------- bf16 --------------------
def bf16_bits(x) -> np.ndarray:
    """float -> bf16 bit pattern: first to float32 (RNE), then round-to-nearest-even to the
    top 16 bits; NaN stays NaN (quiet)."""
    f = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    r = np.where(nan, ((u >> 16) | 0x40).astype(np.uint16), r)
    return r.astype(np.uint16)


def bf16_value(bits) -> np.ndarray:
    """bf16 bit pattern -> float64 value (exact)."""
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return b.view(np.float32).astype(np.float64)


def bf16(x) -> np.ndarray:
    """Round to bf16 and return the (exactly representable) float64 value."""
    return bf16_value(bf16_bits(x))


def exact(x) -> np.ndarray:
    return np.asarray(x, dtype=np.float64)


# ---------------------------------------------------------------- ops ---------------------
def rmsnorm(x: np.ndarray, w: np.ndarray, eps: float, rnd=bf16) -> np.ndarray:
    """y_i = rnd(x_i * r * w_i), r = 1/sqrt(mean_j x_j^2 + eps) (Llama RMSNorm, eps = 1e-5).
    One rounding; the weight is applied before it."""
    ms = np.mean(x * x, axis=-1, keepdims=True)
    r = 1.0 / np.sqrt(ms + eps)
    return rnd(x * r * w)


def rmsnorm_split(x: np.ndarray, w: np.ndarray, eps: float, rnd=bf16):
    """The RMSNorm that feeds a linear layer (steps 4.1 and 4.7, reading R10b): in
    real arithmetic (x r w) W^T = r ((x w) W^T) with r = 1/sqrt(mean_j x_j^2 + eps), so the
    materialised operand is a = rnd(x_i * w_i) and the per-row scale r multiplies the product
    before its rounding (the consumer computes rnd(r * linear(a, W))).  Returns (a, r[.., 1])."""
    ms = np.mean(x * x, axis=-1, keepdims=True)
    r = 1.0 / np.sqrt(ms + eps)
    return rnd(x * w), r


def linear(x: np.ndarray, W: np.ndarray, acc=np.float64) -> np.ndarray:
    """x [T,K] @ W[N,K]^T accumulated in float64, unrounded (the consumer rounds).
    ``acc=np.float32`` gives the same product accumulated in float32: it is only used to
    measure the noise floor any fp32-accumulating implementation has against this oracle
    (DESIGN.md "Tolerance"), never as the reference."""
    if acc is np.float64:
        return x @ W.T
    return (x.astype(acc) @ W.T.astype(acc)).astype(np.float64)


def silu(g: np.ndarray) -> np.ndarray:
    return g / (1.0 + np.exp(-g))


def rope_cos_sin(positions: np.ndarray, head_dim: int, theta: float, table_f32: bool = True):
    """inv_f_i = theta^(-2i/d), angle = p * inv_f_i (float64); c, s = cos, sin, stored as
    float32 values (the table precision of DESIGN.md) unless table_f32 is False."""
    i = np.arange(head_dim // 2, dtype=np.float64)
    inv_f = theta ** (-2.0 * i / head_dim)
    ang = np.asarray(positions, dtype=np.float64)[:, None] * inv_f[None, :]
    c, s = np.cos(ang), np.sin(ang)
    if table_f32:
        c, s = c.astype(np.float32).astype(np.float64), s.astype(np.float32).astype(np.float64)
    return c, s


def rope(x: np.ndarray, c: np.ndarray, s: np.ndarray, rnd=bf16) -> np.ndarray:
    """Rotate-half RoPE on x [T, n_heads, d] with per-token tables c, s [T, d/2]:
    x'_i = x_i c_i - x_{i+d/2} s_i ;  x'_{i+d/2} = x_{i+d/2} c_i + x_i s_i."""
    h = x.shape[-1] // 2
    x1, x2 = x[..., :h], x[..., h:]
    cc, ss = c[:, None, :], s[:, None, :]
    return rnd(np.concatenate([x1 * cc - x2 * ss, x2 * cc + x1 * ss], axis=-1))


def attention_one(q: np.ndarray, K: np.ndarray, V: np.ndarray, rnd=bf16) -> np.ndarray:
    """One query position over its visible keys, all heads.
    q [nh, d]; K, V [n_keys, nh, d].  s_j = (q . k_j) / sqrt(d);  m = max s;  e = exp(s - m);
    o = rnd(sum_j e_j v_j / sum_j e_j)  (float64 throughout, one rounding)."""
    d = q.shape[-1]
    s = np.einsum("hd,khd->hk", q, K) / np.sqrt(d)
    m = s.max(axis=-1, keepdims=True)
    e = np.exp(s - m)
    o = np.einsum("hk,khd->hd", e, V) / e.sum(axis=-1)[:, None]
    return rnd(o)


def argmax_lowest(logits: np.ndarray) -> int:
    """Greedy choice; ties -> lowest token id (np.argmax returns the first maximum)."""
    return int(np.argmax(logits))
