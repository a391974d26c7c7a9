"""Layer-level teacher-forced parity of the CUDA path against the oracle (test helper).

Why layer by layer: comparing only final logits lets every bf16 rounding flip
of 32-40 layers cascade into the bound.  Here the GPU's own hidden state at each capture point
(hs_debug_capture: the input of layer l, its h = x + Attention(RMSNorm(x)) W_o^T, its output)
is fed to the oracle's half-layer (oracle.decoder.Worker.attention_half / mlp_half, SURVEY
§8(c) steps 4.1-4.6 / 4.7-4.9) and the oracle's result is compared with the GPU's next
capture point.  The attention half reads the GPU's KV cache for earlier positions (pool
entries copied from hs_debug_read_kv), so every comparison covers one half-layer of arithmetic
and nothing else.  PAPER.md:139-141: a pipeline-parallel group computes exactly the layers of
the unpartitioned model, so the same check holds on every stage.

Acceptance per half-layer ("layer-level bound"):
  * every element within one bf16 ulp at its row's scale, |d| <= 2^(floor(log2 max_j |row_j|) - 7);
  * at least MIN_EQUAL of the elements bit-identical, at most MAX_GT1 more than one ulp of
    their own magnitude away;
  * K/V written by the GPU for the call's positions against the oracle's k', v: v one row-ulp,
    k' two (two consecutive roundings, bf16(k) then bf16(RoPE(k)), with no contraction between);
  * logits from the GPU's final hidden state: max |d| <= 2e-2 (the north star's bound) against
    the oracle's final RMSNorm + lm_head of the same hidden state, and the greedy token equal
    to the oracle's argmax unless the oracle's top-2 margin is below 2x that difference.
"""
from __future__ import annotations

import json
import os

import numpy as np

from oracle.decoder import BLOCK, Worker
from oracle.numerics import argmax_lowest, bf16_value

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LOGIT_TOL = 2e-2          # north star: max abs logit error
MIN_EQUAL = 0.90          # bit-identical fraction per half-layer (measured >= 0.97: profiles/r02_parity_*.json)
MAX_GT1 = 0.01            # fraction more than 1 ulp of their own magnitude away


def ulp(v):
    """bf16 ulp of |v| (normal range): 2^(floor(log2 |v|) - 7)."""
    a = np.abs(np.asarray(v, dtype=np.float64))
    return np.exp2(np.floor(np.log2(np.maximum(a, 2.0 ** -126))) - 7)


def half_stats(gpu_vals, ref_vals):
    """Error statistics of one half-layer output [rows, H] (float64 values of bf16)."""
    d = np.abs(gpu_vals - ref_vals)
    row_ulp = ulp(np.abs(ref_vals).max(axis=1, keepdims=True))
    own = ulp(np.maximum(np.abs(gpu_vals), np.abs(ref_vals)))
    return dict(max_row_ulps=float((d / row_ulp).max()), frac_equal=float((d == 0).mean()),
                frac_gt1=float((d > own).mean()), max_abs=float(d.max()))


def check_half(st, what, row_ulps=1.0):
    """row_ulps: one per bf16 rounding between the GPU's input and the compared value that is not
    followed by a contraction (k' = bf16(RoPE(bf16(k))): two; every half-layer output: one)."""
    assert st["max_row_ulps"] <= row_ulps, (what, st)
    assert st["frac_equal"] >= MIN_EQUAL, (what, st)
    assert st["frac_gt1"] <= MAX_GT1, (what, st)


class Recorder:
    """Per-sequence capture rows of every call (positions + capture points), for a later
    layer-by-layer oracle pass, plus the GPU logits of every call for the head check."""

    def __init__(self, cfg, points=None):
        self.cfg = cfg
        self.L = cfg["n_layers"]
        self.points = points if points is not None else list(range(2 * self.L + 1))
        self.rows = {}      # seq -> list of (positions, {point: bits [m, H]})
        self.heads = []     # (seq list, last-row bits [n, H], gpu logits [n, V], gpu tokens)

    def record(self, g, seq_ids, lens, logits=None, tokens=None, want=None):
        """After a call: reads every capture point of the rows of the sequences in `want`
        (default all).  lens: tokens per sequence in the call (decode: all 1)."""
        want = set(seq_ids if want is None else want)
        row0 = 0
        last_rows = []
        for sid, m in zip(seq_ids, lens):
            if sid in want:
                pts = {pt: g.read_hidden(pt, row0, m) for pt in self.points}
                hist = self.rows.setdefault(sid, [])
                p0 = hist[-1][0][-1] + 1 if hist else 0
                hist.append((np.arange(p0, p0 + m), pts))
                last_rows.append(pts[2 * self.L][-1])
            row0 += m
        if logits is not None:
            sel = [i for i, s in enumerate(seq_ids) if s in want]
            self.heads.append(([seq_ids[i] for i in sel], np.stack(last_rows), logits[sel], None if tokens is None else tokens[sel]))

    def phase(self, sid, start_call, end_call=None):
        """Concatenated (positions, {point: bits}) of calls [start_call, end_call) of sid."""
        h = self.rows[sid][start_call:end_call]
        pos = np.concatenate([p for p, _ in h])
        pts = {pt: np.concatenate([d[pt] for _, d in h]) for pt in h[0][1]}
        return pos, pts


def check_layers(cfg, W, rec: Recorder, g, layers, phases, results, tag="", evict=False):
    """phases: list of (name, {sid: (start_call, end_call)}).  For each layer and phase: the
    oracle's attention half from the GPU's layer input (earlier positions' K/V from the GPU's
    cache) and its MLP half from the GPU's h; both compared with the GPU's capture points, plus
    the GPU's K/V for the phase's positions against the oracle's k', v."""
    nh, d = cfg["n_heads"], cfg["head_dim"]
    for l in layers:
        for name, sel in phases:
            batch, xs, hs_gpu, outs = [], [], [], []
            max_pos = max(rec.phase(s, *sel[s])[0][-1] for s in sel) + 1
            nb_seq = (max_pos + BLOCK - 1) // BLOCK
            wk = Worker(cfg, W, l, l + 1, num_blocks=nb_seq * len(sel))
            for i, sid in enumerate(sel):
                pos, pts = rec.phase(sid, *sel[sid])
                table = list(range(i * nb_seq, (i + 1) * nb_seq))
                p0 = int(pos[0])
                if p0 > 0:  # earlier positions' K/V: the GPU's cache, bit for bit
                    kv = g.read_kv(sid, l, 0, p0)           # [p0, 2, nh, d]
                    for p in range(p0):
                        wk.kv[l][table[p // BLOCK], :, :, p % BLOCK, :] = kv[p]
                slots = [(table[p // BLOCK], p % BLOCK) for p in pos]
                batch.append((sid, pos, slots, table))
                xs.append(bf16_value(pts[2 * l]))
                hs_gpu.append(bf16_value(pts[2 * l + 1]))
                outs.append(bf16_value(pts[2 * l + 2]))
            x, hg, og = np.concatenate(xs), np.concatenate(hs_gpu), np.concatenate(outs)
            tr = {}
            h_ref = wk.attention_half(l, x, batch, tr)
            st_a = half_stats(hg, h_ref)
            # the GPU's K/V for the phase's positions vs the oracle's k' (after RoPE) and v
            kg, vg = [], []
            for (sid, pos, _, _) in batch:
                kv = g.read_kv(sid, l, int(pos[0]), len(pos))
                kg.append(bf16_value(kv[:, 0]).reshape(len(pos), nh * d))
                vg.append(bf16_value(kv[:, 1]).reshape(len(pos), nh * d))
            st_k = half_stats(np.concatenate(kg), tr["k"].reshape(-1, nh * d))
            st_v = half_stats(np.concatenate(vg), tr["v"].reshape(-1, nh * d))
            out_ref = wk.mlp_half(l, hg)
            st_m = half_stats(og, out_ref)
            key = f"{tag}layer{l}.{name}"
            results[key] = dict(attention_half=st_a, mlp_half=st_m, k=st_k, v=st_v, rows=int(x.shape[0]))
            check_half(st_a, key + ".attention_half")
            check_half(st_m, key + ".mlp_half")
            check_half(st_k, key + ".k", row_ulps=2.0)
            check_half(st_v, key + ".v")
        if evict:  # full-size models: keep one layer's float64 weights in memory at a time
            W._layers.pop(l, None)


def check_heads(cfg, W, rec: Recorder, results, tag=""):
    """GPU logits vs the oracle's final RMSNorm + lm_head of the GPU's own final hidden state."""
    wk = Worker(cfg, W, cfg["n_layers"], cfg["n_layers"], num_blocks=1)
    errs, ties = [], 0
    for (sids, rows, logits, toks) in rec.heads:
        ref = wk.head(bf16_value(rows))
        e = float(np.abs(logits.astype(np.float64) - ref).max())
        errs.append(e)
        assert e <= LOGIT_TOL, (tag, e)
        if toks is not None:
            for i in range(len(sids)):
                r = argmax_lowest(ref[i])
                if toks[i] != r:
                    top2 = np.sort(ref[i])[-2:]
                    assert top2[1] - top2[0] < 2 * e, (tag, "token mismatch without a tie", sids[i])
                    ties += 1
    results[f"{tag}head"] = dict(max_abs_logit_err=max(errs), calls=len(errs), ties=ties)
    return errs


def save(results, name):
    """Persist the measured errors (gpurun_out/ on the GPU box; copied to profiles/)."""
    out = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, f"parity_{name}.json"), "w") as f:
        json.dump(results, f, indent=1, sort_keys=True)


def summary(results):
    """Worst case over all half-layers (for the JSON header / DESIGN.md)."""
    keys = ["attention_half", "mlp_half", "k", "v"]
    agg = {}
    for k in keys:
        vals = [v[k] for v in results.values() if isinstance(v, dict) and k in v]
        if vals:
            agg[k] = dict(max_row_ulps=max(x["max_row_ulps"] for x in vals),
                          min_frac_equal=min(x["frac_equal"] for x in vals),
                          max_frac_gt1=max(x["frac_gt1"] for x in vals))
    heads = [v for k, v in results.items() if k.endswith("head")]
    if heads:
        agg["max_abs_logit_err"] = max(h["max_abs_logit_err"] for h in heads)
    return agg
