"""CPU pin of the layer-level parity harness (tests/layerwise.py) used by the GPU tests: run
through the oracle itself (an oracle group that records every capture point the way
hs_debug_capture does), the harness must reproduce every half-layer, the K/V of every position
and every logit EXACTLY.  This fixes the harness's bookkeeping (positions, block tables, the
injected K/V of earlier positions, the decode steps replayed as one causal chunk, row order of
packed multi-sequence calls) independently of any GPU."""
import numpy as np
import pytest

import hsgen
from oracle.decoder import Group, Weights
from oracle.numerics import bf16_bits

import layerwise as LW


class OracleCapture(Group):
    """An oracle group exposing the capture interface of paper_2502_15524_b200.hs.Group."""

    def _run(self, seq_ids, toks_per_seq):
        batch, tokens = [], []
        for sid, toks in zip(seq_ids, toks_per_seq):
            c0 = self.bm.ctx.get(sid, 0)
            slots = self.bm.append(sid, len(toks))
            batch.append((sid, np.arange(c0, c0 + len(toks)), slots, self.bm.tables[sid]))
            tokens.extend(int(t) for t in toks)
        x = self.w.embed_rows(tokens)
        pts = [bf16_bits(x)]
        wk = self.workers[0]
        for l in wk.layers:
            h = wk.attention_half(l, x, batch)
            x = wk.mlp_half(l, h)
            pts += [bf16_bits(h), bf16_bits(x)]
        self.points = pts
        last = np.cumsum([len(t) for t in toks_per_seq]) - 1
        logits = wk.head(x[last])
        return [int(np.argmax(r)) for r in logits], logits

    def read_hidden(self, pt, row0, n):
        return self.points[pt][row0:row0 + n]


def test_harness_reproduces_the_oracle_exactly(tiny_cfg):
    cfg = tiny_cfg
    W = Weights(cfg)
    g = OracleCapture(cfg, W, pp=1, num_blocks=64)
    prompts = [hsgen.tokens(1, 23, cfg["vocab"]), hsgen.tokens(2, 40, cfg["vocab"])]
    rec = LW.Recorder(cfg)
    toks, logits = g.prefill([5, 9], prompts)
    rec.record(g, [5, 9], [23, 40], logits, np.array(toks))
    for _ in range(6):
        toks, logits = g.decode([5, 9], toks)
        rec.record(g, [5, 9], [1, 1], logits, np.array(toks))
    res = {}
    phases = [("prefill", {5: (0, 1), 9: (0, 1)}), ("decode", {5: (1, None), 9: (1, None)})]
    LW.check_layers(cfg, W, rec, g, range(cfg["n_layers"]), phases, res)
    LW.check_heads(cfg, W, rec, res)
    for k, v in res.items():
        if k.endswith("head"):
            assert v["max_abs_logit_err"] == 0.0
            continue
        for part in ("attention_half", "mlp_half", "k", "v"):
            assert v[part]["frac_equal"] == 1.0 and v[part]["max_abs"] == 0.0, (k, part, v[part])


def test_harness_detects_a_wrong_layer(tiny_cfg):
    """A capture point perturbed like a plausible kernel bug (one head's attention output
    dropped) fails the bound."""
    cfg = tiny_cfg
    W = Weights(cfg)
    g = OracleCapture(cfg, W, pp=1, num_blocks=64)
    prompts = [hsgen.tokens(3, 32, cfg["vocab"])]
    rec = LW.Recorder(cfg)
    toks, logits = g.prefill([0], prompts)
    wk = g.workers[0]
    # recompute layer 1's h without head 2's contribution
    from oracle.numerics import bf16, bf16_value
    x1 = bf16_value(g.points[2])
    tr = {}
    wk2 = OracleCapture(cfg, W, pp=1, num_blocks=64).workers[0]
    batch = [(0, np.arange(32), [(b, o) for b, o in ((p // 16, p % 16) for p in range(32))], [0, 1])]
    wk2.attention_half(1, x1, batch, tr)
    o = tr["o"].copy()
    o[:, 2, :] = 0.0
    h_bad = bf16(x1 + o.reshape(32, -1) @ W.layer(1)["wo"].T)
    g.points[3] = bf16_bits(h_bad)
    rec.record(g, [0], [32], logits, np.array(toks))
    with pytest.raises(AssertionError):
        LW.check_layers(cfg, W, rec, g, [1], [("prefill", {0: (0, 1)})], {})
    del wk
