"""Run-to-run determinism of the whole tiny prefill + 8 decode steps (PP = 1 and 2 on one GPU):
30 fresh groups, logits and tokens compared bitwise with the first.  The prefill attention
kernel is chosen by HS_ATTN_TC."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hsgen  # noqa: E402
from paper_2502_15524_b200 import hs  # noqa: E402

cfg = hsgen.CONFIGS["tiny"]
h = hs.image_layout(cfg)
img = hs.HostImage(h, 0, h.total_bytes)
hsgen.image_fill(hsgen.image_header(cfg), hsgen.WEIGHT_SEED, img.ptr, 0, h.total_bytes)
prompts = hsgen.prompts(2, 32, cfg["vocab"])
ref = None
bad = []
for it in range(30):
    pp = 1 + it % 2
    gpus = [dict(device=0, h2d_gbps=50.0, free_bytes=8 << 30)] * 2
    plan = hs.plan_stages(cfg, gpus, pp, 1)
    for k in range(pp):
        plan.device[k] = 0
    g = hs.Group(cfg, plan, img, num_blocks=64, max_seqs=8, max_tokens=256)
    g.load_stage_async(-1)
    out = [g.prefill([0, 1], prompts, want_logits=True)]
    for _ in range(8):
        out.append(g.decode_step([0, 1], want_logits=True))
    g.destroy()
    if ref is None:
        ref = out
        continue
    for step, ((t0, l0), (t1, l1)) in enumerate(zip(ref, out)):
        if not (np.array_equal(t0, t1) and np.array_equal(l0, l1)):
            bad.append((it, pp, step, float(np.abs(l0 - l1).max())))
            break
print(f"HS_ATTN_TC={os.environ.get('HS_ATTN_TC', '0')}: {len(bad)} of 29 runs differ from run 0: {bad[:10]}")
