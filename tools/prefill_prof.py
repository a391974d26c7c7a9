"""Warm prefill (weights resident) per-kernel profile of the 7B model: T tokens, 1 sequence."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hsgen  # noqa: E402
from paper_2502_15524_b200 import hs  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 512
cfg = dict(hsgen.CONFIGS["llama2-7b"])
h = hs.image_layout(cfg)
img = hs.HostImage(h, h.embed_off, h.total_bytes)
hsgen.image_fill(hsgen.image_header(cfg), hsgen.WEIGHT_SEED, img.ptr, h.embed_off, h.total_bytes)
plan = hs.plan_stages(cfg, [dict(device=0, h2d_gbps=55.0, free_bytes=180 << 30)], 1, 1)
g = hs.Group(cfg, plan, img, num_blocks=T // 16 + 8, max_seqs=1, max_tokens=T)
g.load_stage_async(-1)
p = hsgen.prompts(1, T, cfg["vocab"])
for it in range(3):
    g.prefill([0], p)
    g.release_seq(0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for it in range(5):
    g.prefill([0], p)
    g.release_seq(0)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"prefill_ms": round(e0.elapsed_time(e1) / 5, 3)}))
g.profile(True)
g.prefill([0], p)
g.profile(False)
g.release_seq(0)
for k, v in sorted(g.profile_read(reset=True).items()):
    print(json.dumps({"kind": k, "count": v["count"], "us_per": round(1e3 * v["ms"] / v["count"], 2),
                      "tflops": round(v["flops"] / (v["ms"] / 1e3) / 1e12, 1) if v["flops"] else None}))
g.destroy()
