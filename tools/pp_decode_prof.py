"""Decode-step breakdown at PP = s on s GPUs (local mode: one process drives every stage):
device time per step and the per-kernel-kind event profile summed over the stages."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hsgen  # noqa: E402
from paper_2502_15524_b200 import hs  # noqa: E402

pp = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = dict(hsgen.CONFIGS["llama2-7b"])
h = hs.image_layout(cfg)
img = hs.HostImage(h, h.embed_off, h.total_bytes)
hsgen.image_fill(hsgen.image_header(cfg), hsgen.WEIGHT_SEED, img.ptr, h.embed_off, h.total_bytes)
n = torch.cuda.device_count()
gpus = [dict(device=d % n, h2d_gbps=55.0, free_bytes=180 << 30) for d in range(pp)]
plan = hs.plan_stages(cfg, gpus, pp, 1)
for k in range(pp):
    plan.device[k] = k % n
g = hs.Group(cfg, plan, img, num_blocks=64, max_seqs=1, max_tokens=512)
g.load_stage_async(-1)
g.prefill([0], hsgen.prompts(1, 512, cfg["vocab"]))
for _ in range(8):
    g.decode_step([0])
dev = 0.0
import time
t0 = time.perf_counter()
for _ in range(32):
    g.decode_step([0])
    dev += g.timing(pp - 1).call_ms
host = (time.perf_counter() - t0) / 32 * 1e3
print(json.dumps({"pp": pp, "gpus": n, "ms_per_step_host": round(host, 3), "ms_per_step_last_stage_device": round(dev / 32, 3)}))
g.profile(True)
for _ in range(8):
    g.decode_step([0])
g.profile(False)
for k, v in sorted(g.profile_read(reset=True).items()):
    print(json.dumps({"kind": k, "count": v["count"], "us_per": round(1e3 * v["ms"] / v["count"], 2)}))
g.destroy()
