"""Targets for ncu range replay (`--replay-mode app-range`, profiler start/stop around one phase):
  load  : 7B PP=1 cold-start load (copy-engine H2D of 13.5 GB)            -> PCIe counters
  cons  : 7B PP=2 on GPUs 0, 1 in ONE process (local mode), consolidation into stage 0
          (copy_list_kernel pulls stage 1's slice + KV over NVLink)       -> NVLink / DRAM counters
usage: python tools/ncu_ranges.py load|cons"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hsgen  # noqa: E402
from paper_2502_15524_b200 import hs  # noqa: E402

what = sys.argv[1]
cfg = dict(hsgen.CONFIGS["llama2-7b"])
h = hs.image_layout(cfg)
img = hs.HostImage(h, 0, h.total_bytes)
hsgen.image_fill(hsgen.image_header(cfg), hsgen.WEIGHT_SEED, img.ptr, 0, h.total_bytes)
pp = 1 if what == "load" else 2
gpus = [dict(device=d, h2d_gbps=55.0, free_bytes=180 << 30) for d in range(pp)]
plan = hs.plan_stages(cfg, gpus, pp, 1)
for k in range(pp):
    plan.device[k] = k
g = hs.Group(cfg, plan, img, num_blocks=160, max_seqs=2, max_tokens=512)
prompt = hsgen.prompts(1, 512, cfg["vocab"])
if what == "load":
    g.load_stage_async(-1)  # warm
    g.load_stats(0)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    g.load_stage_async(-1)
    g.load_stats(0)
    torch.cuda.profiler.stop()
else:
    g.load_stage_async(-1)
    g.prefill([0], prompt)
    for _ in range(64):
        g.decode_step([0])
    for d in range(pp):
        torch.cuda.synchronize(d)
    torch.cuda.profiler.start()
    st = g.consolidate(0)
    torch.cuda.profiler.stop()
    print(f"consolidation {st.weight_bytes + st.kv_bytes} B in {st.seconds * 1e3:.2f} ms, pause {st.pause_seconds * 1e3:.2f} ms")
g.destroy()
