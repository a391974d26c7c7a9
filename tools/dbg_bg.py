"""Repro harness: repeated 7B cold starts with the background host load, local mode, 1 GPU."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import hsgen
from paper_2502_15524_b200 import hs
cfg = dict(hsgen.CONFIGS["llama2-7b"])
h = hs.image_layout(cfg)
img = hs.HostImage(h, h.embed_off, h.total_bytes)
hsgen.image_fill(hsgen.image_header(cfg), hsgen.WEIGHT_SEED, img.ptr, h.embed_off, h.total_bytes)
pp = int(sys.argv[1]) if len(sys.argv) > 1 else 2
bg = "--nobg" not in sys.argv
gpus = [dict(device=d, h2d_gbps=55.0, free_bytes=180 << 30) for d in range(pp)]
plan = hs.plan_stages(cfg, gpus, pp, 1)
for k in range(pp):
    plan.device[k] = 0
prompt = hsgen.prompts(1, 512, cfg["vocab"])
for it in range(5):
    g = hs.Group(cfg, plan, img, num_blocks=60, max_seqs=1, max_tokens=512)
    g.load_stage_async(-1)
    g.prefill([0], prompt)
    if bg:
        g.load_background_async(0)
    try:
        for s in range(64):
            g.decode_step([0])
        st = g.consolidate(0)
        for s in range(64):
            g.decode_step([0])
        print("iter", it, "ok", st.weight_bytes, st.weight_bytes_host, flush=True)
    except Exception as e:
        print("iter", it, "FAILED at", s, e, flush=True)
        raise
    g.destroy()
