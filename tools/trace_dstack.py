"""Phase timeline of the decode-stack kernel (7B, PP=1, B=1 or --batch N): per-layer stamps,
relative to the moment the layer's QKV activations were first loaded anywhere."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hsgen  # noqa: E402
from paper_2502_15524_b200 import hs  # noqa: E402

NAMES = ["B0 qkv act", "B1 o act", "B2 gu act", "B3 down act", "B3 down act end", "E qkv done", "E attn done",
         "E o done", "E norm_f", "E gu done", "E down done", "E norm_a", "A1 o w", "A2 gu w", "A3 down w", "A0 qkv w",
         "o grid-last", "o norm pass1 (wave 0)", "o norm pass2 (wave 0)", "d grid-last", "d norm start", "d norm done",
         "attn flags ok", "attn kv done", "qkv tfull", "qkv last-arriver", "qkv published",
         "qkv seg0 drained", "qkv seg0 atom", "qkv vals", "qkv stores", "attn item end"]

model = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "llama2-7b"
batch = int(sys.argv[sys.argv.index("--batch") + 1]) if "--batch" in sys.argv else 1
cfg = dict(hsgen.CONFIGS[model])
h = hs.image_layout(cfg)
img = hs.HostImage(h, h.embed_off, h.total_bytes)
hsgen.image_fill(hsgen.image_header(cfg), hsgen.WEIGHT_SEED, img.ptr, h.embed_off, h.total_bytes)
gpus = [dict(device=0, h2d_gbps=55.0, free_bytes=180 << 30)]
plan = hs.plan_stages(cfg, gpus, 1, 1)
g = hs.Group(cfg, plan, img, num_blocks=64 * batch, max_seqs=batch, max_tokens=512 * batch)
g.load_stage_async(-1)
ids = list(range(batch))
g.prefill(ids, hsgen.prompts(batch, 512, cfg["vocab"]))
for _ in range(8):
    g.decode_step(ids)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(16):
    g.decode_step(ids)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"ms_per_step": round(e0.elapsed_time(e1) / 16, 3)}))
hs.dstack_trace(True)
g.decode_step(ids)
G = torch.cuda.get_device_properties(0).multi_processor_count
L = cfg["n_layers"]
tr, per = hs.dstack_trace(True, G, L)
tr = tr.astype(np.int64)
per = per.astype(np.int64)
ref = np.array([tr[:, l, 0][tr[:, l, 0] > 0].min() for l in range(L)])
print(json.dumps({"layer_us_median": round(float(np.median(np.diff(ref))) / 1e3, 2),
                  "layer_us": [round(float(x) / 1e3, 1) for x in np.diff(ref)]}))
rows = []
for k, n in enumerate(NAMES):
    vals = []
    for l in range(2, L - 2):
        v = tr[:, l, k]
        v = v[v > 0]
        if len(v):
            vals.append(((v.min() - ref[l]) / 1e3, (np.median(v) - ref[l]) / 1e3, (v.max() - ref[l]) / 1e3, len(v)))
    if vals:
        a = np.array(vals)
        rows.append({"slot": n, "min": round(float(np.median(a[:, 0])), 2), "med": round(float(np.median(a[:, 1])), 2),
                     "max": round(float(np.median(a[:, 2])), 2), "n_ctas": int(np.median(a[:, 3]))})
for r in sorted(rows, key=lambda r: r["med"]):
    print(json.dumps(r))
nq = 3 * cfg["hidden"] // 128
for l in (10, 20):
    tq = (per[l, :nq] - ref[l]) / 1e3
    th = (per[l, 128:128 + cfg["n_heads"]] - ref[l]) / 1e3
    print(json.dumps({"layer": l, "qkv_tile_pub_us": [round(float(x), 1) for x in tq]}))
    print(json.dumps({"layer": l, "head_attn_pub_us": [round(float(x), 1) for x in th]}))
out = os.environ.get("TRACE_NPZ")
if out:  # raw stamps for offline analysis: tr[G][L][32] (ns), per-tile / per-head publish times, ref
    np.savez_compressed(out, tr=tr, per=per, ref=ref)
hs.dstack_trace(False)
g.destroy()
