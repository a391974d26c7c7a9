"""Stress the decode-stack kernel at the 7B shape (test tool, GPU): PP=1 and PP=2-on-one-GPU
groups, a 512-token prefill, then many decode steps (per-step calls with logits, as
tests/test_fullsize_gpu.py does, plus device-fed decode_steps).  Prints one JSON line; on a
CUDA failure the decode stack's failure record (hs_debug_dstack_diag) goes to stderr.

  python tools/stress_dstack.py --steps 300 [--pp 1 2] [--capture]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import hsgen  # noqa: E402
from paper_2502_15524_b200 import hs  # noqa: E402

CFG = dict(hsgen.CONFIGS["llama2-7b"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--pp", type=int, nargs="+", default=[1, 2])
    ap.add_argument("--capture", action="store_true")
    ap.add_argument("--both", action="store_true", help="PP=1 and PP=2 groups alive together, alternating "
                    "steps (as test_7b_pp_invariance_and_consolidation_bitwise)")
    a = ap.parse_args()
    h = hs.image_layout(CFG)
    img = hs.HostImage(h, 0, h.total_bytes)
    hsgen.image_fill(hsgen.image_header(CFG), hsgen.WEIGHT_SEED, img.ptr, 0, h.total_bytes)
    out = {"env": {k: v for k, v in os.environ.items() if k.startswith("HS_")}, "steps": a.steps, "runs": []}
    prompt = hsgen.prompts(1, 512, CFG["vocab"])
    status = "ok"
    def mk(pp):
        gpus = [dict(device=0, h2d_gbps=55.0, free_bytes=180 << 30) for _ in range(pp)]
        plan = hs.plan_stages(CFG, gpus, pp, 1)
        for k in range(pp):
            plan.device[k] = 0
        g = hs.Group(CFG, plan, img, num_blocks=160, max_seqs=2, max_tokens=512)
        g.load_stage_async(-1)
        return g

    try:
        if a.both:
            g1, g2 = mk(1), mk(2)
            g1.prefill([0], prompt, want_logits=True)
            g2.prefill([0], prompt, want_logits=True)
            for _ in range(a.steps):
                x, y = g1.decode_step([0], want_logits=True), g2.decode_step([0], want_logits=True)
                assert (x[0] == y[0]).all() and (x[1] == y[1]).all()
            out["runs"].append({"both": True, "steps": a.steps})
            g1.destroy()
            g2.destroy()
        for pp in ([] if a.both else a.pp):
            gpus = [dict(device=0, h2d_gbps=55.0, free_bytes=180 << 30) for _ in range(pp)]
            plan = hs.plan_stages(CFG, gpus, pp, 1)
            for k in range(pp):
                plan.device[k] = 0
            g = hs.Group(CFG, plan, img, num_blocks=160, max_seqs=2, max_tokens=512)
            g.load_stage_async(-1)
            if a.capture:
                g.capture(True)
            t0 = time.time()
            g.prefill([0], prompt, want_logits=True)
            n = 0
            for _ in range(a.steps):
                g.decode_step([0], want_logits=True)
                n += 1
            out["runs"].append({"pp": pp, "per_step_calls": n, "s": round(time.time() - t0, 2)})
            g.destroy()
    except hs.HsError as e:
        status = f"error: {e}"
        out["diag_rows"] = hs.lib().hs_debug_dstack_diag(1)
    out["status"] = status
    print(json.dumps(out), flush=True)
    return 0 if status == "ok" else 1


if __name__ == "__main__":
    sys.exit(main())
