"""Per-CTA phase timeline of the stream-K decode GEMM (HS debug trace)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_15524_b200 import hs

ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
hs.gemm_trace(True)
for M, K in [(4096, 4096), (22016, 4096), (4096, 11008)]:
    W = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    X = torch.randn(16, K, device="cuda").to(torch.bfloat16)
    out = torch.empty(1, M, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        hs.k_gemm(W, X, 1, 0, out, ws=ws)
    torch.cuda.synchronize()
    tr = hs.gemm_trace(True, 148).astype(np.int64)
    t0 = tr[:, 0].min()
    rel = (tr - t0) / 1000.0  # us
    names = ["start", "A requested", "dep resolved", "first full", "mma done", "epi done", "cta end"]
    stats = {n: (round(float(rel[:, i].min()), 2), round(float(np.median(rel[:, i])), 2), round(float(rel[:, i].max()), 2))
             for i, n in enumerate(names)}
    print(json.dumps({"M": M, "K": K, "MB": M * K * 2 / 1e6, "phases_us(min,med,max)": stats}))
