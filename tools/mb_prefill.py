"""Prefill GEMM shapes of a 7B layer (T tokens) with their real epilogues, per kernel choice
(HS_TP_BN in the environment forces one: 128 = single CTA, 2128 / 2256 = CTA pair)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_15524_b200 import hs  # noqa: E402
T = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
for name, M, K, epi in (("qkv", 12288, 4096, 0), ("o", 4096, 4096, 1), ("gate_up", 22016, 4096, 2), ("down", 4096, 11008, 1)):
    Ws = [torch.randn(M, K, device="cuda").to(torch.bfloat16) * K ** -0.5 for _ in range(3)]
    X = torch.randn(T, K, device="cuda").to(torch.bfloat16)
    ocols = M // 2 if epi == 2 else M
    out = torch.empty(T, ocols, device="cuda", dtype=torch.bfloat16)
    resid = torch.randn(T, M, device="cuda").to(torch.bfloat16) if epi == 1 else None
    for i in range(3):
        hs.k_gemm(Ws[i % 3], X, T, epi, out, resid=resid, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(20):
        hs.k_gemm(Ws[i % 3], X, T, epi, out, resid=resid, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(json.dumps({"force": os.environ.get("HS_TP_BN", "auto"), "case": name, "T": T, "us": round(us, 1),
                      "tflops": round(2 * M * T * K / us / 1e6, 1)}))
    del Ws
