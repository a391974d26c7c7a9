"""Kernel micro-benchmarks through include/hs_kernels.h (CUDA events, warm L2 excluded by
rotating buffers larger than L2 for the weight operands).  Prints one JSON line per case.
Usage: python tools/microbench.py [gemm|attn|all] [--iters N]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_15524_b200 import hs  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))


def timeit(fn, iters):
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3  # us


def gemm_cases(iters):
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    for name, M, K, N in [("qkv", 12288, 4096, 1), ("o", 4096, 4096, 1), ("gate_up", 22016, 4096, 1),
                          ("down", 4096, 11008, 1), ("gate_up_b16", 22016, 4096, 16), ("lm_head", 32000, 4096, 1),
                          ("qkv_13b_b16", 15360, 5120, 16), ("prefill_qkv", 12288, 4096, 512),
                          ("prefill_gate_up", 22016, 4096, 512), ("prefill_o", 4096, 4096, 512),
                          ("prefill_down", 4096, 11008, 512)]:
        nrot = max(1, int(400e6 // (M * K * 2)) + 1)
        Ws = [torch.randn(M, K, device="cuda").to(torch.bfloat16) * K ** -0.5 for _ in range(nrot)]
        X = torch.randn(max(N, 16), K, device="cuda").to(torch.bfloat16)
        out = torch.empty(N, M, device="cuda", dtype=torch.bfloat16)
        us = timeit(lambda i: hs.k_gemm(Ws[i % nrot], X, N, 0, out, ws=ws), iters)
        byts = 2 * (M * K + N * K + N * M)
        fl = 2 * M * N * K
        print(json.dumps({"case": name, "M": M, "K": K, "N": N, "us": round(us, 2),
                          "gbs": round(byts / us / 1e3, 1), "hbm_frac": round(byts / us / 1e3 / PEAK["hbm_gbs"], 3),
                          "tflops": round(fl / us / 1e6, 1),
                          "tensor_frac": round(fl / us / 1e6 / PEAK["bf16_tflops"], 3)}), flush=True)
        del Ws


def overhead_cases(iters):
    """Fixed cost of the decode GEMM: time vs bytes at constant M (one tile row per SM)."""
    ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    for M, K in [(18944, 128), (18944, 256), (18944, 1024), (18944, 2048), (18944, 4096), (4096, 4096), (8192, 4096)]:
        nrot = max(1, int(400e6 // (M * K * 2)) + 1)
        Ws = [torch.randn(M, K, device="cuda").to(torch.bfloat16) for _ in range(nrot)]
        X = torch.randn(16, K, device="cuda").to(torch.bfloat16)
        out = torch.empty(1, M, device="cuda", dtype=torch.bfloat16)
        us = timeit(lambda i: hs.k_gemm(Ws[i % nrot], X, 1, 0, out, ws=ws), iters)
        print(json.dumps({"case": "overhead", "M": M, "K": K, "MB": round(M * K * 2 / 1e6, 2), "us": round(us, 2)}), flush=True)
        del Ws
    # the same GEMMs without the counter memset of hs_k_gemm (ws=None -> tiled split path) for reference
    a = torch.zeros(1, 16, device="cuda", dtype=torch.float32)
    t = torch.zeros(1, device="cuda", dtype=torch.int32)
    us = timeit(lambda i: hs.k_argmax(a, t), iters)
    print(json.dumps({"case": "tiny kernel (argmax 16)", "us": round(us, 2)}), flush=True)
    us = timeit(lambda i: ws[:65536].zero_(), iters)
    print(json.dumps({"case": "64KB memset", "us": round(us, 2)}), flush=True)


def attn_cases(iters):
    for nh, d, ctx, B in [(32, 128, 544, 1), (40, 128, 576, 16), (32, 128, 4000, 1)]:
        nblk = B * ((ctx + 15) // 16) + 4
        pool = torch.randn(nblk, 2, nh, 16, d, device="cuda").to(torch.bfloat16)
        maxb = (ctx + 15) // 16 + 1
        tables = torch.arange(B * maxb, device="cuda", dtype=torch.int32).reshape(B, maxb) % nblk
        seqs = torch.tensor([[i, 1, ctx - 1, i] for i in range(B)], dtype=torch.int32, device="cuda")
        q = torch.randn(B, nh * d, device="cuda").to(torch.bfloat16)
        o = torch.empty_like(q)
        ws = torch.empty(B * nh * 64 * (d + 2), dtype=torch.float32, device="cuda")
        us = timeit(lambda i: hs.k_attention(q, pool, seqs, 1, ctx, tables, o, nh, d, True, ws), iters)
        byts = B * ctx * 2 * nh * d * 2
        print(json.dumps({"case": f"attn_decode nh{nh} ctx{ctx} B{B}", "us": round(us, 2), "gbs": round(byts / us / 1e3, 1)}), flush=True)
        # prefill
    for nh, d, T in [(32, 128, 512)]:
        nblk = (T + 15) // 16 + 1
        pool = torch.randn(nblk, 2, nh, 16, d, device="cuda").to(torch.bfloat16)
        tables = torch.arange(nblk, device="cuda", dtype=torch.int32).reshape(1, nblk)
        seqs = torch.tensor([[0, T, 0, 0]], dtype=torch.int32, device="cuda")
        q = torch.randn(T, nh * d, device="cuda").to(torch.bfloat16)
        o = torch.empty_like(q)
        us = timeit(lambda i: hs.k_attention(q, pool, seqs, T, T, tables, o, nh, d, False, None), max(3, iters // 10))
        fl = 4 * nh * d * T * (T + 1) / 2
        print(json.dumps({"case": f"attn_prefill nh{nh} T{T}", "us": round(us, 2), "tflops": round(fl / us / 1e6, 2)}), flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 50
    if what in ("gemm", "all"):
        gemm_cases(iters)
    if what in ("attn", "all"):
        attn_cases(iters)
    if what in ("overhead", "all"):
        overhead_cases(iters)
