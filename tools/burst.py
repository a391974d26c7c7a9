"""BASELINE config 5: simultaneous cold starts of mixed
7B / 13B-shaped models on the GPUs of one box, bursty arrivals, naive vs contention-aware
placement.  4-GPU variant: 2 x 7B + 2 x 13B (8 GPUs: 4 + 4).

Arrivals: inter-arrival gaps ~ Gamma(shape 1/CV^2, scale CV^2/rate), CV = 8, rate = 8/s,
seed 7 (PAPER.md:859's burst model).  Each request is one 512-token prompt; TTFT = host time
from its arrival to its first token on the host (weights in pinned host memory at T0).

Policies (placement is decided at each arrival from the state the scheduler sees then):
  naive   : model j -> PP = 1 on GPU j mod n (its own PCIe link, no coordination);
  hydra   : the library's hs_place_cold_start (Alg. 1 on the contended links + Eq. 3 admission
            + Eq. 4 bookkeeping, R20), one link group per GPU at its measured isolated
            pinned-H2D bandwidth.
This file is harness only: the placement policy lives in the library."""
from __future__ import annotations

import json
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hsgen  # noqa: E402
from paper_2502_15524_b200 import hs  # noqa: E402

def arrivals(n, cv=8.0, rate=8.0, seed=7):
    rng = np.random.default_rng(seed)
    gaps = rng.gamma(1.0 / cv ** 2, cv ** 2 / rate, size=n)
    t = np.cumsum(gaps)
    return (t - t[0]).tolist()


def measure_links(n_gpus, img):
    """Isolated pinned-H2D bandwidth of every GPU's link (GB/s, best of 3) and the concurrent sum."""
    probe = min(1 << 30, img.buf.numel())
    bufs = [torch.empty(probe, dtype=torch.uint8, device=f"cuda:{d}") for d in range(n_gpus)]
    streams = [torch.cuda.Stream(device=d) for d in range(n_gpus)]
    iso = []
    for d in range(n_gpus):
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize(d)
            t0 = time.perf_counter()
            with torch.cuda.stream(streams[d]):
                bufs[d].copy_(img.buf[:probe], non_blocking=True)
            torch.cuda.synchronize(d)
            best = min(best, time.perf_counter() - t0)
        iso.append(probe / best / 1e9)
    conc = 0.0
    for _ in range(3):
        for d in range(n_gpus):
            torch.cuda.synchronize(d)
        t0 = time.perf_counter()
        for d in range(n_gpus):
            with torch.cuda.stream(streams[d]):
                bufs[d].copy_(img.buf[:probe], non_blocking=True)
        for d in range(n_gpus):
            torch.cuda.synchronize(d)
        conc = max(conc, n_gpus * probe / (time.perf_counter() - t0) / 1e9)
    del bufs
    return iso, conc


def place(policy, models, offs, cfgs, n_gpus, link_gbs, slo_s):
    """Placement of every request at its arrival.  naive: PP = 1 on GPU j mod n.  hydra: the
    library's contention-aware placement (hs_place_cold_start: Alg. 1 + Eq. 3/4 over the GPUs'
    host links, one link group per GPU with its measured isolated bandwidth)."""
    plans = []
    if policy == "naive":
        for j, m in enumerate(models):
            gpus = [dict(device=j % n_gpus, h2d_gbps=link_gbs[j % n_gpus], free_bytes=170 << 30)]
            plans.append(hs.plan_stages(cfgs[m], gpus, 1, 0))
        return plans
    links = hs.Links([g * 1e9 for g in link_gbs])
    gpus = [dict(device=d, h2d_gbps=link_gbs[d], link_group=d, free_bytes=170 << 30) for d in range(n_gpus)]
    for j, m in enumerate(models):
        pl, pred, ok, _ = links.place(cfgs[m], gpus, offs[j], slo_s, max_pp=n_gpus)
        plans.append(pl)
    return plans


def run(policy, models, offs, cfgs, imgs, n_gpus, link_gbs, slo_s):
    plans = place(policy, models, offs, cfgs, n_gpus, link_gbs, slo_s)
    groups = []
    for j, m in enumerate(models):
        groups.append(hs.Group(cfgs[m], plans[j], imgs[m], num_blocks=40, max_seqs=1, max_tokens=512))
    for d in range(n_gpus):
        torch.cuda.synchronize(d)
    prompts = {j: hsgen.prompts(1, 512, cfgs[m]["vocab"], 42 + j) for j, m in enumerate(models)}
    res = [None] * len(models)
    t0 = time.perf_counter() + 0.05

    def worker(j):
        g = groups[j]
        while time.perf_counter() < t0 + offs[j]:
            time.sleep(0.0002)
        ta = time.perf_counter()
        g.load_stage_async(-1)
        toks, _ = g.prefill([j], prompts[j])
        res[j] = dict(model=models[j], arrival_s=round(offs[j], 4), pp=plans[j].pp,
                      devices=[plans[j].device[k] for k in range(plans[j].pp)],
                      ttft_s=round(time.perf_counter() - ta, 4))

    th = [threading.Thread(target=worker, args=(j,)) for j in range(len(models))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    t_end = max(r["arrival_s"] + r["ttft_s"] for r in res)
    total = sum(sum(p.stage_bytes[k] for k in range(p.pp)) for p in plans)
    for g in groups:
        g.destroy()
    return dict(policy=policy, requests=res, mean_ttft_s=round(float(np.mean([r["ttft_s"] for r in res])), 4),
                max_ttft_s=round(max(r["ttft_s"] for r in res), 4),
                aggregate_h2d_gbs=round(total / t_end / 1e9, 1))


def main(n_gpus=None):
    n_gpus = n_gpus or torch.cuda.device_count()
    n_each = max(1, n_gpus // 2)
    models = [m for _ in range(n_each) for m in ("llama2-7b", "llama2-13b")]
    cfgs = {m: dict(hsgen.CONFIGS[m]) for m in set(models)}
    imgs = {}
    for m in sorted(cfgs):
        h = hs.image_layout(cfgs[m])
        imgs[m] = hs.HostImage(h, h.embed_off, h.total_bytes)
        hsgen.image_fill(hsgen.image_header(cfgs[m]), hsgen.WEIGHT_SEED, imgs[m].ptr, h.embed_off, h.total_bytes)
    offs = arrivals(len(models))
    link_gbs, conc = measure_links(n_gpus, imgs["llama2-7b"])
    slo = 0.25  # TTFT SLO (s): about one 7B PP=1 load over one link
    out = dict(n_gpus=n_gpus, models=models, arrivals_s=[round(x, 4) for x in offs],
               host_concurrent_h2d_gbs=round(conc, 1), link_gbs=[round(x, 1) for x in link_gbs], slo_ttft_s=slo,
               runs=[run(p, models, offs, cfgs, imgs, n_gpus, link_gbs, slo) for p in ("naive", "hydra")])
    return out


if __name__ == "__main__":
    print(json.dumps(main()))
