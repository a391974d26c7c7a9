#!/usr/bin/env python3
"""Benchmark of the HydraServe cold-start path on B200 (BASELINE.json metric).

One *step* = one whole pass of the hot path over one synthetic request:
  plan (a1) -> T0: issue the chunked pinned-host->HBM load of every stage (a3, a4) ->
  prefill of the prompt through the stages (a5-a15; stage hand-offs a13) -> first token on
  the host (TTFT) -> D greedy decode steps (a16) -> [N > 1] consolidation into stage 0 (a17)
  -> D more decode steps on the single endpoint.
N = 1 runs BASELINE config 2 (Llama-2-7B shape, 512-token prompt, PP = 1); N > 1 (torchrun,
one process per GPU) runs config 3 (PP = N, one stage per GPU, CUDA-IPC peer memory over
NVLink).  --config 4 selects the 13B PP=4 16 x 512 workload.

value   = device-timed cold-start TTFT (s): per rank, CUDA events from the stage's first load
          chunk to the end of its prefill work (the last stage: token on host), max over ranks.
e2e     = the same TTFT on the host clock around the C-ABI calls (weights from pinned host
          memory, prompt H2D and token D2H inside), max over ranks.
Weights (13.5 GB) are larger than L2 (126 MB): no flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cold-start TTFT (s) and decode tok/s at PP=1/2/4/8; consolidation GB/s vs NVLink"
NVLINK_GBS = 900.0         # nominal per direction per GPU (north star); measured P2P 770
PROFILE_STEPS = int(os.environ.get("HS_PROFILE_STEPS", "8"))  # decode steps per timed step under the event profile


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:  # noqa
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "_fallback": True}


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, path):
        self.path = path
        self.p = None

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:  # noqa
            self.p = None

    def stop(self, n_gpus):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9 or not parts[0].isdigit() or int(parts[0]) >= n_gpus:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        loaded = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def workload(args, world):
    import hsgen
    cfgn = args.config or (2 if world == 1 else 3)
    if args.model:
        model = args.model
    else:
        model = "llama2-13b" if cfgn == 4 else "llama2-7b"
    cfg = dict(hsgen.CONFIGS[model])
    if cfgn == 4:
        n_seqs, plen, dsteps = 16, 512, 64
    else:
        n_seqs, plen, dsteps = 1, args.prompt_len, args.decode_steps
    if model == "tiny":
        plen = min(plen, 32)
    cfg["max_seq"] = max(cfg["max_seq"], plen + 2 * dsteps + 16)
    return cfgn, model, cfg, n_seqs, plen, dsteps


def run_ours(args):
    import numpy as np
    import torch

    import hsgen
    from paper_2502_15524_b200 import hs

    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    local = env_int("LOCAL_RANK", rank)
    if world != args.gpus:  # main() launches N ranks when WORLD_SIZE is unset: never measure N=1 as N
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dist = None
    comm = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = hs.DistComm()
    cfgn, model, cfg, n_seqs, plen, dsteps = workload(args, world)
    pp = world
    if cfgn == 4 and world == 1:
        pp = 1
    hdr = hs.image_layout(cfg)

    def gather(v):
        if not dist:
            return [v]
        t = torch.tensor([float(v)], dtype=torch.float64, device="cuda")
        out = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return [x.item() for x in out]

    # host->device link of every stage GPU, measured here from a 1 GiB pinned buffer: alone (one
    # rank at a time: p_i of Eq. 1/5, the load roofline's per-link peak) and all at once (shared
    # uplinks show up as a lower concurrent sum)
    iso_gbs, conc_gbs = link_probe(torch, dist, rank, world)
    p_iso = gather(iso_gbs)
    gpus = [dict(device=i, h2d_gbps=p_iso[i] if world > 1 else iso_gbs, free_bytes=torch.cuda.mem_get_info(local)[1])
            for i in range(pp)]
    plan = hs.plan_stages(cfg, gpus, pp, pp if args.scale_up else 1)
    for k in range(pp):
        plan.device[k] = k if world > 1 else local
    pd = plan.as_dict()
    # host image: this rank's stage slice (whole model at N = 1), pinned, pre-faulted
    b, e = pd["slices"][rank if world > 1 else 0] if world > 1 else (hdr.embed_off, hdr.total_bytes)
    if args.bg_load and rank == 0:  # the consolidation target streams the rest over its own link
        b, e = hdr.embed_off, hdr.total_bytes
    t_img = time.time()
    img = hs.HostImage(hdr, b, e)
    hsgen.image_fill(hsgen.image_header(cfg), hsgen.WEIGHT_SEED, img.ptr, b, e,
                     nthreads=max(1, cpu_cores() // max(1, world)))
    t_img = time.time() - t_img
    prompts = hsgen.prompts(n_seqs, plen, cfg["vocab"])
    ids = list(range(n_seqs))
    nb = n_seqs * ((plen + 2 * dsteps + 15) // 16 + 1) + 8
    kw = dict(num_blocks=nb, max_seqs=max(n_seqs, 1), max_tokens=n_seqs * plen, comm=comm)
    stage = rank if world > 1 else 0
    consolidate = world > 1

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def new_group():
        if world > 1:
            return hs.Group(cfg, plan, None, [img if k == rank else None for k in range(pp)], **kw)
        return hs.Group(cfg, plan, img, **kw)

    state = {"g": None}

    def one_step(profile):
        g = state["g"]
        if g is None:
            g = state["g"] = new_group()
        r = {}
        barrier()
        t0 = time.perf_counter()
        g.load_stage_async(-1, args.chunk_mb << 20)
        toks, _ = g.prefill(ids, prompts)
        t1 = time.perf_counter()
        r["ttft_host"] = t1 - t0
        r["ttft_dev"] = g.timing(stage).since_load_ms / 1e3
        r["load_ms"] = g.timing(stage).load_ms
        r["loaded_bytes"] = g.load_stats(stage).bytes
        if consolidate and args.bg_load:
            g.load_background_async(0, args.chunk_mb << 20)
        if consolidate and args.bg_pull:  # weights over NVLink before the pause: it moves KV only
            g.pull_background_async(0)
        dev = 0.0
        t2 = time.perf_counter()
        if args.micro > 1 and pp > 1:  # pipelined decode: micro-batches through the stages at once
            last_toks = g.decode_steps(ids, dsteps, n_micro=args.micro)[-1]
            dev += g.timing(stage).call_ms
        else:
            for _ in range(dsteps):
                last_toks, _ = g.decode_step(ids)
                dev += g.timing(stage).call_ms
        r["decode_host"] = time.perf_counter() - t2
        r["decode_dev"] = dev / 1e3
        if profile:  # per-kernel event profile on extra decode steps (events break PDL overlap)
            g.profile(True)
            for _ in range(PROFILE_STEPS):
                g.decode_step(ids)
            g.profile(False)
        if consolidate and args.scale_up:
            # every stage becomes an endpoint (all-gather of the weights + each sequence's KV)
            eps, st = g.scale_up()
            r["cons_s"], r["cons_pause"] = st.seconds, st.pause_seconds
            r["cons_bytes"] = st.weight_bytes + st.kv_bytes
            r["cons_w"], r["cons_kv"], r["cons_w_host"] = st.weight_bytes, st.kv_bytes, 0
            ep = eps[0]
            if rank == 0:  # sequence 0 lives on endpoint 0
                dev2 = 0.0
                t3 = time.perf_counter()
                ep.decode_step(ids, last_toks)
                for _ in range(dsteps - 1):
                    ep.decode_step(ids)
                    dev2 += ep.timing(0).call_ms
                r["decode2_host"] = time.perf_counter() - t3
                r["decode2_dev"] = dev2 / 1e3
            r["prof"] = g.profile_read(reset=True) if profile else {}
            barrier()
            g.destroy()  # closes this rank's peer mappings (collective) before the endpoints free
            for e in eps:
                e.destroy()
            state["g"] = None
            return r
        if consolidate:
            st = g.consolidate(0)
            r["cons_s"] = st.seconds
            r["cons_pause"] = st.pause_seconds
            r["cons_bytes"] = st.weight_bytes + st.kv_bytes
            r["cons_w"], r["cons_kv"] = st.weight_bytes, st.kv_bytes
            r["cons_w_host"] = st.weight_bytes_host
            r["cons_w_bg"] = st.weight_bytes_background
            if rank == 0:
                dev2 = 0.0
                t3 = time.perf_counter()
                for _ in range(dsteps):
                    g.decode_step(ids)
                    dev2 += g.timing(0).call_ms
                r["decode2_host"] = time.perf_counter() - t3
                r["decode2_dev"] = dev2 / 1e3
        r["prof"] = g.profile_read(reset=True) if profile else {}
        if consolidate:
            g.release_peer_memory()  # collective: the sources' released HBM is freed here
            barrier()
            g.destroy()
            state["g"] = None
        else:
            for i in ids:
                g.release_seq(i)
            if profile:  # warm prefill (weights resident) for the per-kernel prefill profile
                g.profile(True)
                g.prefill(ids, prompts)
                g.profile(False)
                r["prof"] = g.profile_read(reset=True) | {k: v for k, v in r["prof"].items() if k.endswith(".decode")}
                for i in ids:
                    g.release_seq(i)
        return r

    for _ in range(args.warmup):
        one_step(False)
    clocks = Clocks(os.path.join(ROOT, "gpurun_out", f"clocks_r{rank}.csv")) if rank == 0 else None
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    barrier()
    l0 = hs.Group.launch_count()
    if clocks:
        clocks.start()
    steps = [one_step(True) for _ in range(args.steps)]
    barrier()
    launches = hs.Group.launch_count() - l0
    ck = clocks.stop(world) if clocks else None

    def agg_max(v):
        if not dist:
            return v
        t = torch.tensor([float(v)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def agg_sum(v):
        if not dist:
            return v
        t = torch.tensor([float(v)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.item()

    med = lambda k: statistics.median(s[k] for s in steps)  # noqa: E731
    ttft_dev = agg_max(med("ttft_dev"))
    ttft_host = agg_max(med("ttft_host"))
    load_ms = agg_max(med("load_ms"))
    loaded = agg_sum(med("loaded_bytes"))
    dec_dev = agg_max(med("decode_dev"))
    dec_host = agg_max(med("decode_host"))
    launches = int(agg_sum(launches))
    h2d_concurrent = agg_sum(conc_gbs)
    h2d_isolated_sum = agg_sum(iso_gbs)
    # per-kind profile (this rank) -> dominant decode GEMM
    prof = {}
    for s in steps:
        for k, v in s["prof"].items():
            a = prof.setdefault(k, dict(count=0, ms=0.0, bytes=0.0, flops=0.0))
            for f in a:
                a[f] += v[f]
    pk = peaks()
    # dominant decode kernel: the decode stack (every layer of a stage in one launch); the
    # per-kernel path (HS_DSTACK=0) reports its stream-K decode GEMMs instead
    if "decode_stack.decode" in prof:
        dec_gemm = [prof["decode_stack.decode"]]
        kname = ("dstack_kernel<16> (decode stack: all decoder layers of the stage in one persistent tcgen05/TMA "
                 "kernel per step; weights + KV read/write per launch)")
        traffic_file = "r02_decode_stack_traffic.json"
    else:
        dec_gemm = [v for k, v in prof.items() if k.startswith("gemm_") and k.endswith(".decode") and "lm_head" not in k]
        kname = "gemm_sk_kernel<16> (tcgen05 stream-K weight-streaming decode GEMM: qkv/o/gate_up/down, fused epilogues)"
        traffic_file = "r01_decode_gemm_traffic.json"
    g_ms = sum(v["ms"] for v in dec_gemm)
    g_bytes = sum(v["bytes"] for v in dec_gemm)
    g_count = sum(v["count"] for v in dec_gemm)
    achieved = (g_bytes / (g_ms / 1e3) / 1e9) if g_ms > 0 else 0.0
    roof = {"kernel": kname,
            "bound": "hbm", "achieved": round(achieved, 1),
            "peak": pk.get("hbm_gbs"), "unit": "GB/s",
            "frac": round(achieved / pk.get("hbm_gbs", 6650.0), 4), "traffic": None,
            "bytes_per_launch": (g_bytes / g_count) if g_count else None,
            "ms_per_launch": (g_ms / g_count) if g_count else None,
            "share_of_kernel_time": round(g_ms / max(1e-9, sum(v["ms"] for k, v in prof.items() if k.endswith(".decode"))), 3),
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if not pk.get("_fallback") else "fallback"}
    try:  # dram__bytes_read + write per launch of this kernel from the committed ncu --set full capture
        tr = json.load(open(os.path.join(ROOT, "profiles", traffic_file)))
        alg = tr.get("algorithmic_bytes_per_launch")
        bpl = roof["bytes_per_launch"]
        if alg and bpl and abs(bpl - alg) <= 0.02 * alg:  # the captured launch is this workload's launch
            roof["traffic"] = round(tr["mean_bytes_per_launch"])
            roof["traffic_source"] = tr["source"]
        else:
            roof["traffic_note"] = ("no ncu --set full capture of this workload's launch (the committed one, " +
                                    tr["source"] + ", is " + tr["launches"][0] + ")")
    except Exception:  # noqa
        pass
    pre_gemm = [v for k, v in prof.items() if k.startswith("gemm_") and k.endswith(".prefill")]
    out = None
    if rank == 0:
        agg_link = h2d_isolated_sum
        load_gbs = loaded / (load_ms / 1e3) / 1e9
        out = {
            "metric": METRIC, "value": round(ttft_dev, 5), "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * statistics.median(
                s["ttft_host"] + s["decode_host"] + s.get("decode2_host", 0) + s.get("cons_pause", 0) for s in steps), 2),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init Llama-2-shaped weights, seeded; uniform random prompt tokens)",
            "config": {"workload": f"config {cfgn}: {model} PP={pp}, {n_seqs}x{plen}-token prompt, "
                                   f"{dsteps} greedy decode steps" + (", consolidate to stage 0, "
                                                                      f"{dsteps} more steps" if consolidate else ""),
                       "pp": pp, "prompt_tokens": plen, "n_seqs": n_seqs, "decode_steps": dsteps,
                       "decode_micro_batches": args.micro if (args.micro > 1 and pp > 1) else 1,
                       "chunk_mb": args.chunk_mb, "l2": "inputs > L2 (weights 13.5 GB), no flush needed",
                       "parallelism": f"pp{pp} (one process per GPU)" if world > 1 else "pp1"},
            "ttft": {"device_s": round(ttft_dev, 5), "host_s": round(ttft_host, 5),
                     "pred_eq5_s": round(pd["pred_ttft_s"], 5),
                     "per_step_device_s": [round(s["ttft_dev"], 5) for s in steps]},
            "load": {"bytes_per_stage_max": max(pd["stage_bytes"]), "bytes_total": int(loaded),
                     "stage_load_ms_max": round(load_ms, 2), "achieved_gbs": round(load_gbs, 2),
                     "peak_gbs_isolated_sum": round(agg_link, 1),
                     "peak_gbs_isolated_per_gpu": [round(x, 1) for x in p_iso],
                     "frac_of_isolated_sum": round(load_gbs / agg_link, 4),
                     "peak_gbs_measured_concurrent": round(h2d_concurrent, 1),
                     "frac_of_measured_concurrent": round(load_gbs / h2d_concurrent, 4)},
            "decode": {"tok_s_device": round(n_seqs * dsteps / dec_dev, 2), "tok_s_host": round(n_seqs * dsteps / dec_host, 2),
                       "hbm_roofline_tok_s": None},
            "roofline": roof,
            "kernels": {k: {"count": v["count"], "ms": round(v["ms"], 3),
                            "gbs": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1) if v["ms"] else None,
                            "tflops": round(v["flops"] / (v["ms"] / 1e3) / 1e12, 2) if v["ms"] and v["flops"] else None}
                        for k, v in sorted(prof.items())},
            "prefill_gemm_tflops": round(sum(v["flops"] for v in pre_gemm) / max(1e-9, sum(v["ms"] for v in pre_gemm) / 1e3) / 1e12, 1),
            "gpu_launches": launches,
            "clocks": ck,
            "e2e": {"value": round(ttft_host, 5), "unit": "s", "h2d_bytes_per_step": int(loaded + plen * n_seqs * 4),
                    "d2h_bytes_per_step": int(4 * n_seqs * (1 + dsteps * (2 if consolidate else 1)))},
            "image_gen_s": round(t_img, 2),
        }
        # decode roofline: weights (minus embedding) + KV read per step
        H, L, V = cfg["hidden"], cfg["n_layers"], cfg["vocab"]
        wbytes = hdr.param_bytes - 2 * V * H
        kv = n_seqs * (plen + dsteps // 2) * 2 * H * 2 * L
        out["decode"]["hbm_roofline_tok_s"] = round(n_seqs / ((wbytes + kv) / (pk.get("hbm_gbs", 6650) * 1e9)), 1)
        if consolidate:
            cs = statistics.median(s["cons_s"] for s in steps)
            cb = statistics.median(s["cons_bytes"] for s in steps)
            out["consolidation"] = {"mode": "scale-up (all-gather to every stage)" if args.scale_up else "scale-down to stage 0",
                                    "bytes": int(cb), "weight_bytes": int(steps[0]["cons_w"]), "kv_bytes": int(steps[0]["cons_kv"]),
                                    "weight_bytes_via_host_background": int(steps[0]["cons_w_host"]),
                                    "weight_bytes_pulled_before_pause": int(steps[0].get("cons_w_bg", 0)),
                                    "seconds": round(cs, 5), "gbs": round(cb / cs / 1e9, 1),
                                    "frac_of_nvlink_900": round(cb / cs / 1e9 / NVLINK_GBS, 4),
                                    "pause_s": round(statistics.median(s["cons_pause"] for s in steps), 4)}
            out["decode"]["after_consolidation_tok_s_device"] = round(
                n_seqs * dsteps / statistics.median(s["decode2_dev"] for s in steps), 2)
        # every part of the path against its own roofline (the "roofline" key above is the
        # dominant kernel, the decode stack): load / PCIe, prefill GEMMs / tensor, decode / HBM,
        # consolidation / NVLink
        pre_ms = sum(v["ms"] for v in pre_gemm)
        pre_tf = sum(v["flops"] for v in pre_gemm) / max(1e-12, pre_ms / 1e3) / 1e12
        rl = [{"part": "load (a3)", "bound": "pcie", "achieved": round(load_gbs, 2), "unit": "GB/s",
               "peak": round(agg_link, 1), "frac": round(load_gbs / agg_link, 4),
               "peak_source": f"sum over the {pp} stage GPUs of the isolated pinned-H2D probe in this run"},
              {"part": "prefill GEMMs (a7, a10-a12, a14), warm", "bound": "tensor", "achieved": round(pre_tf, 1),
               "unit": "TFLOP/s", "peak": pk.get("bf16_tflops"), "frac": round(pre_tf / pk.get("bf16_tflops", 1659.3), 4),
               "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst: a prefill is a few ms)"},
              {"part": "decode stack (a16)", "bound": "hbm", "achieved": roof["achieved"], "unit": "GB/s",
               "peak": roof["peak"], "frac": roof["frac"], "peak_source": roof["peak_source"]}]
        if consolidate:
            cgbs = statistics.median(s["cons_bytes"] for s in steps) / statistics.median(s["cons_s"] for s in steps) / 1e9
            rl.append({"part": "consolidation (a17)", "bound": "nvlink", "achieved": round(cgbs, 1), "unit": "GB/s",
                       "peak": NVLINK_GBS, "frac": round(cgbs / NVLINK_GBS, 4),
                       "peak_source": "NVLink 5 nominal per direction (target ingress)"})
        out["rooflines"] = rl
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(cfg, plen, n_seqs)
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return out


def link_probe(torch, dist, rank, world, nbytes=1 << 30):
    """Pinned host -> HBM copy bandwidth of this rank's GPU (GB/s): isolated (the ranks take
    turns) and concurrent (all at once); best of 5 each, CUDA events around the copy of 1 GiB
    as 32 back-to-back 32 MiB copies (the loader's chunk size)."""
    src = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    src.fill_(1)
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    chunk = 32 << 20

    def timed():
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for o in range(0, nbytes, chunk):
                dst[o:o + chunk].copy_(src[o:o + chunk], non_blocking=True)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        return nbytes / best / 1e9

    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    iso = 0.0
    for r in range(world):
        if dist:
            dist.barrier()
        if r == rank:
            iso = timed()
    if dist:
        dist.barrier()
    conc = timed()
    del src, dst
    return iso, conc


def oracle_sample(cfg, plen, n_seqs, decode_steps=4, layers=1):
    """The oracle as it stands, on a bounded sample of the workload: the real prompt(s) through
    `layers` decoder layers (+ embedding, final norm, lm_head), then `decode_steps` cached decode
    steps; per-layer times extrapolated linearly to all layers.  Weights are drawn before the
    timer (input generation is not the oracle's work).  Returns (prefill_s, decode_s_per_step,
    sampled seconds)."""
    import hsgen
    from oracle.decoder import Group, Weights
    W = Weights(cfg, cache=True)
    sub = dict(cfg)
    sub["n_layers"] = layers
    for l in range(layers):
        W.layer(l)
    W.lm_head()
    W.final_norm()
    prompts = hsgen.prompts(n_seqs, plen, cfg["vocab"])
    ids = list(range(n_seqs))
    g = Group(sub, W, pp=1, num_blocks=n_seqs * ((plen + decode_steps) // 16 + 2))
    t0 = time.perf_counter()
    toks, _ = g.prefill(ids, prompts)
    t_pre = time.perf_counter() - t0
    t1 = time.perf_counter()
    for _ in range(decode_steps):
        toks, _ = g.decode(ids, toks)
    t_dec = (time.perf_counter() - t1) / max(1, decode_steps)
    L = cfg["n_layers"]
    return t_pre * L / layers, t_dec * L / layers, t_pre + t_dec * decode_steps


def oracle_copy_gbs(nbytes=1 << 30, piece=None):
    """The oracle's load and consolidation are byte copies: host memcpy
    bandwidth of numpy copies, whole (load: a stage slice) or in KV-block pieces."""
    import numpy as np
    src = np.ones(nbytes, dtype=np.uint8)
    dst = np.empty_like(src)
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        if piece:
            for o in range(0, nbytes, piece):
                dst[o:o + piece] = src[o:o + piece]
        else:
            np.copyto(dst, src)
        best = min(best, time.perf_counter() - t0)
    return nbytes / best / 1e9


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # noqa
        return os.cpu_count()


def cpu_baseline(cfg, plen, n_seqs):
    """CPU oracle on this host (SURVEY §8(d) "CPU oracle beside it"): TTFT-equivalent = load
    (memcpy of the model image at the oracle's copy bandwidth) + prefill; decode s/token;
    consolidation copy GB/s (KV-block pieces)."""
    import hsgen
    pre, dec, sampled = oracle_sample(cfg, plen, n_seqs)
    load_gbs = oracle_copy_gbs()
    kv_block = 16 * 2 * cfg["hidden"] * 2
    cons_gbs = oracle_copy_gbs(piece=kv_block)
    img = hsgen.image_header(cfg).param_bytes
    ttft = img / (load_gbs * 1e9) + pre
    return {"value": round(ttft, 3), "unit": "s", "cores": cpu_cores(), "kind": "oracle",
            "prefill_s": round(pre, 3), "load_s": round(img / (load_gbs * 1e9), 3), "load_gbs": round(load_gbs, 2),
            "decode_s_per_token": round(dec / n_seqs, 4), "decode_tok_s": round(n_seqs / dec, 3),
            "consolidation_copy_gbs": round(cons_gbs, 2),
            "sample": f"numpy-fp64 oracle: the {n_seqs}x{plen}-token prefill and 4 cached decode steps through 1 of "
                      f"{cfg['n_layers']} layers (+ embedding, lm_head) in {sampled:.2f} s, extrapolated x{cfg['n_layers']}; "
                      f"load = {img / 1e9:.2f} GB image at the measured numpy copy bandwidth (1 GiB sample); "
                      f"consolidation copy = 1 GiB in {kv_block // 1024} KiB KV-block pieces; value = load + prefill"}


def run_reference(args):
    """--impl reference: the CPU oracle as it stands on this host, the same workload and metric
    (TTFT-equivalent: image load at the oracle's copy bandwidth + prefill), each step a bounded
    sample (cpu_baseline).  Under torchrun only rank 0 works."""
    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    if rank != 0:
        return
    cfgn, model, cfg, n_seqs, plen, dsteps = workload(args, world)
    vals, last = [], None
    for i in range(args.warmup + args.steps):
        last = cpu_baseline(cfg, plen, n_seqs)
        if i >= args.warmup:
            vals.append(last["value"])
    v = statistics.median(vals)
    cb = dict(last)
    cb["value"] = round(v, 3)
    out = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "higher_is_better": False, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"config {cfgn}: {model}, {n_seqs}x{plen}-token prompt (oracle TTFT-equivalent)"},
           "cpu_baseline": cb,
           "e2e": {"value": round(v, 3), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def relaunch(n):
    """`python bench.py --gpus N` without a launcher: start N ranks (one process per GPU) with
    torch.distributed.run on 127.0.0.1 and pass their output and exit status through."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=0)
    ap.add_argument("--model", default="")
    ap.add_argument("--prompt-len", type=int, default=512)
    ap.add_argument("--decode-steps", type=int, default=64)
    ap.add_argument("--chunk-mb", type=int, default=32)
    ap.add_argument("--micro", type=int, default=0,
                    help="N>1: decode the batch as this many micro-batches flowing through the stages "
                         "concurrently (hs_decode_steps, 'virtual engines'); 0 = one step per call")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scale-up", action="store_true",
                    help="N>1: every stage becomes a standalone endpoint (scale-up consolidation) instead of "
                         "scale-down into stage 0")
    ap.add_argument("--bg-pull", action="store_true",
                    help="N>1: the target pulls the other stages' weights over NVLink in the background after "
                         "the first token; the consolidation pause then moves KV only")
    ap.add_argument("--bg-load", action="store_true",
                    help="N>1: the target loads the other stages' weights over its own PCIe link in the "
                         "background after the first token (paper's mechanism); consolidation moves KV only")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.config != 5:
        sys.exit(relaunch(args.gpus))
    if args.config == 5:
        run_burst(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


def run_burst(args):
    """BASELINE config 5 (one process, all visible GPUs): bursty simultaneous cold starts of
    mixed 7B / 13B models, naive vs contention-aware placement (tools/burst.py)."""
    if args.impl == "reference":
        print(json.dumps({"impl": "reference", "unavailable": "config 5 is a placement scenario of the GPU path; "
                          "the oracle has no load / placement model to time"}))
        return
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import burst
    r = burst.main()
    hy = next(x for x in r["runs"] if x["policy"] == "hydra")
    nv = next(x for x in r["runs"] if x["policy"] == "naive")
    print(json.dumps({
        "metric": "config 5 burst cold-start TTFT (s, mean over requests)", "value": hy["mean_ttft_s"], "unit": "s",
        "n_gpus": r["n_gpus"], "steps": 1, "warmup": 0, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init Llama-2-shaped weights, seeded)",
        "config": {"workload": f"config 5 ({r['n_gpus']}-GPU variant): " + ", ".join(r["models"]) +
                               "; Gamma(CV=8, rate 8/s, seed 7) arrivals; 1 x 512-token prompt each",
                   "parallelism": "per-request PP chosen at arrival"},
        "naive_mean_ttft_s": nv["mean_ttft_s"], "hydra_mean_ttft_s": hy["mean_ttft_s"],
        "naive_max_ttft_s": nv["max_ttft_s"], "hydra_max_ttft_s": hy["max_ttft_s"],
        "detail": r}))


if __name__ == "__main__":
    main()
