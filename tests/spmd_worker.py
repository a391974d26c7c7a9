"""One rank of the SPMD (one process per GPU) pipeline test, launched by
tests/test_spmd_gpu.py under torch.distributed.run.  Each rank owns one stage of the tiny
model (its own slice of the host image, its own GPU); activations and tokens cross over CUDA
IPC peer mappings, consolidation pulls the peer's weights and KV over NVLink.  The group is
created, run and destroyed ROUNDS times (as bench.py does per step).  Rounds 0 and 2 are
teacher-forced (decode inputs read from argv[1]) and write the logits each rank owns to
argv[2] + f".{rank}.npz"; round 1 decodes with hs_decode_steps (2 micro-batches in flight
through the stages, device feedback) and writes its tokens.  No oracle code runs here."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import hsgen  # noqa: E402
from paper_2502_15524_b200 import hs  # noqa: E402

CFG = hsgen.CONFIGS["tiny"]
PRE, POST = 8, 20  # decode steps before / after consolidation
ROUNDS = 3


def main():
    teacher = np.load(sys.argv[1])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    comm = hs.DistComm()
    h = hs.image_layout(CFG)
    gpus = [dict(device=d, h2d_gbps=50.0, free_bytes=8 << 30) for d in range(world)]
    plan = hs.plan_stages(CFG, gpus, world, 1)
    for k in range(world):
        plan.device[k] = k
    b, e = plan.as_dict()["slices"][rank]
    img = hs.HostImage(h, b, e)
    hsgen.image_fill(hsgen.image_header(CFG), hsgen.WEIGHT_SEED, img.ptr, b, e)
    prompts = hsgen.prompts(2, 32, CFG["vocab"])
    out = {}
    for r in range(ROUNDS):
        g = hs.Group(CFG, plan, None, [img if k == rank else None for k in range(world)],
                     num_blocks=64, max_seqs=8, max_tokens=256, comm=comm)
        last = rank == world - 1
        g.load_stage_async(-1)
        if r == 1:  # pipelined decode: 8 sequences as 2 micro-batches in flight (hs_decode_steps)
            ids8 = list(range(8))
            toks, _ = g.prefill(ids8, hsgen.prompts(8, 32, CFG["vocab"]))
            out[f"r{r}_tok0"] = np.array(toks)
            out[f"r{r}_ve"] = g.decode_steps(ids8, PRE, n_micro=2)
        else:
            toks, logits = g.prefill([0, 1], prompts, want_logits=last)
            out[f"r{r}_tok0"] = np.array(toks)
            if last:
                out[f"r{r}_log0"] = logits.copy()
            for step in range(1, PRE + 1):
                toks, logits = g.decode_step([0, 1], teacher[step - 1], want_logits=last)
                out[f"r{r}_tok{step}"] = np.array(toks)
                if last:
                    out[f"r{r}_log{step}"] = logits.copy()
        st = g.consolidate(0)
        out[f"r{r}_cons_bytes"] = np.array([st.weight_bytes, st.kv_bytes])
        if r % 2 == 0:  # the sources free their HBM before the target decodes on (else: at destroy)
            g.release_peer_memory()
        if rank == 0 and r != 1:
            for step in range(PRE + 1, POST + 1):
                toks, logits = g.decode_step([0, 1], teacher[step - 1], want_logits=True)
                out[f"r{r}_tok{step}"] = np.array(toks)
                out[f"r{r}_log{step}"] = logits.copy()
        dist.barrier()
        g.destroy()
    np.savez(sys.argv[2] + f".{rank}.npz", **out)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
