"""SPMD mode (one process per GPU, the product's multi-GPU launch): the 2- and 4-rank pipeline
and its consolidation on BASELINE config 1 (tiny decoder, two 32-token prompts), teacher-forced,
with the group created / run / consolidated / destroyed three times in a row (repeated CUDA IPC
export, mapping and release, as bench.py does per step), and one round of pipelined decode
(hs_decode_steps, 8 sequences as 2 micro-batches in flight).  Acceptance: bitwise equal to the
same calls on a single-process PP=1 group in this process (a pipeline group
computes exactly the unpartitioned model; the PP=1 path is layer-level equal to the oracle in
tests/test_group_gpu.py), every step's logits and tokens, before and after consolidation."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import hsgen  # noqa: E402
from oracle.decoder import Group as OGroup, Weights  # noqa: E402

CFG = hsgen.CONFIGS["tiny"]
HERE = os.path.dirname(os.path.abspath(__file__))
PRE, POST, ROUNDS = 8, 20, 3


@pytest.fixture(scope="module")
def reference():
    """Single-process PP=1 run of the same calls on cuda:0: teacher-forced logits/tokens of the
    two prompts (teacher = the oracle's greedy tokens), and the free-running tokens of 8 prompts."""
    from paper_2502_15524_b200 import hs
    W = Weights(CFG)
    og = OGroup(CFG, W, pp=1, num_blocks=64)
    prompts = hsgen.prompts(2, 32, CFG["vocab"])
    toks, _ = og.prefill([0, 1], prompts)
    teacher = [np.array(toks)]
    for _ in range(POST):
        toks, _ = og.decode([0, 1], toks)
        teacher.append(np.array(toks))
    h = hs.image_layout(CFG)
    img = hs.HostImage(h, 0, h.total_bytes)
    hsgen.image_fill(hsgen.image_header(CFG), hsgen.WEIGHT_SEED, img.ptr, 0, h.total_bytes)
    plan = hs.plan_stages(CFG, [dict(device=0, h2d_gbps=50.0, free_bytes=8 << 30)], 1, 1)
    g = hs.Group(CFG, plan, img, num_blocks=64, max_seqs=8, max_tokens=256)
    g.load_stage_async(-1)
    ref = [g.prefill([0, 1], prompts, want_logits=True)]
    for step in range(1, POST + 1):
        ref.append(g.decode_step([0, 1], teacher[step - 1], want_logits=True))
    g.destroy()
    g = hs.Group(CFG, plan, img, num_blocks=64, max_seqs=8, max_tokens=256)
    g.load_stage_async(-1)
    ve = [g.prefill(list(range(8)), hsgen.prompts(8, 32, CFG["vocab"]))[0]]
    for _ in range(PRE):
        ve.append(g.decode_step(list(range(8)))[0])
    g.destroy()
    return np.stack(teacher), ref, np.stack(ve)


@pytest.mark.parametrize("world", [2, 4])
def test_spmd_pipeline_and_consolidation(reference, tmp_path, world):
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    teacher_toks, ref, ve_ref = reference
    teacher = tmp_path / "teacher.npy"
    np.save(teacher, teacher_toks.astype(np.int32))
    out = str(tmp_path / "res")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(29400 + os.getpid() % 500 + world),
           os.path.join(HERE, "spmd_worker.py"), str(teacher), out]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-4000:]
    r0 = np.load(out + ".0.npz")
    r1 = np.load(out + f".{world - 1}.npz")  # the last stage returns the logits before consolidation
    for r in (0, 2):
        assert r0[f"r{r}_cons_bytes"][0] > 0 and r0[f"r{r}_cons_bytes"][1] > 0
        for step in range(POST + 1):
            src = r1 if step <= PRE else r0
            assert np.array_equal(src[f"r{r}_log{step}"], ref[step][1]), (r, step)
            for rr in ((r0, r1) if step <= PRE else (r0,)):  # every rank returns the tokens
                assert np.array_equal(rr[f"r{r}_tok{step}"], ref[step][0]), (r, step)
    # pipelined decode (2 micro-batches in flight) == stepwise PP=1 decode, on both end ranks
    for rr in (r0, r1):
        assert np.array_equal(rr["r1_tok0"], ve_ref[0])
        assert np.array_equal(rr["r1_ve"], ve_ref[1:])
