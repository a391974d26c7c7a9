"""SPMD mode (one process per GPU, the product's multi-GPU launch): parity of the 2- and
4-rank pipeline and of its consolidation against the oracle, on BASELINE config 1 (tiny decoder, two
32-token prompts), teacher-forced, with the group created / run / consolidated / destroyed three
times in a row (repeated CUDA IPC export, mapping and release, as bench.py does per step).
Same acceptance as tests/test_group_gpu.py: max |logit - oracle| <= TOL on every step, and the
returned greedy tokens equal the oracle's except at ties (top-2 margin < 2x the logit error)."""
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
def oracle_hist():
    W = Weights(CFG)
    g = OGroup(CFG, W, pp=1, num_blocks=64)
    f = OGroup(CFG, W, pp=1, num_blocks=64, acc=np.float32)
    prompts = hsgen.prompts(2, 32, CFG["vocab"])
    toks, logits = g.prefill([0, 1], prompts)
    _, lf = f.prefill([0, 1], prompts)
    floor = [np.abs(logits - lf).max()]
    hist = [(np.array(toks), logits)]
    for _ in range(POST):
        t_in = toks
        toks, logits = g.decode([0, 1], t_in)
        _, lf = f.decode([0, 1], t_in)
        floor.append(np.abs(logits - lf).max())
        hist.append((np.array(toks), logits))
    return hist, max(2e-2, 1.5 * max(floor))


@pytest.mark.parametrize("world", [2, 4])
def test_spmd_pipeline_and_consolidation(oracle_hist, tmp_path, world):
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    hist, tol = oracle_hist
    teacher = tmp_path / "teacher.npy"
    np.save(teacher, np.stack([h[0] for h in hist]).astype(np.int32))
    out = str(tmp_path / "res")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(29400 + os.getpid() % 500 + world),
           os.path.join(HERE, "spmd_worker.py"), str(teacher), out]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-4000:]
    r0 = np.load(out + ".0.npz")
    r1 = np.load(out + f".{world - 1}.npz")  # the last stage returns the logits before consolidation
    for r in range(ROUNDS):
        assert r0[f"r{r}_cons_bytes"][0] > 0 and r0[f"r{r}_cons_bytes"][1] > 0
        for step in range(POST + 1):
            src = r1 if step <= PRE else r0
            logits = src[f"r{r}_log{step}"]
            ref_tok, ref_log = hist[step]
            err = np.abs(logits.astype(np.float64) - ref_log).max()
            assert err <= tol, f"round {r} step {step}: max |dlogit| {err} > {tol}"
            for rr in ((r0, r1) if step <= PRE else (r0,)):  # every rank returns the tokens
                tok = rr[f"r{r}_tok{step}"]
                for i in range(len(ref_tok)):
                    if tok[i] != ref_tok[i]:
                        top2 = np.sort(ref_log[i])[-2:]
                        assert top2[1] - top2[0] < 2 * err, f"round {r} step {step} seq {i}: mismatch without a tie"
