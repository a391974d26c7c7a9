"""Builds libhs.so (the C-ABI library, sm_100a) in-tree with nvcc.  No torch involved."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libhs.so")
PROBES = os.path.join(HERE, "probes")
PROBE_SO = os.path.join(HERE, "libhs_probe.so")  # test-only hardware probes (never in libhs.so)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-diag-suppress", "177"]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cc")))


def headers():
    inc = os.path.join(os.path.dirname(HERE), "include")
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))] + \
        [os.path.join(inc, f) for f in os.listdir(inc)]


def probe_sources():
    return sorted(os.path.join(PROBES, f) for f in os.listdir(PROBES) if f.endswith(".cu"))


def stale() -> bool:
    if not os.path.exists(SO) or not os.path.exists(PROBE_SO):
        return True
    t = min(os.path.getmtime(SO), os.path.getmtime(PROBE_SO))
    return any(os.path.getmtime(f) > t for f in sources() + probe_sources() + headers())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return SO
    objs = []
    os.makedirs(os.path.join(HERE, "build"), exist_ok=True)
    procs = []
    for src in sources():
        obj = os.path.join(HERE, "build", os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
        if src.endswith(".cc"):
            cmd = [NVCC, "-x", "cu", *ARCH, *FLAGS, "-c", src, "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    logs = []
    for cmd, p in procs:
        out, _ = p.communicate()
        logs.append(out)
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    with open(os.path.join(HERE, "build", "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", SO, *objs, "-Xcompiler", "-fPIC"])
    # test-only probes: a separate library linked against libhs.so
    pobjs = []
    for src in probe_sources():
        obj = os.path.join(HERE, "build", "probe_" + os.path.basename(src) + ".o")
        subprocess.check_call([NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj], stdout=subprocess.DEVNULL)
        pobjs.append(obj)
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", PROBE_SO, *pobjs, "-Xcompiler", "-fPIC",
                           "-L" + HERE, "-lhs", "-Xlinker", "-rpath,$ORIGIN"])
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
