"""Builds the library of another git revision as paper_2502_15524_b200/libhs_<name>.so, for
same-box A/B of two builds (bench.py / tests load it with HS_LIB_VARIANT=libhs_<name>.so).
Measurement tooling only: the product loads libhs.so.

    python tools/build_variant.py <rev> <name>
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_15524_b200 import build as B  # noqa: E402


def main(rev: str, name: str) -> None:
    with tempfile.TemporaryDirectory() as tmp:
        # the revision's sources and headers (csrc/ includes ../../include)
        arch = subprocess.run(["git", "-C", ROOT, "archive", rev, "paper_2502_15524_b200/csrc", "include"],
                              check=True, capture_output=True).stdout
        subprocess.run(["tar", "-x", "-C", tmp], input=arch, check=True)
        csrc = os.path.join(tmp, "paper_2502_15524_b200", "csrc")
        objs, procs = [], []
        for f in sorted(os.listdir(csrc)):
            if not f.endswith((".cu", ".cc")):
                continue
            obj = os.path.join(tmp, f + ".o")
            cmd = [B.NVCC, *(["-x", "cu"] if f.endswith(".cc") else []), *B.ARCH, *B.FLAGS, "-c",
                   os.path.join(csrc, f), "-o", obj]
            procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
            objs.append(obj)
        for cmd, p in procs:
            out, _ = p.communicate()
            if p.returncode != 0:
                sys.stderr.write(out)
                raise SystemExit("nvcc failed: " + " ".join(cmd))
        so = os.path.join(ROOT, "paper_2502_15524_b200", f"libhs_{name}.so")
        subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", so, *objs, "-Xcompiler", "-fPIC"], check=True)
        print(so)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
