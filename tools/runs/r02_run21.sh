#!/bin/bash
# round-2 GPU run 21: raw decode-stack traces with the fix-up stamps on each GEMM kind (tail analysis)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build21.log 2>&1
for K in 0 1 2 3; do
  HS_DSTACK_TRACE_K=$K TRACE_NPZ=gpurun_out/trace21_k$K.npz timeout 600 python tools/trace_dstack.py > gpurun_out/trace21_k$K.txt 2>&1
done
