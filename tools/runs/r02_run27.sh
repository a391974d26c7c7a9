#!/bin/bash
# round-2 GPU run 27: norm weight of the held tile read early (B=1) — parity subset, bench, traces of the O / gate_up fix-ups
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build27.log 2>&1
timeout 1500 python -m pytest tests/test_group_gpu.py tests/test_fullsize_gpu.py -q -x -rA --timeout 900 -k "not 13b" > gpurun_out/gputest27.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest27.log
for r in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/b27_$r.json 2> gpurun_out/b27_$r.err; done
for K in 1 2; do
  HS_DSTACK_TRACE_K=$K TRACE_NPZ=gpurun_out/trace27_7b_k$K.npz timeout 600 python tools/trace_dstack.py > gpurun_out/trace27_7b_k$K.txt 2>&1
done
