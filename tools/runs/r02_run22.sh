#!/bin/bash
# round-2 GPU run 22: stream-K parts as tagged words (no per-part flag / fence) — parity, bench, traces
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build22.log 2>&1
timeout 1800 python -m pytest tests/test_group_gpu.py tests/test_kernels_gpu.py tests/test_fullsize_gpu.py -q -x -rA --timeout 1200 > gpurun_out/gputest22.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest22.log
for r in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/b22_$r.json 2> gpurun_out/b22_$r.err; done
timeout 900 python bench.py --config 4 --gpus 1 --steps 3 --warmup 3 > gpurun_out/b22_c4.json 2> gpurun_out/b22_c4.err
for K in 0 3; do
  HS_DSTACK_TRACE_K=$K TRACE_NPZ=gpurun_out/trace22_k$K.npz timeout 600 python tools/trace_dstack.py > gpurun_out/trace22_k$K.txt 2>&1
done
