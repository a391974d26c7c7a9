#!/bin/bash
# round-2 GPU run 24: early reads of the held tile's parts/residual + tagged o / a words (B=1) — parity, A/B, trace
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build24.log 2>&1
timeout 1800 python -m pytest tests/test_group_gpu.py tests/test_fullsize_gpu.py -q -x -rA --timeout 1200 > gpurun_out/gputest24.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest24.log
for r in 1 2; do
  for V in 0 1; do
    HS_DSTACK_TAGACT=$V timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/b24_tag${V}_$r.json 2> gpurun_out/b24_tag${V}_$r.err
  done
done
timeout 900 python bench.py --config 4 --gpus 1 --steps 3 --warmup 3 > gpurun_out/b24_c4.json 2> gpurun_out/b24_c4.err
for K in 0 1 3; do
  HS_DSTACK_TRACE_K=$K TRACE_NPZ=gpurun_out/trace24_7b_k$K.npz timeout 600 python tools/trace_dstack.py > gpurun_out/trace24_7b_k$K.txt 2>&1
done
