#!/bin/bash
# round-2 GPU run 23: tagged stream-K parts, group re-polls — parity + bench B=1 / 13B B=16
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build23.log 2>&1
timeout 1800 python -m pytest tests/test_group_gpu.py tests/test_fullsize_gpu.py -q -x -rA --timeout 1200 > gpurun_out/gputest23.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest23.log
for r in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/b23_$r.json 2> gpurun_out/b23_$r.err; done
timeout 900 python bench.py --config 4 --gpus 1 --steps 3 --warmup 3 > gpurun_out/b23_c4.json 2> gpurun_out/b23_c4.err
HS_DSTACK_TRACE_K=3 TRACE_NPZ=gpurun_out/trace23_13b_k3.npz timeout 600 python tools/trace_dstack.py llama2-13b --batch 16 > gpurun_out/trace23_13b_k3.txt 2>&1
