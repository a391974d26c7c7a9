#!/bin/bash
# round-2 GPU run 20: designated-finisher stream-K fix-up (HS_DSTACK_FINISHER) — parity, A/B, trace
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build20.log 2>&1
timeout 1800 python -m pytest tests/test_group_gpu.py tests/test_kernels_gpu.py tests/test_fullsize_gpu.py -q -x -rA --timeout 1200 > gpurun_out/gputest20.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest20.log
for r in 1 2; do
  for V in "HS_DSTACK_FINISHER=0" "HS_DSTACK_FINISHER=1"; do
    env $V timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/ab20_${V#HS_DSTACK_}_$r.json 2> gpurun_out/ab20_${V#HS_DSTACK_}_$r.err
  done
done
timeout 600 python tools/trace_dstack.py > gpurun_out/trace20_7b.txt 2>&1
timeout 600 python tools/trace_dstack.py llama2-13b --batch 16 > gpurun_out/trace20_13b_b16.txt 2>&1
for V in "HS_DSTACK_FINISHER=0" "HS_DSTACK_FINISHER=1"; do
  env $V timeout 900 python bench.py --config 4 --gpus 1 --steps 3 --warmup 3 > gpurun_out/ab20_c4_${V#HS_DSTACK_}.json 2> gpurun_out/ab20_c4_${V#HS_DSTACK_}.err
done
