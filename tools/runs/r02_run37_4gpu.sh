#!/bin/bash
# round-2 GPU run 37 (4 GPUs): final multi-GPU measurements, final decode stack
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build37.log 2>&1
nvidia-smi topo -m > gpurun_out/topo37.txt 2>&1
timeout 900 python -m pytest tests/test_spmd_gpu.py tests/test_group_gpu.py -q -rA --timeout 600 -k "spmd or two_gpu or pull" > gpurun_out/gputest37.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest37.log
HS_DEBUG_CONS=1 timeout 900 python bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/f37_n4.json 2> gpurun_out/f37_n4.err
HS_DEBUG_CONS=1 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/f37_n2.json 2> gpurun_out/f37_n2.err
HS_DEBUG_CONS=1 timeout 1200 python bench.py --gpus 4 --config 4 --steps 3 --warmup 3 > gpurun_out/f37_c4.json 2> gpurun_out/f37_c4.err
HS_DEBUG_CONS=1 timeout 1200 python bench.py --gpus 4 --config 4 --micro 4 --bg-pull --steps 3 --warmup 3 > gpurun_out/f37_c4_micro4_pull.json 2> gpurun_out/f37_c4_micro4_pull.err
HS_DEBUG_CONS=1 timeout 900 python bench.py --gpus 4 --scale-up --steps 3 --warmup 2 > gpurun_out/f37_n4_scaleup.json 2> gpurun_out/f37_n4_scaleup.err
timeout 900 python bench.py --config 5 > gpurun_out/f37_c5.json 2> gpurun_out/f37_c5.err
timeout 900 python bench.py --gpus 4 --impl reference --steps 1 --warmup 0 > gpurun_out/f37_n4_ref.json 2> gpurun_out/f37_n4_ref.err
