#!/bin/bash
# round-2 GPU run 6 (4 GPUs): SPMD 4-rank test, bench N=4 (config 3), config 4 (13B PP=4, 16 x 512,
# consolidation mid-decode) stepwise and with 4 decode micro-batches, config 5 burst placement
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo4.txt 2>&1
timeout 900 python -m pytest tests/test_spmd_gpu.py -q -rA --timeout 600 > gpurun_out/gputest6.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest6.log
HS_DEBUG_CONS=1 timeout 900 python bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo "bench rc=$?" >> gpurun_out/bench_n4.err
HS_DEBUG_CONS=1 timeout 1200 python bench.py --gpus 4 --config 4 --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?" >> gpurun_out/bench_c4.err
HS_DEBUG_CONS=1 timeout 1200 python bench.py --gpus 4 --config 4 --micro 4 --steps 3 --warmup 3 > gpurun_out/bench_c4_micro4.json 2> gpurun_out/bench_c4_micro4.err; echo "bench rc=$?" >> gpurun_out/bench_c4_micro4.err
timeout 900 python bench.py --config 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench rc=$?" >> gpurun_out/bench_c5.err
