#!/bin/bash
# round-2 GPU run 5 (2 GPUs): SPMD + two-GPU tests, bench N=2 (config 3: PP=2 cold start +
# consolidation), scale-up at N=2
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo2.txt 2>&1
timeout 900 python -m pytest tests/test_spmd_gpu.py tests/test_group_gpu.py -q -rA --timeout 600 -k "spmd or two_gpu" > gpurun_out/gputest5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest5.log
HS_DEBUG_CONS=1 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "bench rc=$?" >> gpurun_out/bench_n2.err
HS_DEBUG_CONS=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 2 --scale-up > gpurun_out/bench_n2_scaleup.json 2> gpurun_out/bench_n2_scaleup.err; echo "bench rc=$?" >> gpurun_out/bench_n2_scaleup.err
timeout 600 python tools/stream_probe.py > gpurun_out/stream_probe2.txt 2>&1
