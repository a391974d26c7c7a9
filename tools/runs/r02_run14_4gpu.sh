#!/bin/bash
# round-2 GPU run 14 (4 GPUs): background NVLink pull (tests + config 3/4 benches: KV-only pause)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build14.log 2>&1
timeout 900 python -m pytest tests/test_group_gpu.py tests/test_spmd_gpu.py -q -rA --timeout 600 -k "pull or two_gpu or spmd" > gpurun_out/gputest14.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest14.log
HS_DEBUG_CONS=1 timeout 1200 python bench.py --gpus 4 --config 4 --micro 4 --bg-pull --steps 3 --warmup 3 > gpurun_out/bench_c4_pull.json 2> gpurun_out/bench_c4_pull.err; echo "bench rc=$?" >> gpurun_out/bench_c4_pull.err
HS_DEBUG_CONS=1 timeout 900 python bench.py --gpus 4 --bg-pull --steps 5 --warmup 3 > gpurun_out/bench_n4_pull.json 2> gpurun_out/bench_n4_pull.err; echo "bench rc=$?" >> gpurun_out/bench_n4_pull.err
