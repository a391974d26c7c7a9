#!/bin/bash
# round-2 GPU run 3: tiny GPU suite (decode_steps, prefetch watermark, chunked prefill), probes, bench N=1
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke3.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke3.log
timeout 1200 python -m pytest tests/test_group_gpu.py tests/test_kernels_gpu.py -q -rA --timeout 900 > gpurun_out/gputest3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest3.log
timeout 600 python tools/stream_probe.py > gpurun_out/stream_probe.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench rc=$?" >> gpurun_out/bench3.err
