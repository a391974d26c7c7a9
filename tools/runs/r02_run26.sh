#!/bin/bash
# round-2 GPU run 26: reading R10b (RMSNorm scale after the GEMM) in the oracle, the prefill /
# per-kernel paths and the decode stack (per-tile operand flags, no grid-wide norm barrier)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build26.log 2>&1
timeout 900 python -m pytest tests/test_group_gpu.py -q -x -rA --timeout 600 > gpurun_out/gputest26a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest26a.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/b26_1.json 2> gpurun_out/b26_1.err
HS_DSTACK=0 timeout 600 python -m pytest tests/test_group_gpu.py -q -x --timeout 600 -k "layerwise" > gpurun_out/gputest26_perkernel.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest26_perkernel.log
timeout 2400 python -m pytest tests -m gpu -q -x -rA --timeout 1200 > gpurun_out/gputest26.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest26.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/b26_2.json 2> gpurun_out/b26_2.err
timeout 900 python bench.py --config 4 --gpus 1 --steps 3 --warmup 3 > gpurun_out/b26_c4.json 2> gpurun_out/b26_c4.err
HS_DSTACK_TRACE_K=3 TRACE_NPZ=gpurun_out/trace26_7b_k3.npz timeout 600 python tools/trace_dstack.py > gpurun_out/trace26_7b_k3.txt 2>&1
