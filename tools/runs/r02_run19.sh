#!/bin/bash
# round-2 GPU run 19: O-producer split merge (HS_DSTACK_OMERGE) — parity and A/B at N = 1
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build19.log 2>&1
timeout 1500 python -m pytest tests/test_group_gpu.py tests/test_kernels_gpu.py tests/test_fullsize_gpu.py -q -x -rA --timeout 900 -k "not 13b" > gpurun_out/gputest19.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest19.log
for r in 1 2; do
  for V in 0 1; do
    HS_DSTACK_OMERGE=$V timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/ab19_om${V}_$r.json 2> gpurun_out/ab19_om${V}_$r.err
  done
done
