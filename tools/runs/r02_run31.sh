#!/bin/bash
# round-2 GPU run 31: attention units on half CTAs (HS_DSTACK_AHALF) — parity subset, A/B B=1 and 13B B=16
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build31.log 2>&1
timeout 1500 python -m pytest tests/test_group_gpu.py tests/test_fullsize_gpu.py -q -x -rA --timeout 900 > gpurun_out/gputest31.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest31.log
for r in 1 2; do
  for V in 0 1; do
    HS_DSTACK_AHALF=$V timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b31_ah${V}_$r.json 2> gpurun_out/b31_ah${V}_$r.err
  done
done
for V in 0 1; do
  HS_DSTACK_AHALF=$V timeout 900 python bench.py --config 4 --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b31_c4_ah$V.json 2> gpurun_out/b31_c4_ah$V.err
done
