#!/bin/bash
# round-2 GPU run 38: designated split merger with tagged partials (B=1) — parity subset + same-box A/B
# against libhs_base.so (HEAD abc8a7e)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build38.log 2>&1
timeout 1500 python -m pytest tests/test_group_gpu.py tests/test_fullsize_gpu.py -q -x -rA --timeout 900 -k "not 13b" > gpurun_out/gputest38.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest38.log
for r in 1 2 3; do
  HS_LIB_VARIANT=libhs_base.so timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b38_base_$r.json 2> gpurun_out/b38_base_$r.err
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b38_new_$r.json 2> gpurun_out/b38_new_$r.err
done
