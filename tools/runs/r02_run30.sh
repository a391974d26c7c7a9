#!/bin/bash
# round-2 GPU run 36 (final code, 1 GPU; script r02_run30.sh): full GPU suite, smoke, bench N=1 + reference arm, then ONE
# ncu --set full capture of the decode stack (after the same command exited 0 without ncu)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build30.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rA --timeout 1200 > gpurun_out/gputest30.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest30.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke30.log 2>&1
for r in 1 2; do timeout 900 python bench.py > gpurun_out/final30_n1_$r.json 2> gpurun_out/final30_n1_$r.err; done
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/final30_ref.json 2> gpurun_out/final30_ref.err
timeout 900 python bench.py --config 4 --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final30_c4_pp1.json 2> gpurun_out/final30_c4_pp1.err
CMD="python bench.py --steps 1 --warmup 1 --decode-steps 8 --no-cpu-baseline"
$CMD > gpurun_out/ncu30_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:dstack_kernel -s 2 -c 1 -o gpurun_out/r02_final_dstack $CMD > gpurun_out/ncu30_ds.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu30_ds.log
