#!/bin/bash
# round-2 GPU run 46 (final code): launch list of a short bench (ncu gpu__time_duration, one ncu
# tool in this call, after the same command exited 0 without ncu) + final bench N=1 with the new probe
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build46.log 2>&1
timeout 900 python bench.py > gpurun_out/final46_n1.json 2> gpurun_out/final46_n1.err
CMD="python bench.py --steps 1 --warmup 1 --decode-steps 8 --no-cpu-baseline"
$CMD > gpurun_out/ncu46_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r02_final_launches.csv $CMD > gpurun_out/ncu46_list.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu46_list.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/smoke46.log 2>&1
