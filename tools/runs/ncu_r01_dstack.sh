# Round-1 evidence for the decode stack: plain bench line, launch list, --set full capture of
# one dstack_kernel launch (each ncu pass only after the same command exited 0 without ncu).
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_r01c.json 2> gpurun_out/bench_r01c.err
CMD="python bench.py --steps 1 --warmup 1 --decode-steps 8 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_r01c.csv $CMD > gpurun_out/ncu_launch.log 2>&1
$CMD > gpurun_out/ncu_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dstack -s 4 -c 1 -o gpurun_out/prof_ds_r01c $CMD > gpurun_out/ncu_full.log 2>&1
echo done
