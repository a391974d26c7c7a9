# Round-1 evidence: plain bench line, launch list, and a --set full capture of the decode GEMM.
set -x
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err
CMD="python bench.py --steps 1 --warmup 1 --decode-steps 8 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_r01b.csv $CMD > gpurun_out/ncu_launch.log 2>&1
$CMD > gpurun_out/ncu_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_sk -s 8 -c 4 -o gpurun_out/prof_sk_r01b $CMD > gpurun_out/ncu_full.log 2>&1
echo done
