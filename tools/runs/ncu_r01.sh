set -x
CMD="python bench.py --steps 1 --warmup 1 --decode-steps 8 --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_r01.csv $CMD > gpurun_out/ncu_launch.log 2>&1 ; \
$CMD > gpurun_out/ncu_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 300 -c 4 -o gpurun_out/prof_gemm_r01 $CMD > gpurun_out/ncu_full.log 2>&1
echo done
