CMD="python bench.py --steps 1 --warmup 1 --decode-steps 8 --no-cpu-baseline"
$CMD > gpurun_out/ncu_sk_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_sk -s 8 -c 4 -o gpurun_out/prof_sk_fused $CMD > gpurun_out/ncu_sk_fused.log 2>&1
tail -2 gpurun_out/ncu_sk_fused.log
