#!/bin/bash
# round-2 ncu evidence (one GPU, single process): launch list of a short bench, full capture of the
# decode stack and of a prefill CTA-pair GEMM, range counters (PCIe) of the 7B load
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --decode-steps 8 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
$CMD > gpurun_out/ncu_plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:dstack_kernel -s 2 -c 1 -o gpurun_out/r02_dstack $CMD > gpurun_out/ncu_ds.log 2>&1
$CMD > gpurun_out/ncu_plain3.log 2>&1 &&
ncu --set full --clock-control none -k regex:"gemm_tp2_kernel|attn_prefill_kernel|copy_list" -s 4 -c 2 -o gpurun_out/r02_prefill $CMD > gpurun_out/ncu_pre.log 2>&1
ncu --query-metrics > gpurun_out/ncu_query_metrics.txt 2>&1
python tools/ncu_ranges.py load > gpurun_out/ncu_plain4.log 2>&1 &&
ncu --replay-mode app-range --metrics gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum --csv --log-file gpurun_out/r02_load_range.csv python tools/ncu_ranges.py load > gpurun_out/ncu_range.log 2>&1
echo done >> gpurun_out/ncu_list.log
