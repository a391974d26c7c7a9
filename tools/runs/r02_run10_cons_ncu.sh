#!/bin/bash
# round-2 GPU run 10 (2 GPUs, ONE process in local mode): NVLink counters of the consolidation
# copy (stage 1 on GPU 1 -> stage 0 on GPU 0) via ncu range replay
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python tools/ncu_ranges.py cons > gpurun_out/ncu_cons_plain.log 2>&1 &&
ncu --replay-mode app-range --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r02_cons_range.csv python tools/ncu_ranges.py cons > gpurun_out/ncu_cons.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_cons.log
