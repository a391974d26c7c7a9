# ncu full capture of one decode-stack launch (7B, B=1); run the same command without ncu first.
CMD="python tools/trace_dstack.py"
$CMD > gpurun_out/ds_plain.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:dstack -s 12 -c 1 -o gpurun_out/prof_ds $CMD > gpurun_out/ncu_ds.log 2>&1
tail -3 gpurun_out/ncu_ds.log
