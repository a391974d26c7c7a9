#!/bin/bash
# round-2 GPU run 9: A/B plain runs (attention split granularity, O-proj split-K), then the ncu
# evidence (tools/r02_ncu.sh: launch list, full captures, load range counters)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build9.log 2>&1
for V in "" "HS_DSTACK_MINCH=64" "HS_DSTACK_MINCH=18"; do
  echo "== $V" >> gpurun_out/exp9.txt
  env $V timeout 300 python tools/trace_dstack.py > gpurun_out/t9.txt 2>&1
  head -2 gpurun_out/t9.txt >> gpurun_out/exp9.txt
  grep -E '"(qkv published|attn flags ok|attn kv done|E attn done|B1 o act|E o done|o grid-last)"' gpurun_out/t9.txt >> gpurun_out/exp9.txt
done
for V in "" "HS_TP2_SPLIT_MINKB=64"; do
  echo "== prefill $V" >> gpurun_out/exp9.txt
  env $V timeout 300 python tools/prefill_prof.py 512 >> gpurun_out/exp9.txt 2>&1
done
bash tools/runs/r02_ncu.sh
