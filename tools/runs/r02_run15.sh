#!/bin/bash
# round-2 GPU run 15: prefill GEMM kernel choice per shape (HS_TP_BN forces one kernel for every GEMM)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build15.log 2>&1
for V in "" "HS_TP_BN=128" "HS_TP_BN=256" "HS_TP_BN=2128" "HS_TP_BN=2256" "HS_TP2=0"; do
  for T in 512 1024 2048; do
    echo "== $V T=$T" >> gpurun_out/exp15.txt
    env $V timeout 300 python tools/prefill_prof.py $T 2>&1 | grep -E "prefill_ms|gemm" >> gpurun_out/exp15.txt
  done
done
