#!/bin/bash
# round-2 GPU run 17: run-to-run determinism of tiny prefill+decode with each prefill attention kernel
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build17.log 2>&1
for V in "HS_ATTN_TC=0" "HS_ATTN_TC=1" "HS_ATTN_TC=1"; do env $V timeout 600 python tools/prefill_det.py >> gpurun_out/det17.txt 2>&1; done
