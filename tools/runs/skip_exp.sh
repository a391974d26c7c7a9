for k in 0 1 2 4 8 16 32 31 63; do
  HS_DEBUG_SKIP=$k timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('skip', $k, 'ms/step', round(1000/d['decode']['tok_s_device'],3))"
done
