for dm in 8 12 16 20 24; do for sb in 2 4 8; do
  r=$(NGPRT_DECODE_MIN=$dm NGPRT_STEP_BURST=$sb timeout 120 python bench.py --steps 6 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['kernel_ms']['march_K1'],3))")
  echo "dm=$dm sb=$sb $r"
done; done
