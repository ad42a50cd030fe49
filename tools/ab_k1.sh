#!/bin/bash
# A/B K1 timing of library variants (tools/build_variant.py) and policy env
# settings: each argument is "<label>:<lib path or 'base'>:<env assignments>".
# Prints label, fps and K1/K2 ms of two short bench runs each. BENCH_ARGS adds
# bench.py arguments (e.g. BENCH_ARGS="--config c3_1080p_f32").
for spec in "$@"; do
  IFS=: read -r label lib envs <<< "$spec"
  [ "$lib" = base ] && lib="" 
  for rep in 1 2; do
    r=$(env NGPRT_LIB="$lib" $envs timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $BENCH_ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['kernel_ms']['march_K1'],4), round(d['kernel_ms']['shade_K2'],4))" 2>&1)
    echo "$label $rep $r"
  done
done
