# All BASELINE configs on one B200 (tensor MLP), one JSON line each -> gpurun_out/configs_<tag>.jsonl
tag=${1:-r01}
out=gpurun_out/configs_$tag.jsonl; : > $out
run() { timeout 600 python bench.py --steps ${STEPS:-8} --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | tail -1 >> $out; }
run --config c1_256
run --config c2_blob800
run --config c2_blob800 --batch 50
run --config c3_1080p
run --config c3_1080p --mlp exact
run --config c3_1080p_f32
run --config c3_mip360
run --config c3_1080p --shard tiles
run --config c4_1080p_x64
run --config c4_1080p_x64 --batch 64
for nb in 10 35 140 560 2240; do run --config c5_2160p --scene n_boxes=$nb; done
run --config c5_2160p --shard tiles
python - <<'PY' $out
import json,sys
for l in open(sys.argv[1]):
    if not l.strip(): continue
    d=json.loads(l); c=d["config"]
    print(f'{c["workload"][:60]:60s} {d["value"]:8.1f} fps {d["mrays_per_s"]:7.1f} Mrays/s  K1 {d["kernel_ms"]["march_K1"]:.3f} ms  K2 {d["kernel_ms"]["shade_K2"]:.3f} ms  frac {d["roofline"]["frac"]:.3f}  rays {c["mean_ray_stats"]}')
PY
