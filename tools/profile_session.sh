#!/bin/bash
# One GPU session's measurement artefacts for tools/profile_report.py <tag>:
# bench line, reference arm, config sweep, ncu launch list and one ncu --set full
# capture of K0/K1/K2 (taken from warm-up frames, after each plain run exited 0).
tag=${1:?tag}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err || exit 1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/reference_$tag.json 2>&1
STEPS=8 bash tools/bench_configs.sh $tag > gpurun_out/configs_$tag.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches_$tag.log 2>&1
# bench's first renders are the untimed counter renders (4 cameras x 3 kernels); skip them
ncu --set full --import-source on --clock-control none -k 'regex:raygen|march_kernel|shade_tc' -s 15 -c 3 \
    -o gpurun_out/prof_$tag python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_$tag.log 2>&1
echo session_done
