#!/bin/bash
# Round-end evidence, call A: full GPU suite, smoke, bench (c2) + reference arm + 8(f) rows, and the
# ncu launch list of the bench command (the only ncu run of this call).
tag=${1:-final_a}
out=gpurun_out/$tag
mkdir -p $out
bash scripts/gpu_full.sh $tag
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
timeout 300 $B > $out/bench_short.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
     --log-file $out/launches.csv $B > $out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
