#!/bin/bash
# One-kernel build beyond 2^21 entries (c3, f4 batch) vs the general build; ncu launch list of a c1 build
out=gpurun_out/${1:-r02_small_build2}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
for i in 1 2; do
  for c in c1 c3 f4; do
    CLEORA_SMALL_BUILD=0 timeout 300 python scripts/r02_build_time.py $c >> $out/build_time.jsonl 2>> $out/err.txt
    CLEORA_SMALL_MAX_ENTRIES=40000000 timeout 300 python scripts/r02_build_time.py $c >> $out/build_time.jsonl 2>> $out/err.txt
  done
done
cat $out/build_time.jsonl; tail -3 $out/err.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c1.csv python scripts/run_spmm.py c1 4 > $out/ncu.log 2>&1
python scripts/launch_summary.py $out/launches_c1.csv 1 > $out/launches_c1_summary.txt 2>&1; cat $out/launches_c1_summary.txt | head -30
