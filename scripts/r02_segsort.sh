#!/bin/bash
out=gpurun_out/${1:-r02_segsort}
mkdir -p $out
for args in "5700000 1130000" "69000000 4850000" "700000000 10400000" "1400000000 20800000"; do
  timeout 600 ./scripts/segsort_bench $args >> $out/segsort.jsonl 2>&1
done
cat $out/segsort.jsonl
