#!/bin/bash
# c4 half-row passes: heavy threshold x light-chunk rows; c5: heavy threshold x chunk rows
out=gpurun_out/${1:-r02_sweep}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
run() { echo -n "$1 $2 | "; env $2 timeout 300 python scripts/run_spmm.py $1 4 2>&1 | sed 's/.*hot rows/hot rows/'; }
{
for t in 128 256 512; do for c in 8 12 16 24; do run c4 "CLEORA_HEAVY_THRESH=$t CLEORA_CHUNK_ROWS=$c"; done; done
run c4 ""
for t in 256 512 1024; do for c in 16 31; do run c5 "CLEORA_HEAVY_THRESH=$t CLEORA_CHUNK_ROWS=$c"; done; done
} > $out/sweep.txt 2>&1
cat $out/sweep.txt
