#!/bin/bash
# A/B of the half-row passes on c4 (min / mean ms per SpMM step = both passes)
out=gpurun_out/${1:-r02_halves_ab}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
run() { echo -n "$1 | "; env $2 timeout 300 python scripts/run_spmm.py c4 4 2>&1 | sed 's/.*hot rows/hot rows/'; }
{
run "whole bulk" "CLEORA_HALVES=0"
run "halves bulk t64 c6" "CLEORA_HALVES=1"
run "halves async t64 c6" "CLEORA_HALVES=1 CLEORA_GATHER=async CLEORA_HEAVY_THRESH=64 CLEORA_CHUNK_ROWS=6"
run "halves bulk t256 c6" "CLEORA_HALVES=1 CLEORA_HEAVY_THRESH=256"
run "halves bulk t64 c12" "CLEORA_HALVES=1 CLEORA_CHUNK_ROWS=12"
run "halves async t256 c12" "CLEORA_HALVES=1 CLEORA_GATHER=async CLEORA_HEAVY_THRESH=256 CLEORA_CHUNK_ROWS=12"
run "halves bulk hot96" "CLEORA_HALVES=1 CLEORA_HOT_MB=96"
run "halves bulk hot48" "CLEORA_HALVES=1 CLEORA_HOT_MB=48"
run "whole bulk again" "CLEORA_HALVES=0"
} > $out/ab.txt 2>&1
cat $out/ab.txt
