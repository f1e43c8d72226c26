#!/bin/bash
# ncu --set full (with source) of the f4 batch SpMM launch (register kernel, d = 128, ~8 entries per row)
tag=${1:-r7}
out=gpurun_out/$tag
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
timeout 300 python scripts/run_batch.py > $out/batch.txt 2>&1; cat $out/batch.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 1 -c 1 \
     -o $out/spmm_f4 python scripts/run_batch.py 3 > $out/ncu_f4.log 2>&1; echo "ncu f4 rc=$?"
