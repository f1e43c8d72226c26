#!/bin/bash
# ncu --set full of the f4 batch SpMM (paired short rows)
out=gpurun_out/${1:-r12}
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 1 -c 1 \
     -o $out/spmm_f4 python scripts/run_batch.py 3 > $out/ncu_f4.log 2>&1; echo "ncu f4 rc=$?"
