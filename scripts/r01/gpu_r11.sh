#!/bin/bash
# e2e pipeline host timeline + D2H bandwidth alone and beside a running step; ncu of the f4 SpMM
out=gpurun_out/${1:-r11}
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
timeout 300 python scripts/e2e_trace.py 6 > $out/e2e_trace.txt 2>&1; cat $out/e2e_trace.txt
timeout 300 python scripts/d2h_bw.py > $out/d2h.json 2>&1; cat $out/d2h.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 1 -c 1 \
     -o $out/spmm_f4 python scripts/run_batch.py 3 > $out/ncu_f4.log 2>&1; echo "ncu f4 rc=$?"
