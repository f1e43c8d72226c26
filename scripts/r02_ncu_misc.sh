#!/bin/bash
# ncu of the L2 gather probe at 64 B and 4 KB rows (32 MiB table), and of one c5 SpMM launch
out=gpurun_out/${1:-r02_ncu_misc}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for rb in 64 4096; do
  timeout 300 python scripts/r02_probe_one.py $rb 33554432 > $out/probe_$rb.txt 2>&1
  timeout 600 ncu --set full --clock-control none -k regex:k_probe_gather -s 3 -c 1 -o $out/ncu_probe_$rb \
      python scripts/r02_probe_one.py $rb 33554432 > $out/ncu_probe_$rb.log 2>&1; echo "probe $rb ncu rc=$?"
done
timeout 600 python scripts/run_spmm.py c5 2 > $out/c5_plain.log 2>&1; cat $out/c5_plain.log
timeout 1500 ncu --set full --clock-control none -k regex:k_spmm -s 1 -c 1 -o $out/ncu_spmm_c5 \
   python scripts/run_spmm.py c5 2 > $out/ncu_c5.log 2>&1; echo "c5 ncu rc=$?"
