#!/bin/bash
# Round-2 baseline on the current build: c4 bench line, c4 SpMM times vs hot budget, ncu --set full of one c4 SpMM launch
out=gpurun_out/${1:-r02_base}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu > $out/bench_c4.json 2> $out/bench_c4.err; echo "bench rc=$?"
for mb in 0 36 72 96; do
  if [ $mb = 0 ]; then CLEORA_NO_HOT=1 timeout 300 python scripts/run_spmm.py c4 4 >> $out/hot_c4.txt 2>&1;
  else CLEORA_HOT_MB=$mb timeout 300 python scripts/run_spmm.py c4 4 >> $out/hot_c4.txt 2>&1; fi
done
CLEORA_GATHER=async timeout 300 python scripts/run_spmm.py c4 4 >> $out/hot_c4.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 1 -c 1 \
   -o $out/ncu_spmm_c4 python scripts/run_spmm.py c4 2 > $out/ncu.log 2>&1; echo "ncu rc=$?"
