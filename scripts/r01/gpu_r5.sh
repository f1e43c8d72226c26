#!/bin/bash
# parity (all GPU tests but c5), kernel times, bench c2, launch list, ncu of the steady-state SpMM launch
out=gpurun_out/${1:-r5}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen_cache
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
CLEORA_SKIP_C5=1 timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu.log
for c in c1 c2 c3 c4; do timeout 600 python scripts/run_spmm.py $c 4; done > $out/times.txt 2>&1; cat $out/times.txt
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"; cat $out/bench.json
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
timeout 300 $B > $out/bench_short.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
     --log-file $out/launches.csv $B > $out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spmm|k_degree" -s 10 -c 5 \
     -o $out/step_full $B > $out/ncu_full.log 2>&1; echo "ncu full rc=$?"
