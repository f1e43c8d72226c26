#!/bin/bash
# Round-end evidence, call B: per-config SpMM times, c5 bench line, and one ncu --set full capture of
# a bench step's degree kernel + 4 SpMM launches (the only ncu run of this call).
tag=${1:-final_b}
out=gpurun_out/$tag
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen_cache
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
for c in c1 c2 c3 c4; do timeout 600 python scripts/run_spmm.py $c 4; done > $out/times.txt 2>&1; cat $out/times.txt
timeout 900 python scripts/run_spmm.py c5 4 > $out/spmm_c5.txt 2>&1; cat $out/spmm_c5.txt
timeout 1200 python bench.py --config c5 --steps 3 --warmup 3 > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 rc=$?"; cat $out/bench_c5.json
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spmm|k_degree" -s 10 -c 5 \
     -o $out/step_full $B > $out/ncu_full.log 2>&1; echo "ncu full rc=$?"
