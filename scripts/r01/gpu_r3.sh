#!/bin/bash
# LDGSTS-for-hot-rows experiment: parity, timings c2/c3/c4 both ways, ncu captures of c2 both ways,
# launch list of the bench step.
out=gpurun_out/${1:-r3}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen_cache
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
CLEORA_HOT_LDGSTS=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tiny or hub or c2 or tma or threshold" > $out/pytest_ldgsts.log 2>&1; echo "pytest ldgsts rc=$?"; tail -2 $out/pytest_ldgsts.log
for c in c2 c3 c4; do for v in 0 1; do CLEORA_HOT_LDGSTS=$v timeout 600 python scripts/run_spmm.py $c 4 | sed "s/^/[ldgsts $v] /"; done; done > $out/times.txt 2>&1; cat $out/times.txt
for v in 0 1; do
  CLEORA_HOT_LDGSTS=$v timeout 300 python scripts/run_spmm.py c2 3 > /dev/null 2>&1 && \
  CLEORA_HOT_LDGSTS=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 1 -c 1 \
     -o $out/spmm_c2_ldgsts$v python scripts/run_spmm.py c2 3 > $out/ncu_c2_$v.log 2>&1; echo "ncu c2 $v rc=$?"
done
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
timeout 300 $B > $out/bench_short.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
     --log-file $out/launches.csv $B > $out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
