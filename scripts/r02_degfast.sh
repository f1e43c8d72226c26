#!/bin/bash
# exact-order-independent degree sums: CSR tests (bit-exact degrees), c4 build time and launch list
out=gpurun_out/${1:-r02_degfast}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_small_build.py tests/test_gpu_shard.py tests/test_gpu_batch.py tests/test_gpu_next.py -q -m gpu -x > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log
for i in 1 2; do timeout 600 python scripts/r02_build_time.py c4 >> $out/build_time.jsonl 2>> $out/err.txt; done; cat $out/build_time.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c4_build.csv python scripts/run_spmm.py c4 1 > $out/ncu.log 2>&1
python scripts/launch_summary.py $out/launches_c4_build.csv 1 > $out/launches_summary.txt 2>&1; grep -i "degree\|all" $out/launches_summary.txt
