#!/bin/bash
out=gpurun_out/${1:-r02_small_build4}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_small_build.py -q -m gpu -x > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest.log
for i in 1 2; do timeout 300 python scripts/r02_c1_trace.py c1 >> $out/c1_trace.jsonl 2>> $out/err.txt; done
cat $out/c1_trace.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c1.csv python scripts/run_spmm.py c1 4 > $out/ncu.log 2>&1
python scripts/launch_summary.py $out/launches_c1.csv 1 > $out/launches_c1_summary.txt 2>&1; cat $out/launches_c1_summary.txt | head -30
