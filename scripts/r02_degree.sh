#!/bin/bash
# long rows' degree folds one warp per row: c4 build time, launch list of one c4 build, CSR parity (c4 full, hubs)
out=gpurun_out/${1:-r02_degree}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for i in 1 2; do timeout 600 python scripts/r02_build_time.py c4 >> $out/build_time.jsonl 2>> $out/err.txt; done
cat $out/build_time.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c4_build.csv python scripts/run_spmm.py c4 1 > $out/ncu.log 2>&1
python scripts/launch_summary.py $out/launches_c4_build.csv 1 > $out/launches_summary.txt 2>&1; head -20 $out/launches_summary.txt
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c4_full or hub or tiny or c2_full or c3_full" > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest.log
