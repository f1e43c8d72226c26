#!/bin/bash
# static chunk round robin for small graphs + the wider one-kernel build grid: c1 trace, launch list, tests
out=gpurun_out/${1:-r02_small_build3}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
for i in 1 2; do timeout 300 python scripts/r02_c1_trace.py c1 >> $out/c1_trace.jsonl 2>> $out/err.txt; done
cat $out/c1_trace.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c1.csv python scripts/run_spmm.py c1 4 > $out/ncu.log 2>&1
python scripts/launch_summary.py $out/launches_c1.csv 1 > $out/launches_c1_summary.txt 2>&1; cat $out/launches_c1_summary.txt | head -30
timeout 1500 python -m pytest tests/test_gpu_small_build.py tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_next.py tests/test_gpu_shard.py tests/test_gpu_multi.py tests/test_gpu_ipc.py -q -m gpu -x > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log
