#!/bin/bash
# One-kernel build of small graphs: tests, then the c1 step trace with and without it (alternating)
out=gpurun_out/${1:-r02_small_build}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_small_build.py -q -m gpu -x > $out/pytest_small.log 2>&1; echo "small pytest rc=$?"; tail -3 $out/pytest_small.log
for i in 1 2; do
  for sb in 0 1; do
    CLEORA_SMALL_BUILD=$sb timeout 300 python scripts/r02_c1_trace.py c1 | sed "s/^/{\"small_build\": $sb, \"r\": /; s/$/}/" >> $out/c1_trace.jsonl 2>> $out/err.txt
  done
done
cat $out/c1_trace.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_next.py tests/test_gpu_shard.py -q -m gpu -x > $out/pytest_rest.log 2>&1; echo "rest pytest rc=$?"; tail -3 $out/pytest_rest.log
