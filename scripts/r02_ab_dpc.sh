#!/bin/bash
# A/B: the register kernel with the 512 B stride compiled in (dp = 128) vs the run-time stride
out=gpurun_out/${1:-r02_ab_dpc}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python paper_2102_02302_b200/_build.py --force > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -q -m gpu -x -k "engines or pairs or batch or tiny or c1" > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest.log
run() {
  for k in 1 2; do timeout 300 python scripts/run_batch.py | sed "s/^/[$1] f4 /"; done
  for c in c2 c3 c4; do timeout 300 python scripts/run_spmm.py $c 4 128 | sed "s/^/[$1] /"; done
  timeout 300 python scripts/run_spmm.py c1 8 | sed "s/^/[$1] /"
}
run dpc >> $out/ab.txt 2>&1
CLEORA_NVCC_EXTRA=-DCLEORA_V1_DPC=0 python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1 || echo "build failed"
run runtime >> $out/ab.txt 2>&1
python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1
run dpc2 >> $out/ab.txt 2>&1
cat $out/ab.txt | sed 's/nnz [0-9]* heavy rows [0-9]* items [0-9]* hot rows [0-9]* //'
