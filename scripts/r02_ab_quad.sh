#!/bin/bash
# A/B: four short rows per warp (quarter-warps) at dp <= 128 vs pairs only; correctness first
out=gpurun_out/${1:-r02_ab_quad}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python paper_2102_02302_b200/_build.py --force > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_multi.py -q -m gpu -x -k "engines or light_chunk or pairs or batch or tiny or degenerate or loopback" > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest.log
run() {
  for k in 1 2; do timeout 300 python scripts/run_batch.py | sed "s/^/[$1] f4 /"; done
  for c in c2 c3 c4; do timeout 300 python scripts/run_spmm.py $c 4 128 | sed "s/^/[$1] /"; done
  timeout 300 python scripts/run_spmm.py c4 4 64 | sed "s/^/[$1] /"
  timeout 300 python scripts/run_spmm.py c1 8 | sed "s/^/[$1] /"
}
run quad16pu2 >> $out/ab.txt 2>&1
for v in "-DCLEORA_QUAD_PU=1 quad16pu1" "-DCLEORA_V1_QUAD=8 quad8pu2" "-DCLEORA_V1_QUAD=0 pairs"; do
  set -- $v
  CLEORA_NVCC_EXTRA=$1 python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1 || echo "build $2 failed"
  run $2 >> $out/ab.txt 2>&1
done
python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1
cat $out/ab.txt
