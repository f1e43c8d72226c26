#!/bin/bash
# A/B with the compiled-in stride: neighbours per half-warp step (PAIR_PU) and per single-row batch (V1_U)
out=gpurun_out/${1:-r02_ab_pu}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
run() {
  timeout 300 python scripts/run_batch.py | sed "s/^/[$1] f4 /"
  for c in c2 c4; do timeout 300 python scripts/run_spmm.py $c 4 128 | sed "s/^/[$1] /"; done
  timeout 300 python scripts/run_spmm.py c4 4 64 | sed "s/^/[$1] /"
}
python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1; run base >> $out/ab.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "pairs or engines" > $out/pytest.log 2>&1; echo "pytest rc=$?"
for v in "-DCLEORA_PAIR_PU=2 pu2" "-DCLEORA_PAIR_PU=4 pu4" "-DCLEORA_V1_U=6 u6" "-DCLEORA_V1_U=8 u8"; do
  set -- $v
  CLEORA_NVCC_EXTRA=$1 python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1 || echo "build $2 failed"
  run $2 >> $out/ab.txt 2>&1
done
python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1
cat $out/ab.txt | sed 's/nnz [0-9]* heavy rows [0-9]* items [0-9]* hot rows [0-9]* //'
