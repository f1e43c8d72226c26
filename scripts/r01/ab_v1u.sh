#!/bin/bash
# A/B of the single-row batch width at d <= 128 now that short rows are paired
run() {
  timeout 300 python scripts/run_batch.py | sed "s/^/[$1] f4 /"
  for c in c2 c3 c4; do timeout 300 python scripts/run_spmm.py $c 4 128 | sed "s/^/[$1] /"; done
  timeout 300 python scripts/run_spmm.py c4 4 64 | sed "s/^/[$1] /"
}
for f in 4 6 8; do
  CLEORA_NVCC_EXTRA=-DCLEORA_V1_U=$f python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1 || echo "build failed $f"
  run u$f
done
python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1
