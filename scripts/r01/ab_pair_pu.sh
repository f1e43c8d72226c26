#!/bin/bash
# A/B of the paired-row step width (neighbours per half-warp per step)
run() {
  timeout 300 python scripts/run_batch.py | sed "s/^/[$1] f4 /"
  for c in c2 c3 c4; do timeout 300 python scripts/run_spmm.py $c 4 128 | sed "s/^/[$1] /"; done
}
for f in 2 3 4 1; do
  CLEORA_NVCC_EXTRA=-DCLEORA_PAIR_PU=$f python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1 || echo "build failed $f"
  run pu$f
done
python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1
