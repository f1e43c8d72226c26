#!/bin/bash
# A/B of register-kernel build switches: default vs -DCLEORA_DIV_SQRT (1.0/sqrt instead of rsqrt)
run() {
  for rep in 1 2; do
    timeout 300 python scripts/run_batch.py | sed "s/^/[$1] f4 /"
    for d in 128 256; do for c in c3 c4; do timeout 300 python scripts/run_spmm.py $c 4 $d | sed "s/^/[$1] /"; done; done
  done
}
python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1; run rsqrt
CLEORA_NVCC_EXTRA=-DCLEORA_DIV_SQRT python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1; run divsqrt
