#!/bin/bash
# A/B: paired short rows for rows <= 512 B (pair limit 16 default, 8, 32) vs one row per warp
python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "engines or light_chunk or parity" 2>&1 | tail -2
run() {
  timeout 300 python scripts/run_batch.py | sed "s/^/[$1] f4 /"
  for c in c2 c3 c4; do timeout 300 python scripts/run_spmm.py $c 4 128 | sed "s/^/[$1] /"; done
  timeout 300 python scripts/run_spmm.py c4 4 64 | sed "s/^/[$1] /"
}
run pair16
for f in 8 32 0; do
  CLEORA_NVCC_EXTRA=-DCLEORA_V1_PAIR=$f python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1; run pair$f
done
python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1
