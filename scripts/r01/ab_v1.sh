#!/bin/bash
# A/B of the register kernel for rows <= 512 B (V = 1): neighbours per batch and CTAs per SM
run() {
  timeout 300 python scripts/run_batch.py | sed "s/^/[$1] f4 /"
  timeout 300 python scripts/run_spmm.py c1 4 | sed "s/^/[$1] /"
  for c in c2 c3 c4; do timeout 300 python scripts/run_spmm.py $c 4 128 | sed "s/^/[$1] /"; done
  timeout 300 python scripts/run_spmm.py c4 4 64 | sed "s/^/[$1] /"
}
for f in "" "-DCLEORA_V1_U=4" "-DCLEORA_V1_U=6" "-DCLEORA_V1_BLOCKS=3" "-DCLEORA_V1_BLOCKS=3 -DCLEORA_V1_U=4"; do
  CLEORA_NVCC_EXTRA="$f" python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1 || echo "build failed $f"
  run "${f:-default}"
done
python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_multi.py -q -m gpu -x 2>&1 | tail -2
