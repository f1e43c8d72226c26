#!/bin/bash
# same-box A/B of the bench line: half-row passes off / on (twice each, alternating)
out=gpurun_out/${1:-r02_bench_ab}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for h in 0 1 0 1; do
  CLEORA_HALVES=$h timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-secondary > $out/bench_h$h.json 2>/dev/null
  python - <<PY $out/bench_h$h.json $h
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("halves", sys.argv[2], "step", round(d["ms_per_step"],2), "spmm", round(d["roofline"]["kernel_ms"],3), "value", "%.4g" % d["value"], "sm", d["clocks"]["sm_mhz"])
PY
done
