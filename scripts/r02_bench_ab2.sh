#!/bin/bash
# same-box A/B of the bench line: T_0's hash on a side stream off / on, alternating; then GPU tests
out=gpurun_out/${1:-r02_bench_ab2}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for h in 0 1 0 1; do
  CLEORA_INIT_SIDE=$h timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-secondary > $out/bench_s$h.json 2>/dev/null
  python - <<PY $out/bench_s$h.json $h
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("init_side", sys.argv[2], "step", round(d["ms_per_step"],2), "spmm", round(d["roofline"]["kernel_ms"],3), "value", "%.4g" % d["value"], "sm", d["clocks"]["sm_mhz"])
PY
done
CLEORA_SKIP_C5=1 timeout 2400 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest.log
