#!/bin/bash
out=gpurun_out/${1:-r02_gpu12}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
CLEORA_PARITY_LOG=$out/parity.jsonl CLEORA_SKIP_C5=1 timeout 2400 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest.log
for v in "" "CLEORA_NO_DEMOTE=1" "" "CLEORA_NO_DEMOTE=1"; do
  env $v timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $out/b.json 2>/dev/null
  python - <<PY $out/b.json "$v"
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(repr(sys.argv[2]), "step", round(d["ms_per_step"],2), "spmm", round(d["roofline"]["kernel_ms"],3), "value", "%.4g" % d["value"], "sm", d["clocks"]["sm_mhz"],
      "c2", round(d["secondary"]["c2"]["spmm_ms"],3), "c3", round(d["secondary"]["c3"]["spmm_ms"],3))
PY
done
