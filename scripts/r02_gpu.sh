#!/bin/bash
# GPU tests (optionally a subset), smoke, default bench line.  Usage: r02_gpu.sh <tag> [pytest -k expr]
out=gpurun_out/${1:-r02_gpu}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
if [ -n "$2" ]; then K="-k $2"; else K=""; fi
CLEORA_PARITY_LOG=$out/parity.jsonl CLEORA_SKIP_C5=${SKIP_C5:-1} timeout 2400 python -m pytest tests -m gpu -x -q $K > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
python - <<'PY' $out/bench.json
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print({k: d[k] for k in ("value","ms_per_step","gpu_launches")}, d["config"]["workload"], "frac", round(d["roofline"]["frac"],3),
      "spmm", round(d["roofline"]["kernel_ms"],2), "gather_bound", d["roofline"]["gather_bound"], "e2e", d["e2e"] and round(d["e2e"]["ms_per_step"],1))
print("secondary", {k: (round(v["spmm_ms"],3), round(v["frac"],3)) for k,v in (d["secondary"] or {}).items()})
PY
