#!/bin/bash
# full validation: every GPU test (c5 included), smoke, the driver's two bench commands
out=gpurun_out/${1:-r02_final}
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
s=$(date +%s); CLEORA_PARITY_LOG=$out/parity.jsonl timeout 3000 python -m pytest tests -m gpu -q -rs > $out/pytest.log 2>&1; echo "pytest rc=$? wall $(( $(date +%s) - s )) s"; tail -3 $out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"
s=$(date +%s); python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $out/ref.json 2> $out/ref.err; echo "ref rc=$? wall $(( $(date +%s) - s )) s"
s=$(date +%s); python bench.py --gpus 1 --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err; echo "bench rc=$? wall $(( $(date +%s) - s )) s"
python - <<'PY' $out
import json,sys
for f in ("ref.json","bench.json"):
    d=json.loads(open(sys.argv[1]+"/"+f).read().strip().splitlines()[-1])
    print(f, {k: d.get(k) for k in ("value","ms_per_step","gpu_launches","impl")}, d["config"]["workload"], d.get("clocks"))
    if "roofline" in d: print(" frac", round(d["roofline"]["frac"],3), "gather_bound", d["roofline"].get("gather_bound"), "e2e", d["e2e"])
PY
