#!/bin/bash
# the driver's own commands: reference arm, then the bench at its defaults (N=1), then smoke and the GPU tests
out=gpurun_out/${1:-r02_driver}
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
s=$(date +%s); python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $out/ref.json 2> $out/ref.err; echo "ref rc=$? wall $(( $(date +%s) - s )) s"
s=$(date +%s); python bench.py --gpus 1 --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err; echo "bench rc=$? wall $(( $(date +%s) - s )) s"
python - <<'PY' $out
import json,sys
for f in ("ref.json","bench.json"):
    d=json.loads(open(sys.argv[1]+"/"+f).read().strip().splitlines()[-1])
    print(f, {k: d.get(k) for k in ("value","ms_per_step","gpu_launches","impl")}, d["config"]["workload"], d.get("clocks"))
PY
