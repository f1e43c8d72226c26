#!/bin/bash
# final build: the driver's bench line again (another box), then the c5 and c1 lines
out=gpurun_out/${1:-r02_final10}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
timeout 300 python bench.py --config c1 --steps 50 --warmup 10 --no-cpu --no-secondary > $out/bench_c1.json 2> $out/bench_c1.err; echo "bench c1 rc=$?"
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-secondary > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 rc=$?"
python - <<'PY' $out
import json,sys
for f in ("bench.json","bench_c1.json","bench_c5.json"):
    try:
        d=json.loads(open(sys.argv[1]+"/"+f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f, d["config"]["workload"], {k: d.get(k) for k in ("value","ms_per_step","gpu_launches")}, d.get("clocks"))
    r=d.get("roofline",{}); print("  frac", r.get("frac"), "kernel_ms", r.get("kernel_ms"), "gather", (r.get("gather_bound") or {}).get("frac"), "e2e", d.get("e2e",{}).get("ms_per_step"))
PY
