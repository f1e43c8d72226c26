#!/bin/bash
# c5 bench (allocator trace), next-rows bench, smoke, default bench
out=gpurun_out/${1:-r02_gpu8}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
CLEORA_TRACE=1 timeout 1200 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-secondary > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 rc=$?"
grep -c "out of memory" $out/bench_c5.err
timeout 900 python scripts/bench_next.py > $out/bench_next.json 2> $out/bench_next.err; echo "next rc=$?"; tail -c 1500 $out/bench_next.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
python - <<'PY' $out
import json,sys
for f in ("bench_c5.json","bench.json"):
    try:
        d=json.loads(open(sys.argv[1]+"/"+f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f, d["config"]["workload"], "step ms", round(d["ms_per_step"],3), "spmm", round(d["roofline"]["kernel_ms"],3), "frac", round(d["roofline"]["frac"],3),
          "gbfrac", round(d["roofline"]["gather_bound"]["frac"],3), "e2e", d["e2e"] and (round(d["e2e"]["ms_per_step"],1), d["e2e"]["mode"][:40], d["e2e"].get("oom_fallbacks"), round(d["e2e"]["serial_ms_per_step"],1)))
PY
