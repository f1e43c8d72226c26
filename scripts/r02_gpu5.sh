#!/bin/bash
# GPU tests + c5 bench with allocator trace + default bench
out=gpurun_out/${1:-r02_gpu5}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
CLEORA_PARITY_LOG=$out/parity.jsonl CLEORA_SKIP_C5=${SKIP_C5:-1} timeout 2400 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log
cat $out/parity.jsonl
CLEORA_TRACE=1 timeout 1200 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-secondary > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 rc=$?"
grep -c "out of memory" $out/bench_c5.err
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
