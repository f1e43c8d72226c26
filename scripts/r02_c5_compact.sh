#!/bin/bash
# the bench after the P > 1 compact-e2e change (c4, N = 1), then c5 with the compact e2e (its staging
# buffer may not fit beside the trimmed pipeline: the sliced fallback must run)
out=gpurun_out/${1:-r02_c5_compact}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
[ -n "$SKIP_C4" ] || { timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $out/bench_c4.json 2> $out/bench_c4.err; echo "bench c4 rc=$?"; }
CLEORA_TRACE=1 timeout 2400 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-secondary > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 rc=$?"
grep -c "out of memory" $out/bench_c5.err
tail -3 $out/bench_c5.err
python - <<'PY' $out
import json,sys
for f in ("bench_c4.json", "bench_c5.json"):
    try:
        d=json.loads(open(sys.argv[1]+"/"+f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "no line", e); continue
    print(f, {k: d.get(k) for k in ("value","ms_per_step","gpu_launches")}, d.get("clocks"))
    e=d.get("e2e") or {}
    print(" e2e", e.get("ms_per_step"), e.get("d2h_bytes_per_step"), e.get("mode"), "dense", (e.get("dense_fetch") or {}).get("ms_per_step"), "oom", e.get("oom_fallbacks"))
PY
