#!/bin/bash
# c5 bench e2e with the stream-ordered pool for every allocation (CLEORA_NO_CACHE=1) vs the block cache
out=gpurun_out/${1:-r02_c5pool}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
CLEORA_NO_CACHE=1 CLEORA_TRACE=1 timeout 1500 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-secondary > $out/pool.json 2> $out/pool.err; echo "pool rc=$?"
CLEORA_TRACE=1 timeout 1500 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-secondary > $out/cache.json 2> $out/cache.err; echo "cache rc=$?"
for f in pool cache; do
python - <<PY $out/$f.json $f
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    e=d["e2e"]
    print(sys.argv[2], "step", round(d["ms_per_step"],1), "spmm", round(d["roofline"]["kernel_ms"],1), "e2e", round(e["ms_per_step"],1), e["mode"][:30], "serial", round(e["serial_ms_per_step"],1), "oom", e.get("oom_fallbacks"))
except Exception as x: print(sys.argv[2], "failed", x)
PY
grep -c "out of memory" $out/$f.err
done
