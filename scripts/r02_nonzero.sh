#!/bin/bash
# compact fetch (cleora_fetch_nonzero): its GPU tests, then the driver's bench with the compact e2e,
# and the e2e with the sliced packing path (A/B)
out=gpurun_out/${1:-r02_nonzero}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
s=$(date +%s); timeout 1500 python -m pytest tests/test_gpu_fetch_nonzero.py -q -x -rs > $out/pytest.log 2>&1; echo "pytest rc=$? wall $(( $(date +%s) - s )) s"; tail -15 $out/pytest.log
s=$(date +%s); timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err; echo "bench rc=$? wall $(( $(date +%s) - s )) s"
tail -3 $out/bench.err
CLEORA_FETCH_SLICES=1 timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu --no-secondary > $out/bench_slices.json 2> $out/bench_slices.err; echo "bench slices rc=$?"
python - <<'PY' $out
import json,sys
for f in ("bench.json", "bench_slices.json"):
    d=json.loads(open(sys.argv[1]+"/"+f).read().strip().splitlines()[-1])
    print(f, {k: d.get(k) for k in ("value","ms_per_step","gpu_launches")}, d.get("clocks"))
    print(json.dumps(d["e2e"], indent=1))
PY
