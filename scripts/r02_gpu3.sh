#!/bin/bash
# GPU tests + c1 / c4 bench lines after the sync-free schedule
out=gpurun_out/${1:-r02_gpu3}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
CLEORA_SKIP_C5=1 timeout 2400 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log
timeout 300 python bench.py --config c1 --steps 50 --no-e2e --no-cpu --no-secondary > $out/bench_c1.json 2> $out/bench_c1.err; echo "c1 rc=$?"
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
python - <<'PY' $out
import json,sys
for f in ("bench_c1.json","bench.json"):
    d=json.loads(open(sys.argv[1]+"/"+f).read().strip().splitlines()[-1])
    print(f, d["config"]["workload"], "step ms", round(d["ms_per_step"],4), "spmm", round(d["roofline"]["kernel_ms"],4), "frac", round(d["roofline"]["frac"],3),
          "gb", {k: (round(v,3) if isinstance(v,float) else v) for k,v in d["roofline"]["gather_bound"].items() if k!="how"}, "launches", d["gpu_launches"])
PY
