#!/bin/bash
# closing run after the compact fetch and the never-gathered-row stores: driver commands, smoke, every GPU test, launch list
out=gpurun_out/${1:-r02_final8}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
s=$(date +%s); python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $out/ref.json 2> $out/ref.err; echo "ref rc=$? wall $(( $(date +%s) - s )) s"
s=$(date +%s); python bench.py --gpus 1 --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err; echo "bench rc=$? wall $(( $(date +%s) - s )) s"
python - <<'PY' $out
import json,sys
for f in ("ref.json","bench.json"):
    d=json.loads(open(sys.argv[1]+"/"+f).read().strip().splitlines()[-1])
    print(f, {k: d.get(k) for k in ("value","ms_per_step","gpu_launches","impl")}, d["config"]["workload"], d.get("clocks"))
    if "roofline" in d: print(" frac", round(d["roofline"]["frac"],3), "kernel_ms", d["roofline"]["kernel_ms"], "gather_bound frac", d["roofline"]["gather_bound"]["frac"], "e2e", d["e2e"]["value"], d["e2e"]["ms_per_step"], "dense", d["e2e"].get("dense_fetch",{}).get("ms_per_step"))
PY
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-secondary > $out/bench_c4_short.json 2> $out/bench_c4_short.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $out/launches_c4.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-secondary > $out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python scripts/launch_summary.py $out/launches_c4.csv 5 > $out/launches_c4_summary.txt 2>&1; head -8 $out/launches_c4_summary.txt
s=$(date +%s); CLEORA_PARITY_LOG=$out/parity.jsonl timeout 3600 python -m pytest tests -m gpu -q -rs > $out/pytest.log 2>&1; echo "pytest rc=$? wall $(( $(date +%s) - s )) s"; tail -5 $out/pytest.log
cat $out/parity.jsonl
