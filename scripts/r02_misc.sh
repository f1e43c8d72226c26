#!/bin/bash
out=gpurun_out/${1:-r02_misc}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
(free -g; nproc; lscpu | grep -E "Model name|Socket|Core|Thread") > $out/host.txt 2>&1
timeout 300 python scripts/r02_c1_trace.py c1 > $out/c1_trace.json 2>&1; cat $out/c1_trace.json
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-secondary > $out/bench_c4_short.json 2> $out/bench_c4_short.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $out/launches_c4.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-secondary > $out/ncu_launch.log 2>&1; echo "ncu rc=$?"
cat $out/host.txt
