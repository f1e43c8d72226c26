#!/bin/bash
out=gpurun_out/${1:-r02_trace_c4}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for i in 1 2; do CLEORA_TRACE=1 timeout 300 python scripts/run_spmm.py c4 4 >> $out/trace_c4.txt 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $out/launches_c4.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-secondary > $out/ncu_launch.log 2>&1; echo "ncu rc=$?"
python scripts/launch_summary.py $out/launches_c4.csv 4 | head -30
tail -30 $out/trace_c4.txt
