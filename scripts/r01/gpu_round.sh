#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench (c2 default), then the ncu launch list and one
# `--set full` capture of the dominant kernel of the same bench command.  Logs in gpurun_out/.
# Usage (from this container):  gpurun --timeout 3000 -- 'bash scripts/gpu_round.sh [tag]'
tag=${1:-r01}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $out/pytest_gpu.log
tail -3 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"; cat $out/bench.json
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
timeout 300 $B > $out/bench_short.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
     --log-file $out/launches.csv $B > $out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 4 -c 1 \
     -o $out/spmm_full $B > $out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ls -la $out
