#!/bin/bash
# ncu launch list of the f4 batched step (build_batch + init + 4 iterations), 2 steps
out=gpurun_out/${1:-r13}
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 300 python scripts/run_batch.py > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
     --log-file $out/launches_f4.csv python scripts/run_batch.py 4 > $out/ncu.log 2>&1; echo "ncu rc=$?"
