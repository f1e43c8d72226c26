#!/bin/bash
# ncu --set full of one c4 step's two half-row passes (launches 3 and 4 of k_spmm_tma<4,1,6>), and the
# bench launch list on the current build
out=gpurun_out/${1:-r02_ncu_halves}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 300 python scripts/run_spmm.py c4 2 > $out/plain.log 2>&1; cat $out/plain.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tma -s 2 -c 2 \
   -o $out/ncu_halves_c4 python scripts/run_spmm.py c4 2 > $out/ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $out/launches_c4.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-secondary > $out/ncu_launch.log 2>&1; echo "launch list rc=$?"
