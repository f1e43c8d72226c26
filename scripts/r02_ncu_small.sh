#!/bin/bash
# ncu --set full of the one-kernel build and one c1 SpMM launch; c1 trace with the one-row chunk schedule
out=gpurun_out/${1:-r02_ncu_small}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for i in 1 2; do timeout 300 python scripts/r02_c1_trace.py c1 >> $out/c1_trace.jsonl 2>> $out/err.txt; done
cat $out/c1_trace.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_build_small|k_spmm_norm" -c 3 -o $out/small python scripts/run_spmm.py c1 2 > $out/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $out/small.ncu-rep --page details --csv > $out/small_details.csv 2>&1
timeout 900 python -m pytest tests/test_gpu_small_build.py tests/test_gpu_parity.py tests/test_gpu_batch.py -q -m gpu -x > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log
