#!/bin/bash
out=gpurun_out/${1:-r02_halves}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "half_row or c4_full or engines or hub or tiny or pairs" > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log
for h in 0 1; do CLEORA_HALVES=$h timeout 300 python scripts/run_spmm.py c4 4 >> $out/spmm.txt 2>&1; done
for h in 0 1; do CLEORA_HALVES=$h timeout 300 python scripts/run_spmm.py c2 4 >> $out/spmm.txt 2>&1; done
cat $out/spmm.txt
