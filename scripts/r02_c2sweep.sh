#!/bin/bash
# c2 at d = 1024 (TMA bulk ring): heavy-row threshold x light-chunk rows; then the lazy-step test on the closing code
out=gpurun_out/${1:-r02_c2sweep}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for th in 32 64 128 256; do for cr in 4 6 8; do
  CLEORA_HEAVY_THRESH=$th CLEORA_CHUNK_ROWS=$cr timeout 300 python scripts/run_spmm.py c2 4 | sed "s/^/[th$th cr$cr] /" >> $out/sweep.txt 2>&1
done; done
for rep in 1; do for th in 64; do for cr in 6; do CLEORA_HEAVY_THRESH=$th CLEORA_CHUNK_ROWS=$cr timeout 300 python scripts/run_spmm.py c2 4 | sed "s/^/[default-again] /" >> $out/sweep.txt 2>&1; done; done; done
cat $out/sweep.txt | sed 's/nnz [0-9]* heavy rows \([0-9]*\) items \([0-9]*\) hot rows [0-9]* /heavy \1 items \2 /'
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "lazy" > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest.log
