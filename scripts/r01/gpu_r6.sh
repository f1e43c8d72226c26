#!/bin/bash
# Chunk-row caps: bitwise test, small-d engine checks, and one ncu --set full capture of the c3
# SpMM launch with the 6-row chunks (the recapture DESIGN §7 cites).
tag=${1:-r6}
out=gpurun_out/$tag
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "light_chunk_rows or engines" > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log
for h in 64 256; do
  CLEORA_GATHER=async CLEORA_HEAVY_THRESH=$h timeout 300 python scripts/run_spmm.py c4 4 128 | sed "s/^/[async heavy $h d 128] /"
  CLEORA_GATHER=async CLEORA_HEAVY_THRESH=$h timeout 300 python scripts/run_batch.py | sed "s/^/[async heavy $h] f4 /"
  CLEORA_GATHER=ldg CLEORA_HEAVY_THRESH=$h timeout 300 python scripts/run_spmm.py c4 4 128 | sed "s/^/[ldg heavy $h d 128] /"
done
for c in c1 c2 c3 c4; do timeout 600 python scripts/run_spmm.py $c 4 >> $out/spmm_times.txt 2>&1; done
cat $out/spmm_times.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 1 -c 1 \
     -o $out/spmm_c3 python scripts/run_spmm.py c3 3 > $out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
