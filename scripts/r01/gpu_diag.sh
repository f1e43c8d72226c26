#!/bin/bash
# Diagnostics call: step jitter under each clock-sampling mode, L2 bandwidth microbenchmark,
# per-config kernel times, and ncu full captures of the SpMM on c3 and c4.
tag=${1:-diag}
out=gpurun_out/$tag
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
nproc > $out/host.txt; free -g >> $out/host.txt; lscpu | head -20 >> $out/host.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2bw scripts/l2bw.cu && timeout 120 /tmp/l2bw > $out/l2bw.jsonl 2>&1
cat $out/l2bw.jsonl
for m in none nvml smi none; do timeout 300 python scripts/step_jitter.py $m 30 c2 >> $out/jitter.jsonl 2>&1; done
cat $out/jitter.jsonl
for c in c1 c3 c4; do timeout 600 python scripts/run_spmm.py $c 4 >> $out/spmm_times.txt 2>&1; done
cat $out/spmm_times.txt
timeout 600 python scripts/run_spmm.py c3 3 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 1 -c 1 \
     -o $out/spmm_c3 python scripts/run_spmm.py c3 3 > $out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 1 -c 1 \
     -o $out/spmm_c4 python scripts/run_spmm.py c4 3 > $out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
ls -la $out
