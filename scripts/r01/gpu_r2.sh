#!/bin/bash
# dupmiss microbenchmark, hot-budget sweep (c2, c4, c5), GPU tests (incl. loopback), bench c2.
out=gpurun_out/${1:-r2}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen_cache
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dupmiss scripts/dupmiss.cu && timeout 120 /tmp/dupmiss > $out/dupmiss.jsonl 2>&1; cat $out/dupmiss.jsonl
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu.log
for c in c2 c4 c5; do for mb in 32 48 72 96; do CLEORA_HOT_MB=$mb timeout 600 python scripts/run_spmm.py $c 4 | sed "s/^/[hot $mb] /"; done; done > $out/hot_sweep.txt 2>&1; cat $out/hot_sweep.txt
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"; cat $out/bench.json
