#!/bin/bash
# c5 (full size, 1 GPU): generation, kernel timing, sampled parity test, bench line.
out=gpurun_out/${1:-c5}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen_cache
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
( time python -c "import gen; g=gen.config('c5'); print('c5 edges', g.n_edges, 'N', g.n)" ) > $out/gen.log 2>&1; cat $out/gen.log
timeout 900 python scripts/run_spmm.py c5 4 > $out/spmm_times.txt 2>&1; cat $out/spmm_times.txt
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> $out/spmm_times.txt
timeout 1800 python -m pytest tests/test_gpu_c5.py -x -q -s > $out/pytest_c5.log 2>&1; echo "pytest c5 rc=$?"; tail -5 $out/pytest_c5.log
timeout 1200 python bench.py --config c5 --steps 3 --warmup 3 > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench rc=$?"; cat $out/bench_c5.json; tail -3 $out/bench_c5.err
