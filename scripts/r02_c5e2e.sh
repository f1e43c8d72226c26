#!/bin/bash
# opt-in c5 end-to-end parity (whole-graph oracle on the box host) + the c5 bench line
out=gpurun_out/${1:-r02_c5e2e}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
CLEORA_C5_E2E=1 timeout 4800 python -m pytest tests/test_gpu_c5_e2e.py -m gpu -q -s > $out/pytest_c5_e2e.log 2>&1; echo "e2e rc=$?"
tail -5 $out/pytest_c5_e2e.log
CLEORA_TRACE=1 timeout 1200 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-secondary > $out/bench_c5.json 2> $out/bench_c5.err; echo "bench c5 rc=$?"
grep -c "out of memory" $out/bench_c5.err
