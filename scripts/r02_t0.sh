#!/bin/bash
# T_0 written only for gathered rows (completed on reads): tests, c4 bench A/B (CLEORA_T0_ALL=1/0)
out=gpurun_out/${1:-r02_t0}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
timeout 3000 python -m pytest tests -m gpu -q -x -k "not c5" > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log
for a in 1 0 1 0; do CLEORA_T0_ALL=$a timeout 600 python bench.py --no-cpu --no-secondary --no-e2e --steps 10 --warmup 3 > $out/bench_all$a.json 2>> $out/bench.err; python -c "import json,sys; d=json.loads(open('$out/bench_all$a.json').read().strip().splitlines()[-1]); print('t0_all$a', round(d['ms_per_step'],2), round(d['roofline']['kernel_ms'],3), d['value'])"; done
