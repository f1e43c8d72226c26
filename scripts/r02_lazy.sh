#!/bin/bash
# lazy normalisation between half-row steps (reading R21) + register-first degree folds:
# tests, c4 SpMM A/B (CLEORA_LAZY=0/1 alternating), c4 build time, bench lines lazy off/on
out=gpurun_out/${1:-r02_lazy}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "lazy or half_row or c4_full or composab" > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log
for i in 1 2; do
  for lz in 0 1; do CLEORA_LAZY=$lz timeout 300 python scripts/run_spmm.py c4 4 | sed "s/^/[lazy$lz] /" >> $out/ab.txt 2>&1; done
done
cat $out/ab.txt | sed 's/nnz [0-9]* heavy rows [0-9]* items [0-9]* hot rows [0-9]* //'
timeout 300 python scripts/r02_build_time.py c4 >> $out/build_time.jsonl 2>> $out/err.txt; cat $out/build_time.jsonl
for lz in 0 1 0 1; do CLEORA_LAZY=$lz timeout 600 python bench.py --no-cpu --no-secondary --no-e2e --steps 10 --warmup 3 > $out/bench_lazy$lz.json 2>> $out/bench.err; python -c "import json,sys; d=json.loads(open('$out/bench_lazy$lz.json').read().strip().splitlines()[-1]); print('lazy$lz', round(d['ms_per_step'],2), round(d['roofline']['kernel_ms'],3), d['value'])"; done
