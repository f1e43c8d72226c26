#!/bin/bash
# a lazy call's inner steps write only the gathered empty rows: tests, c4 A/B (CLEORA_INNER_ZERO=0/1)
out=gpurun_out/${1:-r02_innerzero}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_next.py tests/test_gpu_ipc.py tests/test_gpu_multi.py -q -m gpu -x > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log
for i in 1 2; do
  for z in 0 1; do CLEORA_INNER_ZERO=$z timeout 300 python scripts/run_spmm.py c4 4 | sed "s/^/[inner_zero$z] /" >> $out/ab.txt 2>&1; done
done
cat $out/ab.txt | sed 's/nnz [0-9]* heavy rows [0-9]* items [0-9]* hot rows [0-9]* //'
for z in 0 1 0 1; do CLEORA_INNER_ZERO=$z timeout 600 python bench.py --no-cpu --no-secondary --no-e2e --steps 10 --warmup 3 > $out/bench_z$z.json 2>> $out/bench.err; python -c "import json,sys; d=json.loads(open('$out/bench_z$z.json').read().strip().splitlines()[-1]); print('inner_zero$z', round(d['ms_per_step'],2), round(d['roofline']['kernel_ms'],3), d['value'])"; done
