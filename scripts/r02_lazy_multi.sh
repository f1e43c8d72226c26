#!/bin/bash
# lazy steps in loopback / peer modes (scales behind the T rows): tests, then the c4 lazy A/B again
out=gpurun_out/${1:-r02_lazy_multi}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
timeout 2400 python -m pytest tests/test_gpu_shard.py tests/test_gpu_ipc.py tests/test_gpu_multi.py tests/test_gpu_parity.py tests/test_gpu_batch.py -q -m gpu -x > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log
for i in 1 2; do
  for lz in 0 1; do CLEORA_LAZY=$lz timeout 300 python scripts/run_spmm.py c4 4 | sed "s/^/[lazy$lz] /" >> $out/ab.txt 2>&1; done
done
cat $out/ab.txt | sed 's/nnz [0-9]* heavy rows [0-9]* items [0-9]* hot rows [0-9]* //'
for lz in 0 1 0 1; do CLEORA_LAZY=$lz timeout 600 python bench.py --no-cpu --no-secondary --no-e2e --steps 10 --warmup 3 > $out/bench_lazy$lz.json 2>> $out/bench.err; python -c "import json,sys; d=json.loads(open('$out/bench_lazy$lz.json').read().strip().splitlines()[-1]); print('lazy$lz', round(d['ms_per_step'],2), round(d['roofline']['kernel_ms'],3), d['value'])"; done
