#!/bin/bash
# vectorised lazy weight pass: lazy tests, c4 launch times of k_lazy_vals, bench lines
out=gpurun_out/${1:-r02_lazyvals}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_ipc.py -q -m gpu -x -k "lazy or c4_full or deferred or processes or half_row" > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_lazy_vals" --csv --log-file $out/lazyvals.csv python scripts/run_spmm.py c4 4 > $out/ncu.log 2>&1; grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.,]*"' $out/lazyvals.csv | head
for i in 1 2; do timeout 600 python bench.py --no-cpu --no-secondary --no-e2e --steps 10 --warmup 3 > $out/bench$i.json 2>> $out/bench.err; python -c "import json,sys; d=json.loads(open('$out/bench$i.json').read().strip().splitlines()[-1]); print('bench', round(d['ms_per_step'],2), round(d['roofline']['kernel_ms'],3), d['value'])"; done
