#!/bin/bash
# discard.global.L2 of pass 1's pinned first halves of T_in before pass 2 (one GPU): tests, c4 A/B
out=gpurun_out/${1:-r02_discard}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "lazy or half_row or c4_full or composab or partial_t0" > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest.log
CLEORA_HOT_MB=0.5 timeout 1800 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "lazy or half_row" > $out/pytest_hot.log 2>&1; echo "pytest (hot tags on small graphs) rc=$?"; tail -2 $out/pytest_hot.log
for rep in 1 2; do for dc in 0 1; do
  CLEORA_DISCARD=$dc timeout 300 python scripts/run_spmm.py c4 4 | sed "s/^/[discard$dc] /" >> $out/ab.txt 2>&1
  CLEORA_DISCARD=$dc timeout 600 python bench.py --no-cpu --no-secondary --no-e2e --steps 10 --warmup 3 > $out/bench_d$dc.json 2>> $out/bench.err; python -c "import json,sys; d=json.loads(open('$out/bench_d$dc.json').read().strip().splitlines()[-1]); print('discard$dc', round(d['ms_per_step'],2), round(d['roofline']['kernel_ms'],3), d['value'])" >> $out/ab.txt
done; done
cat $out/ab.txt | sed 's/nnz [0-9]* heavy rows [0-9]* items [0-9]* hot rows [0-9]* //'
timeout 1500 ncu --clock-control none -k regex:k_spmm_tma --launch-skip 2 --launch-count 2 --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read_evict_last_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_evict_last_lookup_miss.sum --csv python scripts/run_spmm.py c4 4 > $out/ncu.csv 2> $out/ncu.err; grep -E "gpu__time|dram__bytes|evict_last" $out/ncu.csv | awk -F'","' '{print $1, $13, $15}' | tail -8
