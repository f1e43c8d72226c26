#!/bin/bash
# output rows stored with an explicit L2 evict_first policy (-DCLEORA_STORE_EF=1) vs streaming stores: c4 SpMM + bench, alternating builds
out=gpurun_out/${1:-r02_store_ef}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
for rep in 1 2; do
  for ef in 0 1; do
    CLEORA_NVCC_EXTRA="-DCLEORA_STORE_EF=$ef" python paper_2102_02302_b200/_build.py --force > $out/build$ef.log 2>&1 || { echo BUILD FAILED; exit 1; }
    timeout 300 python scripts/run_spmm.py c4 4 | sed "s/^/[ef$ef] /" >> $out/ab.txt 2>&1
    timeout 600 python bench.py --no-cpu --no-secondary --no-e2e --steps 10 --warmup 3 > $out/bench_ef$ef.json 2>> $out/bench.err; python -c "import json,sys; d=json.loads(open('$out/bench_ef$ef.json').read().strip().splitlines()[-1]); print('ef$ef', round(d['ms_per_step'],2), round(d['roofline']['kernel_ms'],3), d['value'])" >> $out/ab.txt
  done
done
cat $out/ab.txt | sed 's/nnz [0-9]* heavy rows [0-9]* items [0-9]* hot rows [0-9]* //'
CLEORA_NVCC_EXTRA="-DCLEORA_STORE_EF=1" python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1
timeout 1500 ncu --clock-control none -k regex:k_spmm_tma --launch-skip 2 --launch-count 2 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_evict_last_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_evict_last_lookup_miss.sum --csv python scripts/run_spmm.py c4 4 > $out/ncu_ef1.csv 2> $out/ncu.err; grep -E "gpu__time|dram__bytes|evict_last" $out/ncu_ef1.csv | cut -c1-250 | tail -10
