#!/bin/bash
# ncu --set full of the closing build's c4 SpMM: step 2 of iterate(4) (pass 1 + pass 2, lazy), with source
out=gpurun_out/${1:-r02_ncu_final}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tma --launch-skip 2 --launch-count 2 -o $out/c4_step2 python scripts/run_spmm.py c4 4 > $out/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $out/c4_step2.ncu-rep --page details --csv > $out/details.csv 2>&1
ncu -i $out/c4_step2.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_evict_last_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_evict_last_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read_evict_first_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_evict_first_lookup_miss.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed > $out/raw.csv 2>&1
ls -la $out
