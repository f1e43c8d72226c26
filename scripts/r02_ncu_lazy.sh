#!/bin/bash
# ncu --set full of step 2 of iterate(4) on c4 (passes 1 and 2), lazy on / off
out=gpurun_out/${1:-r02_ncu_lazy}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for lz in 1 0; do
  CLEORA_LAZY=$lz timeout 1200 ncu --set full --clock-control none -k regex:k_spmm_tma --launch-skip 2 --launch-count 2 -o $out/lazy$lz python scripts/run_spmm.py c4 4 > $out/ncu$lz.log 2>&1; echo "ncu lazy$lz rc=$?"
  ncu -i $out/lazy$lz.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_evict_last_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_evict_last_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read_evict_first_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read_evict_normal_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_evict_normal_lookup_miss.sum,smsp__cycles_active.avg,sm__warps_active.avg.pct_of_peak_sustained_active > $out/raw$lz.csv 2>&1
done
for lz in 1 0; do echo "== lazy$lz"; python - $out/raw$lz.csv <<'PY'
import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
h=rows[0]
for r in rows[2:]:
    print({h[i]: r[i] for i in range(len(h)) if h[i].startswith(("gpu__","dram","lts","smsp","sm__"))})
PY
done
