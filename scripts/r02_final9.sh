#!/bin/bash
# HEAD's c4 SpMM under ncu after the never-gathered-row stores were dropped: DRAM bytes of every launch of
# one iterate(4), then ncu --set full of step 2's launches (pass 1 + pass 2, lazy), with source
out=gpurun_out/${1:-r02_final9}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 300 python scripts/run_spmm.py c4 4 > $out/run.log 2>&1 || { echo RUN FAILED; tail $out/run.log; exit 1; }
cat $out/run.log
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base -k regex:"k_spmm_tma|k_lazy_vals" --csv --log-file $out/c4_iterate_dram.csv python scripts/run_spmm.py c4 4 > $out/ncu_dram.log 2>&1; echo "ncu dram rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tma --launch-skip 2 --launch-count 2 -o $out/c4_step2 python scripts/run_spmm.py c4 4 > $out/ncu.log 2>&1; echo "ncu full rc=$?"
ncu -i $out/c4_step2.ncu-rep --page details --csv > $out/details.csv 2>&1
ncu -i $out/c4_step2.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed > $out/raw.csv 2>&1
cat $out/raw.csv | tail -4
python - <<'PY' $out
import csv, sys
rows = [r for r in csv.reader(l for l in open(sys.argv[1] + "/c4_iterate_dram.csv") if l.startswith('"'))]
h = rows[0]; ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
ii = h.index("ID")
per = {}
for r in rows[1:]:
    per.setdefault((int(r[ii]), r[ki][:40]), {})[r[mi]] = float(r[vi].replace(",", ""))
tot = 0
for (i, k), m in sorted(per.items()):
    b = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    tot += b
    print(i, k, "ms", m.get("gpu__time_duration.sum", 0) / 1e6, "dram bytes", b, m)
print("total", tot, "per iteration", tot / 4)
PY
rm -f $out/c4_step2.ncu-rep.tmp
ls -la $out
