"""Summarise an ncu --set full report: the metrics DESIGN.md / bench.py cite.
Usage: python scripts/ncu_summary.py report.ncu-rep [label]"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "lts__t_sectors_srcunit_tex_op_read.sum": "l2_read_sectors_from_sm",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct_peak",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_peak",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed_pipe_lsu.sum": "lsu_inst",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
}


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k, name in WANT.items():
            if k in hdr:
                i = hdr.index(k)
                d[name] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
