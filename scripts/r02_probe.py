"""L2->SM random-row gather rate by row size (cleora_probe_gather), L2-resident (64 MiB) and
HBM-resident (8 GiB) tables.  Prints one JSON object per line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_02302_b200 as cl  # noqa: E402

for table in (32 << 20, 64 << 20, 8 << 30):
    for rb in (64, 128, 256, 512, 1024, 2048, 4096):
        n = min((1 << 31) - 1, max(1 << 20, (16 << 30) // rb // 4))
        r = cl.cleora_probe_gather(rb, table, n, 0)
        print(json.dumps({"table_bytes": table, "row_bytes": rb, "gathers": n, "GBps": round(r, 1)}), flush=True)
