"""One cleora_probe_gather run (for ncu): python scripts/r02_probe_one.py row_bytes table_bytes"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_02302_b200 as cl  # noqa: E402

rb, tb = int(sys.argv[1]), int(sys.argv[2])
print(rb, tb, cl.cleora_probe_gather(rb, tb, min((1 << 31) - 1, (4 << 30) // rb), 0))
