#!/bin/bash
# Per-iteration SpMM+normalise kernel time on every single-GPU config (TMA path and register path).
for c in c1 c2 c3 c4; do python scripts/run_spmm.py $c 4; done
for c in c2 c3; do CLEORA_NO_TMA=1 python scripts/run_spmm.py $c 4 | sed 's/^/[no-tma] /'; done
