#!/bin/bash
# L2 hot-row budget / cold-policy sweep (TMA path): per-iteration kernel time per config.
for c in c2 c4 c3; do
  CLEORA_NO_HOT=1 python scripts/run_spmm.py $c 4 | sed "s/^/[nohot] /"
  for mb in 48 72 96; do CLEORA_HOT_MB=$mb python scripts/run_spmm.py $c 4 | sed "s/^/[hot $mb] /"; done
  CLEORA_COLD_FIRST=1 python scripts/run_spmm.py $c 4 | sed "s/^/[hot 72 coldfirst] /"
done
