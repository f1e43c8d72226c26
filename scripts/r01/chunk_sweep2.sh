#!/bin/bash
# light-chunk rows per engine and row size (engine as chosen by gather_mode: d=256/512 cp.async, d<=128 LDG)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 31 24 16 12 8; do
  for d in 256 512; do for c in c3 c4; do CLEORA_CHUNK_ROWS=$r timeout 300 python scripts/run_spmm.py $c 4 $d | sed "s/^/[rows $r] /"; done; done
  for c in c2 c3 c4; do CLEORA_CHUNK_ROWS=$r timeout 300 python scripts/run_spmm.py $c 4 128 | sed "s/^/[rows $r] /"; done
  CLEORA_CHUNK_ROWS=$r timeout 300 python scripts/run_batch.py | sed "s/^/[rows $r] f4 /"
done
