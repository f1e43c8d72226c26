#!/bin/bash
# light-chunk row count vs SpMM time (c2, c3, c4 at d=1024; c3/c4 at d=256 (LDG) and 512 (cp.async))
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 31 8 6 5 4 3; do
  for c in c3 c2; do CLEORA_CHUNK_ROWS=$r timeout 300 python scripts/run_spmm.py $c 4 | sed "s/^/[rows $r] /"; done
  for d in 256 512; do for c in c3 c4; do
    CLEORA_CHUNK_ROWS=$r timeout 300 python scripts/run_spmm.py $c 4 $d | sed "s/^/[rows $r d $d] /"
  done; done
done
