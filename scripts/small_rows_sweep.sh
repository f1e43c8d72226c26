#!/bin/bash
# gather engine x light-chunk rows at d = 128 / 64 (f4 batch, c2-c4 at small d)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for m in ldg async; do for r in 31 8; do
  export CLEORA_GATHER=$m CLEORA_CHUNK_ROWS=$r
  timeout 300 python scripts/run_batch.py | sed "s/^/[$m rows $r] f4 /"
  for c in c2 c3 c4; do timeout 300 python scripts/run_spmm.py $c 4 128 | sed "s/^/[$m rows $r d 128] /"; done
  timeout 300 python scripts/run_spmm.py c4 4 64 | sed "s/^/[$m rows $r d 64] /"
done; done
