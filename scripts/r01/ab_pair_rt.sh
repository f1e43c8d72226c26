#!/bin/bash
# runtime pairing on/off (CLEORA_PAIR_ROWS) with the same binary -- the experiment of a reverted
# variant (a pair_rows kernel argument); kept as the record of DESIGN §7's measurement
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for p in 1 0; do
  export CLEORA_PAIR_ROWS=$p
  timeout 300 python scripts/run_batch.py | sed "s/^/[pair $p] f4 /"
  for c in c2 c3 c4; do timeout 300 python scripts/run_spmm.py $c 4 128 | sed "s/^/[pair $p] /"; done
  timeout 300 python scripts/run_spmm.py c4 4 64 | sed "s/^/[pair $p] /"
done
