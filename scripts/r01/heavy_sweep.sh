#!/bin/bash
# heavy-row threshold vs SpMM time at d = 128 / 256 / 512 (register kernel and cp.async ring)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for h in 64 128 256 512; do
  for d in 128 256 512; do for c in c2 c4; do CLEORA_HEAVY_THRESH=$h timeout 300 python scripts/run_spmm.py $c 4 $d | sed "s/^/[heavy $h] /"; done; done
done
