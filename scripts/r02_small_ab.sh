#!/bin/bash
out=gpurun_out/${1:-r02_small_ab}
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for i in 1 2; do
  timeout 300 python scripts/r02_small_ab.py scratch_r01 >> $out/ab.jsonl 2>> $out/ab.err
  timeout 300 python scripts/r02_small_ab.py . >> $out/ab.jsonl 2>> $out/ab.err
done
cat $out/ab.jsonl; tail -3 $out/ab.err
