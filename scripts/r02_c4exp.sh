#!/bin/bash
out=gpurun_out/${1:-r02_c4exp}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for args in "orig 1024" "relabel 1024" "orig 1024 40" "orig 1024 48" "orig 1024 56" "orig 1024 64" "colmod8192 1024" "colmod16384 1024" "colmod32768 1024" "orig 512" "colmod16384 512" "orig 256" "colmod32768 256"; do
  timeout 300 python scripts/r02_c4exp.py $args >> $out/c4exp.jsonl 2>> $out/c4exp.err
done
cat $out/c4exp.jsonl
