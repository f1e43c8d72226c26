#!/bin/bash
out=gpurun_out/${1:-r02_probe}
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; cat $out/build.log; exit 1; }
timeout 600 python scripts/r02_probe.py > $out/probe.jsonl 2> $out/probe.err; echo "probe rc=$?"
cat $out/probe.jsonl
