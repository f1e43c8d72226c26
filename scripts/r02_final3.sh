#!/bin/bash
# every GPU test (c5 included) and smoke on the closing build
out=gpurun_out/${1:-r02_final3}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"
s=$(date +%s); CLEORA_PARITY_LOG=$out/parity.jsonl timeout 3600 python -m pytest tests -m gpu -q -rs > $out/pytest.log 2>&1; echo "pytest rc=$? wall $(( $(date +%s) - s )) s"; tail -5 $out/pytest.log
cat $out/parity.jsonl
