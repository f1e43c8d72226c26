#!/bin/bash
out=gpurun_out/${1:-r02_ab_arena}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for v in 1 0 1 0; do
  if [ $v = 1 ]; then export CLEORA_NO_ARENA=1; else unset CLEORA_NO_ARENA; fi
  echo -n "no_arena=$v "; timeout 300 python scripts/r02_c1_trace.py c1
  echo -n "no_arena=$v f4/c1 "; timeout 300 python scripts/r02_small_ab.py . | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v,4) for k,v in d.items() if k!='lib'})"
done
unset CLEORA_NO_ARENA
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py tests/test_gpu_batch.py tests/test_gpu_shard.py -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest.log
