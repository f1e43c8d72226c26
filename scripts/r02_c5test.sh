#!/bin/bash
out=gpurun_out/${1:-r02_c5test}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 3000 python -m pytest tests/test_gpu_c5.py -m gpu -q -s > $out/pytest_c5.log 2>&1; echo "c5 rc=$?"; tail -4 $out/pytest_c5.log
