#!/bin/bash
out=gpurun_out/${1:-r02_gpu9}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
timeout 2400 python -m pytest tests/test_gpu_shard.py tests/test_gpu_multi.py tests/test_gpu_ipc.py -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log
