#!/bin/bash
out=gpurun_out/${1:-r02_ipc}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_ipc.py tests/test_gpu_shard.py tests/test_gpu_multi.py -m gpu -q > $out/pytest.log 2>&1; echo "rc=$?"; tail -3 $out/pytest.log
