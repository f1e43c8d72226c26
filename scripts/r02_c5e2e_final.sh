#!/bin/bash
# opt-in c5 end-to-end parity of the final build (whole-graph oracle on the box host vs one iterate(4) call)
out=gpurun_out/${1:-r02_c5e2e_final}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
CLEORA_C5_E2E=1 timeout 2400 python -m pytest tests/test_gpu_c5_e2e.py -m gpu -q -s > $out/pytest_c5_e2e.log 2>&1; echo "e2e rc=$?"
tail -5 $out/pytest_c5_e2e.log
