#!/bin/bash
# register-kernel changes: bitwise engine tests + LDG-path timings (f4 batch, c1, c2-c4 at d = 128 / 256)
tag=${1:-r8}
out=gpurun_out/$tag
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
timeout 1300 python -m pytest tests -q -m gpu -x > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest.log
timeout 300 python scripts/run_batch.py | sed "s/^/f4 /"
timeout 300 python scripts/run_spmm.py c1 4
for d in 128 256; do for c in c2 c3 c4; do timeout 300 python scripts/run_spmm.py $c 4 $d; done; done
