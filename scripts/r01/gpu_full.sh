#!/bin/bash
# Full round-end style validation: build, pytest -m gpu (c5 included), smoke, bench (c2), bench --impl
# reference, the 8(f) measurements.  Logs in gpurun_out/<tag>/.
tag=${1:-full}
out=gpurun_out/$tag
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"; cat $out/smoke.log
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"; cat $out/bench.json
timeout 600 python bench.py --impl reference > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc=$?"; cat $out/bench_ref.json
timeout 900 python scripts/bench_next.py > $out/bench_next.json 2> $out/bench_next.err; echo "next rc=$?"
