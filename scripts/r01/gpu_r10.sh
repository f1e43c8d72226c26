#!/bin/bash
# chunk caps per engine/row size: full GPU suite, 8(f) rows, per-config SpMM times
out=gpurun_out/${1:-r10}
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail $out/build.log; exit 1; }
timeout 1300 python -m pytest tests -q -m gpu -x > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest.log
timeout 900 python scripts/bench_next.py > $out/bench_next.json 2> $out/bench_next.err; echo "next rc=$?"
for d in 128 256 512; do for c in c2 c3 c4; do timeout 300 python scripts/run_spmm.py $c 4 $d; done; done > $out/times.txt 2>&1; cat $out/times.txt
