#!/bin/bash
# lazy steps skip the stores of never-gathered rows: tests of the lazy / half-row / shard / IPC paths, then
# the c4 bench A/B (CLEORA_KEEP_UNGATHERED=0/1 alternating, twice)
out=gpurun_out/${1:-r02_drop}
mkdir -p $out
export CLEORA_GEN_CACHE=/tmp/cleora_gen
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo BUILD FAILED; tail -30 $out/build.log; exit 1; }
s=$(date +%s); timeout 1500 python -m pytest -q -x -rs tests/test_gpu_parity.py -k "lazy or half or partial_t0 or c4_full or composab" tests/test_gpu_shard.py tests/test_gpu_ipc.py tests/test_gpu_fetch_nonzero.py > $out/pytest.log 2>&1; echo "pytest rc=$? wall $(( $(date +%s) - s )) s"; tail -4 $out/pytest.log
for r in 1 2; do
  for keep in 0 1; do
    CLEORA_KEEP_UNGATHERED=$keep timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-secondary > $out/bench_keep${keep}_$r.json 2> $out/bench_keep${keep}_$r.err
    python -c "import json,sys; d=json.loads(open('$out/bench_keep${keep}_$r.json').read().strip().splitlines()[-1]); print('keep=$keep run $r', round(d['ms_per_step'],2), 'ms/step spmm', round(d['roofline']['kernel_ms'],3), 'clk', d['clocks']['sm_mhz'])"
  done
done | tee $out/ab.txt
