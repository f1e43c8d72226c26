#!/bin/bash
out=gpurun_out/${1:-r02_lazy3}
mkdir -p $out
bash scripts/r02_lazy.sh ${1:-r02_lazy3}
bash scripts/r02_ncu_lazy.sh ${1:-r02_lazy3}_ncu
