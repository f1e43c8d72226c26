#!/bin/bash
# A/B of a reverted variant: T_0 values built from the hash word with bit operations (the variant,
# then the default) vs the int->float conversion (-DCLEORA_HASH_I2F, now the only code); record of DESIGN §7
python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "init or c1_full or tiny" 2>&1 | tail -1
timeout 300 python scripts/time_init.py | sed "s/^/[bits] /"
CLEORA_NVCC_EXTRA=-DCLEORA_HASH_I2F python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1
timeout 300 python scripts/time_init.py | sed "s/^/[i2f] /"
python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1
timeout 300 python scripts/time_init.py | sed "s/^/[bits] /"
