#!/bin/bash
# A/B: T_0 value from the hash word without (default) / with (-DCLEORA_HASH_I2F) an int->float convert
python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "init or c1_full or tiny" 2>&1 | tail -1
timeout 300 python scripts/time_init.py | sed "s/^/[bits] /"
CLEORA_NVCC_EXTRA=-DCLEORA_HASH_I2F python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1
timeout 300 python scripts/time_init.py | sed "s/^/[i2f] /"
python paper_2102_02302_b200/_build.py --force > /dev/null 2>&1
timeout 300 python scripts/time_init.py | sed "s/^/[bits] /"
