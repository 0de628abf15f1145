#!/bin/bash
# ncu capture of the c4 hash-grid gather (HBM-resident tables)
python scripts/bench_hash.py c4 1048576 > gpurun_out/hb_c4.log 2>&1 && \
ncu --set full --clock-control none -k regex:k_hash_fwd -s 12 -c 1 -o gpurun_out/prof_hash_c4 \
    python scripts/bench_hash.py c4 1048576 > gpurun_out/ncu_hash_c4.log 2>&1
cat gpurun_out/hb_c4.log
