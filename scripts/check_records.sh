#!/bin/bash
# The sparse exchange's record-reading K5 (vr_packets_index + *_records) against the dense
# slab path: the 2-process tests compare losses, images and gradients with one process.
set -u
mkdir -p gpurun_out
for V in 1 0; do
  VR_RECORDS_K5=$V timeout 900 python -m pytest tests/test_gpu_multirank.py "tests/test_gpu_configs.py::test_c2_two_processes_match_single_process_oracle_and_c1" -q -x -m gpu > gpurun_out/records_$V.log 2>&1
  echo "VR_RECORDS_K5=$V: $(tail -1 gpurun_out/records_$V.log)"
done
