set -u
mkdir -p gpurun_out
cd tmp_ab && python paper_2404_16221_b200/csrc/build.py > /dev/null 2>&1
timeout 900 python -m pytest "tests/test_gpu_configs.py::test_c2_two_processes_match_single_process_oracle_and_c1" -q -s -m gpu > ../gpurun_out/g10_old.log 2>&1
cd ..
grep "per-sample\|passed\|failed" gpurun_out/g10_old.log | cut -c1-200
