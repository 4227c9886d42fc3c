#!/bin/bash
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "prefill or append or fullsize or full" > gpurun_out/pytest_pf.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_pf.log
bash tools/ab_prefill.sh gpurun_ab/lib*.so
