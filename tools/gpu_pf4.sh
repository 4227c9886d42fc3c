#!/bin/bash
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_output_aware.py tests/test_gpu_quant.py -q -x > gpurun_out/pytest_pf.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_pf.log
bash tools/gpu_pf3.sh
