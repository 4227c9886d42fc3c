#!/bin/bash
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_quant.py -q -x > gpurun_out/pytest_quant.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_quant.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -q -x > gpurun_out/pytest_parity.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_parity.log
