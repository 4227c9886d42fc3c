#!/bin/bash
# A/B of prebuilt variants (gpurun_ab/lib*.so) at C2 and C4, then the current tree's parity tests
mkdir -p gpurun_out
for w in C2 C4; do bash tools/ab_libs.sh $w gpurun_ab/lib*.so; done
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -q -x > gpurun_out/pytest_parity.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_parity.log
timeout 300 python tools/prefill_time.py > gpurun_out/prefill_time.txt 2>&1
