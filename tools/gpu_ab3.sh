#!/bin/bash
# dev A/B of prebuilt libraries (gpurun_ab/lib*.so) on C4 and C2, plus parity of the default build
mkdir -p gpurun_out
for w in C4 C2; do bash tools/ab_libs.sh $w gpurun_ab/lib*.so; done
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_quant.py -q -x > gpurun_out/pytest_parity.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_parity.log
