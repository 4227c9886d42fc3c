#!/bin/bash
# dev: GPU tests on the working tree, then interleaved A/B of prebuilt libraries
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
for w in C4 C2 C2_b1; do bash tools/ab_libs.sh $w gpurun_ab/lib_base.so gpurun_ab/lib_new.so; done
