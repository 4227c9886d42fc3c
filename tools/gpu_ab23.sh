#!/bin/bash
# dev: the small-problem CTA merge as its own instantiation, two-phase (weights per warp and head first)
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_ab23.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_ab23.log
for w in C2_b1 C4 C2 C3; do bash tools/ab_libs.sh $w gpurun_ab/lib_head.so gpurun_ab/lib_cm.so; done
