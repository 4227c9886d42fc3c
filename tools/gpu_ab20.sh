#!/bin/bash
# dev: bitmap slots of a partial block zeroed in the stage (unconditional bitmap loads) vs predicated loads
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_ab20.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_ab20.log
for w in C4 C2 C2_b1 C4_q4; do bash tools/ab_libs.sh $w gpurun_ab/lib_uni.so gpurun_ab/lib_zb.so; done
