#!/bin/bash
# dev: warp-uniform TMA operands (shuffled cursor + elect.sync issue) vs the r32 build
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_ab19.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_ab19.log
for w in C4 C2 C4_q4 C2_b1; do bash tools/ab_libs.sh $w gpurun_ab/lib_r32.so gpurun_ab/lib_uni.so; done
