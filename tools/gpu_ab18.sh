#!/bin/bash
# dev: 32-bit record cursor for the TMA issue (addresses formed at issue time) vs 64-bit pointers
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_ab18.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_ab18.log
for w in C4 C2 C4_q4; do bash tools/ab_libs.sh $w gpurun_ab/lib_pfx2.so gpurun_ab/lib_r32.so; done
