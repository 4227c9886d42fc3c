#!/bin/bash
# dev: one TMA stage issued before the first block (the second once it has landed) vs two
mkdir -p gpurun_out
cp gpurun_ab/lib_pre1.so paper_2505_22913_b200/lib/libmustafar.so
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -m gpu -q -x > gpurun_out/pytest_gpu_ab25.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_ab25.log
for w in C2 C3 C4 C2_b1; do bash tools/ab_libs.sh $w gpurun_ab/lib_pre2.so gpurun_ab/lib_pre1.so; done
