#!/bin/bash
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
for w in C2_b1 C3 C2 C4; do bash tools/ab_libs.sh $w gpurun_ab/lib*.so; done
cp gpurun_ab/libE.so paper_2505_22913_b200/lib/libmustafar.so
for T in 4096 32768; do echo "E T=$T $(timeout 300 python tools/small_batch.py 1 $T 32 2>&1 | tail -1)" >> gpurun_out/small.txt; done
