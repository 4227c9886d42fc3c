#!/bin/bash
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_quant.py tests/test_gpu_graph.py -q -x > gpurun_out/pytest_parity.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_parity.log
for w in C4 C2 C2_b1; do bash tools/ab_libs.sh $w gpurun_ab/lib*.so; done
for so in gpurun_ab/lib*.so; do cp $so paper_2505_22913_b200/lib/libmustafar.so; echo $so >> gpurun_out/small.txt; timeout 300 python tools/small_batch.py 1 4096 32 >> gpurun_out/small.txt 2>&1; done
