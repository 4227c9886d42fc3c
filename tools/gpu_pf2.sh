#!/bin/bash
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
for rep in 1 2; do for so in gpurun_ab/lib*.so; do cp $so paper_2505_22913_b200/lib/libmustafar.so
  for vb in 16 4; do echo "$(basename $so) $(timeout 300 python tools/prefill_time.py 16 32 8 4096 39 10 32 $vb 2>&1 | tail -1)" >> gpurun_out/ab.txt; done; done; done
