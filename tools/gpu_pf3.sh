#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do for so in gpurun_ab/lib*.so; do cp $so paper_2505_22913_b200/lib/libmustafar.so
  echo "$(basename $so) $(timeout 300 python tools/prefill_time.py 16 32 8 4096 39 10 32 16 2>&1 | tail -1)" >> gpurun_out/ab.txt
  echo "$(basename $so) $(timeout 300 python tools/prefill_time.py 8 32 8 32768 39 5 32 16 2>&1 | tail -1)" >> gpurun_out/ab.txt; done; done
