#!/bin/bash
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build > gpurun_out/build.log 2>&1
for T in 64 512 4096; do timeout 300 python tools/small_batch.py 1 $T 32 >> gpurun_out/small.txt 2>&1; done
timeout 600 nsys --version >> gpurun_out/small.txt 2>&1
