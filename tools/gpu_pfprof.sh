#!/bin/bash
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 2 -c 1 \
   -o gpurun_out/prof_prefill python tools/prefill_time.py 16 32 8 4096 39 > gpurun_out/ncu_pf.log 2>&1
