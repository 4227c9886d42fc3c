#!/bin/bash
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build > gpurun_out/build.log 2>&1
for q in 1 2 4 8; do MSTF_QMIN=$q timeout 300 python tools/small_batch.py 1 4096 32 >> gpurun_out/small.txt 2>&1; echo "qmin=$q" >> gpurun_out/small.txt; done
timeout 300 python tools/small_batch.py 4 4096 32 >> gpurun_out/small.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"mstf_attn_warp|mstf_warp_combine" -s 6 -c 2 -o gpurun_out/prof_small python tools/small_batch.py 1 4096 4 > gpurun_out/ncu_small.log 2>&1
