#!/bin/bash
mkdir -p gpurun_out
MSTF_NVCC_EXTRA="-DMSTF_TRACE=1" python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
for a in "16 4096" "16 4096 fused" "1 4096" "1 4096 fused" "1 64" "8 131072"; do timeout 300 python tools/trace_attn.py $a >> gpurun_out/trace.txt 2>&1; done
