#!/bin/bash
mkdir -p gpurun_out
MSTF_NVCC_EXTRA="-DMSTF_TRACE=1" python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
for a in "8 131072 nf 16" "16 4096 nf 16"; do timeout 300 python tools/trace_attn.py $a >> gpurun_out/trace.txt 2>&1; done
