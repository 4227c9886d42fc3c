#!/bin/bash
# dev: phase timelines (C2 fused, C2_b1 fused) with the trace build
mkdir -p gpurun_out
MSTF_NVCC_EXTRA="-DMSTF_TRACE=1" python -m paper_2505_22913_b200.build --force > gpurun_out/build_tr.log 2>&1
for a in "16 4096 fused" "1 4096 fused" "16 4096 nf"; do timeout 300 python tools/trace_attn.py $a >> gpurun_out/trace5.txt 2>&1; done
