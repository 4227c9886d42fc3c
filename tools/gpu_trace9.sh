#!/bin/bash
# dev: phase timelines (C4, C2, C2_b1 fused) with the trace build of the final code
mkdir -p gpurun_out
MSTF_NVCC_EXTRA="-DMSTF_TRACE=1" python -m paper_2505_22913_b200.build --force > gpurun_out/build_tr.log 2>&1
for a in "8 131072 fused" "16 4096 fused" "1 4096 fused"; do timeout 300 python tools/trace_attn.py $a >> gpurun_out/trace9.txt 2>&1; done
python -m paper_2505_22913_b200.build --force > /dev/null 2>&1
