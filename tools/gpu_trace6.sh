#!/bin/bash
# dev: phase timeline at C4 (fused)
mkdir -p gpurun_out
MSTF_NVCC_EXTRA="-DMSTF_TRACE=1" python -m paper_2505_22913_b200.build --force > gpurun_out/build_tr.log 2>&1
for a in "8 131072 fused"; do timeout 300 python tools/trace_attn.py $a >> gpurun_out/trace6.txt 2>&1; done
