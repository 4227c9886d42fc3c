#!/bin/bash
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
for w in C2_b1 C2 C4; do bash tools/ab_libs.sh $w gpurun_ab/lib*.so; done
MSTF_NVCC_EXTRA="-DMSTF_TRACE=1" python -m paper_2505_22913_b200.build --force > gpurun_out/build_tr.log 2>&1
for a in "1 4096 fused 15"; do timeout 300 python tools/trace_attn.py $a >> gpurun_out/trace.txt 2>&1; done
