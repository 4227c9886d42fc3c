#!/bin/bash
# dev: GPU tests (working tree), worker-weight skew A/B, traces with and without skew
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
for w in C4 C2 C5; do bash tools/ab_env.sh $w MSTF_SKEW=0 MSTF_SKEW=3 MSTF_SKEW=6; done
MSTF_NVCC_EXTRA="-DMSTF_TRACE=1" python -m paper_2505_22913_b200.build --force > gpurun_out/build_tr.log 2>&1
for sk in 0 3 6; do MSTF_SKEW=$sk timeout 300 python tools/trace_attn.py 8 131072 fused >> gpurun_out/trace7.txt 2>&1; done
python -m paper_2505_22913_b200.build --force > /dev/null 2>&1
