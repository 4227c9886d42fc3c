#!/bin/bash
# GPU suite on a -DMSTF_BOUNDS=1 build of the final code (device-side traps in place of compute-sanitizer)
mkdir -p gpurun_out
MSTF_NVCC_EXTRA="-DMSTF_BOUNDS=1" python -m paper_2505_22913_b200.build --force > gpurun_out/build_bounds.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_bounds.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_bounds.log
python -m paper_2505_22913_b200.build --force > /dev/null 2>&1
