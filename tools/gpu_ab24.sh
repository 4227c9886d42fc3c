#!/bin/bash
# dev: env-knob sweep (cost model, combine sub-warps, min cost per worker) + GPU tests of the prefill launch change
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_ab24.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_ab24.log
bash tools/ab_env.sh C2 MSTF_SKCS=2 MSTF_SKCS=1 MSTF_SKCS=3 MSTF_COMBSUB_MAX=1 MSTF_COMBSUB_MAX=8 MSTF_QMIN=8
bash tools/ab_env.sh C4 MSTF_SKCS=2 MSTF_SKCS=1 MSTF_COMBSUB_MAX=1 MSTF_COMBSUB_MAX=8
bash tools/ab_env.sh C2_b1 MSTF_SKCS=2 MSTF_SKCS=1 MSTF_COMBSUB_MAX=8
