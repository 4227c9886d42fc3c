#!/bin/bash
# quick iteration: parity, quick bench (C2, C4), ncu of the attention kernel at C2
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_parity.log
for w in C2 C4; do
  timeout 300 python bench.py --steps 10 --warmup 3 --workload $w --layers 8 --no-dense --no-cpu-baseline > gpurun_out/q_$w.json 2> gpurun_out/q_$w.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mstf_attn_warp -s 12 -c 1 \
   -o gpurun_out/prof_iter python bench.py --workload C2 --steps 2 --warmup 3 --layers 4 --no-dense --no-cpu-baseline > gpurun_out/ncu_iter.log 2>&1
