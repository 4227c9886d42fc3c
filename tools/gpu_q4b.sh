#!/bin/bash
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "q4" > gpurun_out/pytest_fs_q4.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_fs_q4.log
for w in C4_q4 C2_q4; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --no-dense > gpurun_out/q_$w.json 2> gpurun_out/q_$w.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mstf_attn_warp -s 12 -c 1 \
   -o gpurun_out/prof_C4_q4 python bench.py --workload C4_q4 --steps 2 --warmup 3 --layers 4 --no-dense --no-cpu-baseline --no-graph > gpurun_out/ncu_C4_q4.log 2>&1
