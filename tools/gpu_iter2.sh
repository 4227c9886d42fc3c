#!/bin/bash
# iteration: build, parity tests, quick bench lines (C4, C2, C2_s50), one ncu --set full capture at C4
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_quant.py -q -x > gpurun_out/pytest_parity.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_parity.log
for w in C4 C2 C2_s50; do
  timeout 300 python bench.py --steps 10 --warmup 3 --workload $w --layers 8 --no-dense --no-cpu-baseline > gpurun_out/q_$w.json 2> gpurun_out/q_$w.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mstf_attn_warp -s 12 -c 1 \
   -o gpurun_out/prof_iter python bench.py --workload C4 --steps 2 --warmup 3 --layers 4 --no-dense --no-cpu-baseline --no-graph > gpurun_out/ncu_iter.log 2>&1
