#!/bin/bash
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
for W in C2 C4; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mstf_attn_warp -s 12 -c 1 \
   -o gpurun_out/prof_$W python bench.py --workload $W --steps 2 --warmup 3 --layers 4 --no-dense --no-cpu-baseline --no-graph > gpurun_out/ncu_$W.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 2 -c 1 \
   -o gpurun_out/prof_prefill python tools/prefill_time.py 16 32 8 4096 39 > gpurun_out/ncu_prefill.log 2>&1
