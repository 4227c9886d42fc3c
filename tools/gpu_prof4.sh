#!/bin/bash
# dev: ncu --set full of one attention launch at C4 (current tree) + phase traces
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mstf_attn_warp -s 12 -c 1 \
   -o gpurun_out/prof_attn_C4_new python bench.py --workload C4 --steps 2 --warmup 3 --layers 4 --no-dense --no-cpu-baseline --no-graph > gpurun_out/ncu_f_C4.log 2>&1
MSTF_NVCC_EXTRA="-DMSTF_TRACE=1" python -m paper_2505_22913_b200.build --force > gpurun_out/build_tr.log 2>&1
for a in "8 131072 fused" "16 4096 fused"; do timeout 300 python tools/trace_attn.py $a >> gpurun_out/trace8.txt 2>&1; done
python -m paper_2505_22913_b200.build --force > /dev/null 2>&1
