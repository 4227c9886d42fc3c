#!/bin/bash
# ncu full capture of the attention kernel at C2 (4 layers) + launch list
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
W=${1:-C2}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mstf_attn_warp -s 12 -c 1 \
   -o gpurun_out/prof_r2_$W python bench.py --workload $W --steps 2 --warmup 3 --layers 4 --no-dense --no-cpu-baseline > gpurun_out/ncu_r2_$W.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"mstf_|append_kernel|prefill_kernel" --csv \
   --log-file gpurun_out/launches_r2_$W.csv python bench.py --workload $W --steps 2 --warmup 3 --layers 4 --no-dense --no-cpu-baseline > gpurun_out/ncu_launch_r2.log 2>&1
