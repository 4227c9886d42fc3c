#!/bin/bash
# round-2 evidence: launch lists (C4, C2_b1), full captures of the attention kernel (C4, C2) and prefill
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
for W in C4 C2_b1 C2; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"mstf_|append_kernel|prefill_kernel|set_counters" --csv \
   --log-file gpurun_out/r2_launches_$W.csv python bench.py --workload $W --steps 2 --warmup 3 --layers 8 --no-dense --no-cpu-baseline --no-graph > gpurun_out/ncu_l_$W.log 2>&1
done
for W in C4 C2; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mstf_attn_warp -s 12 -c 1 \
   -o gpurun_out/r2_prof_attn_$W python bench.py --workload $W --steps 2 --warmup 3 --layers 4 --no-dense --no-cpu-baseline --no-graph > gpurun_out/ncu_f_$W.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 2 -c 1 \
   -o gpurun_out/r2_prof_prefill python tools/prefill_time.py 16 32 8 4096 39 > gpurun_out/ncu_pf.log 2>&1
