#!/bin/bash
# copy a finished evidence run (tools/gpu_final2.sh) from gpurun_out/ into profiles/ with a prefix
# usage: bash tools/export_profiles.sh r2f
P=${1:-r2f}
G=gpurun_out
for w in C4 C5 C3 C2 C2_s50 C2_b1 C4_q4 C2_q4; do cp $G/bench_$w.json profiles/${P}_bench_$w.json; done
cp $G/bench_ref.json profiles/${P}_bench_reference.json
for w in C4 C2 C2_b1; do cp $G/launches_$w.csv profiles/${P}_launches_$w.csv; done
for w in C4 C2; do
  ncu -i $G/prof_attn_$w.ncu-rep --page details --csv > profiles/${P}_ncu_attn_${w}_details.csv 2>/dev/null
  ncu -i $G/prof_attn_$w.ncu-rep --page raw --csv > profiles/${P}_ncu_attn_${w}_raw.csv 2>/dev/null
done
ncu -i $G/prof_prefill.ncu-rep --page details --csv > profiles/${P}_ncu_prefill_C2_details.csv 2>/dev/null
ncu -i $G/prof_prefill.ncu-rep --page raw --csv > profiles/${P}_ncu_prefill_C2_raw.csv 2>/dev/null
cp $G/pytest_gpu.log profiles/${P}_pytest_gpu.log
cp $G/smoke.log profiles/${P}_smoke.log
