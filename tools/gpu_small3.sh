#!/bin/bash
mkdir -p gpurun_out
for so in gpurun_ab/libA.so gpurun_ab/libD.so; do
  cp $so paper_2505_22913_b200/lib/libmustafar.so
  for T in 64 4096; do
    timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,smsp__inst_executed.sum --clock-control none -k regex:"mstf_|append" -s 64 -c 6 --csv python tools/small_batch.py 1 $T 4 > gpurun_out/ncu_small_$(basename $so)_$T.csv 2>/dev/null
  done
done
