#!/bin/bash
# A/B: libA (HEAD) vs libE (ca=3) vs libE with MSTF_SKCA=0, interleaved
mkdir -p gpurun_out
one() { timeout 300 env $2 python bench.py --steps 10 --warmup 3 --no-dense --no-cpu-baseline --layers 8 --workload $1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_layer_step'])"; }
for w in C4 C2 C2_b1; do for rep in 1 2; do
  cp gpurun_ab/libA.so paper_2505_22913_b200/lib/libmustafar.so; echo "$w A $(one $w X=1)" >> gpurun_out/ab.txt
  cp gpurun_ab/libE.so paper_2505_22913_b200/lib/libmustafar.so; echo "$w E $(one $w X=1)" >> gpurun_out/ab.txt
  echo "$w E0 $(one $w MSTF_SKCA=0)" >> gpurun_out/ab.txt
done; done
