#!/bin/bash
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build > gpurun_out/build.log 2>&1
one() { timeout 300 env $2 python bench.py --steps 10 --warmup 3 --no-dense --no-cpu-baseline --layers 8 --workload $1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_layer_step'])"; }
for cfg in "X=1" "MSTF_COMBSUB_MAX=1" "MSTF_COMBSUB_MAX=2" "MSTF_QMIN=8" "MSTF_QMIN=8 MSTF_COMBSUB_MAX=1" "MSTF_QMIN=6 MSTF_COMBSUB_MAX=2" "MSTF_QMIN=3"; do
  echo "C2_b1 $cfg $(one C2_b1 "$cfg") $(one C2_b1 "$cfg")" >> gpurun_out/ab.txt
done
