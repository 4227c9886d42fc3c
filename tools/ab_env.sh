#!/bin/bash
# dev: A/B of environment knobs on one library: bash tools/ab_env.sh <workload> "VAR=a" "VAR=b" ...
# each setting benched twice, interleaved, device-timed (8 layer caches).
w=$1; shift
mkdir -p gpurun_out
for rep in 1 2; do
  for e in "$@"; do
    r=$(env $e timeout 300 python bench.py --steps 10 --warmup 3 --no-dense --no-cpu-baseline --layers 8 --workload $w 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_layer_step'], d['decode_step_us_per_call_events'])")
    echo "$w $e rep$rep $r" | tee -a gpurun_out/ab.txt
  done
done
