#!/bin/bash
# dev: A/B prebuilt library variants on one box: bash tools/ab_libs.sh <workload> gpurun_ab/libX.so ...
# each variant is copied over lib/libmustafar.so (newer than the sources, so no rebuild) and
# benched twice, interleaved (ABAB), device-timed.
w=$1; shift
mkdir -p gpurun_out
for rep in 1 2; do
  for so in "$@"; do
    cp "$so" paper_2505_22913_b200/lib/libmustafar.so
    r=$(timeout 300 python bench.py --steps 10 --warmup 3 --no-dense --no-cpu-baseline --layers 8 --workload $w 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_layer_step'], d['decode_step_us_per_call_events'])")
    echo "$w $(basename $so) rep$rep $r" | tee -a gpurun_out/ab.txt
  done
done
