#!/bin/bash
# quick bench lines (8 layers unless given) for a list of workloads + prefill timing
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
for w in "$@"; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/q_$w.json 2> gpurun_out/q_$w.err
done
timeout 300 python tools/prefill_time.py > gpurun_out/prefill_time.txt 2>&1
