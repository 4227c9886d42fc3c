#!/bin/bash
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_quant.py -q -x > gpurun_out/pytest_quant.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_quant.log
for w in C4_q4 C2_q4; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --no-dense --layers 8 > gpurun_out/q_$w.json 2> gpurun_out/q_$w.err
done
