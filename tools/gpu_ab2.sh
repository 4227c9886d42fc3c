#!/bin/bash
mkdir -p gpurun_out
for w in C2 C4; do bash tools/ab_libs.sh $w gpurun_ab/lib*.so; done
cp gpurun_ab/libC.so paper_2505_22913_b200/lib/libmustafar.so
for q in 4 2 1; do
  r=$(MSTF_QMIN=$q timeout 300 python bench.py --steps 10 --warmup 3 --no-dense --no-cpu-baseline --workload C2_b1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_layer_step'], d['decode_step_us_per_call_events'])")
  echo "C2_b1 qmin=$q $r" | tee -a gpurun_out/ab.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_parity.log
