#!/bin/bash
# dev: pre-issue 1 for the fp16 payload, 2 for the 4-bit payload; GPU tests; q4 bench lines
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
for w in C4_q4 C2_q4; do bash tools/ab_libs.sh $w gpurun_ab/lib_pre2.so gpurun_ab/lib_preq.so; done
python -m paper_2505_22913_b200.build --force > /dev/null 2>&1
for w in C4_q4 C2_q4; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
