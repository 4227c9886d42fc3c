#!/bin/bash
# dev: state check -- GPU tests, smoke, short bench lines (no dense baselines)
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
for w in C4 C2 C2_b1; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --no-dense > gpurun_out/chk_$w.json 2> gpurun_out/chk_$w.err
done
