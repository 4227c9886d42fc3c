#!/bin/bash
# r2 kernel bring-up: parity tests, sanitizer on the small cases, r1 vs r2 quick bench lines.
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_parity.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "attention_matches or decode_step_equals or schedules" > gpurun_out/memcheck.log 2>&1
echo "rc=$?" >> gpurun_out/memcheck.log
for impl in r2 r1; do
  for w in C2 C2_b1 C4; do
    MSTF_ATTN=$impl timeout 300 python bench.py --steps 10 --warmup 3 --workload $w --no-dense --no-cpu-baseline > gpurun_out/q_${impl}_$w.json 2> gpurun_out/q_${impl}_$w.err
  done
done
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
