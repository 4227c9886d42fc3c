#!/bin/bash
# dev: GPU tests on a -DMSTF_BOUNDS=1 build (device-side bounds / invariant traps in place of
# compute-sanitizer), then the normal build: 4-bit bench lines and prefill timings
mkdir -p gpurun_out
MSTF_NVCC_EXTRA="-DMSTF_BOUNDS=1" python -m paper_2505_22913_b200.build --force > gpurun_out/build_bounds.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_bounds.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_bounds.log
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
for w in C4_q4 C2_q4; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
for vb in 16 4; do timeout 300 python tools/prefill_time.py 16 32 8 4096 39 10 32 $vb >> gpurun_out/prefill_times.txt 2>&1; done
timeout 300 python tools/prefill_time.py 8 32 8 131072 39 3 32 4 >> gpurun_out/prefill_times.txt 2>&1
