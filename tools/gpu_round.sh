#!/bin/bash
# Round measurement script (run under gpurun): tests, bench lines, launch list, ncu capture.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/smi.txt
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
for w in C2_b1 C2_s50 C3 C4 C5; do
  timeout 600 python bench.py --steps 5 --warmup 3 --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"mstf_|append_kernel|prefill_kernel|set_counters" --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-dense --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mstf_attn -s 40 -c 1 \
   -o gpurun_out/prof_bench python bench.py --steps 2 --warmup 3 --no-dense --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout 300 python tools/prefill_time.py > gpurun_out/prefill_time.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 2 -c 1 \
   -o gpurun_out/prof_prefill python tools/prefill_time.py 16 32 8 4096 39 > gpurun_out/ncu_prefill.log 2>&1
timeout 2000 python tools/batch_sweep.py > gpurun_out/batch_sweep.jsonl 2> gpurun_out/batch_sweep.err
ls -la gpurun_out
