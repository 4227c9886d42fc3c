#!/bin/bash
# round-2 final evidence: tests, smoke, bench lines, reference arm, ncu launch lists + full
# captures, compute-sanitizer on the attention parity tests
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/smi.txt
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
for w in C2 C2_b1 C3 C5 C2_s50 C4_q4 C2_q4; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for W in C4 C2 C2_b1; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"mstf_|append_kernel|prefill_kernel|set_counters" --csv \
   --log-file gpurun_out/launches_$W.csv python bench.py --workload $W --steps 2 --warmup 3 --layers 8 --no-dense --no-cpu-baseline --no-graph > gpurun_out/ncu_l_$W.log 2>&1
done
for W in C4 C2; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mstf_attn_warp -s 12 -c 1 \
   -o gpurun_out/prof_attn_$W python bench.py --workload $W --steps 2 --warmup 3 --layers 4 --no-dense --no-cpu-baseline --no-graph > gpurun_out/ncu_f_$W.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 2 -c 1 \
   -o gpurun_out/prof_prefill python tools/prefill_time.py 16 32 8 4096 39 > gpurun_out/ncu_pf.log 2>&1
# (compute-sanitizer is closed on this pool: see tools/gpu_bounds.sh for the device-side checks)
