#!/bin/bash
# dev: (1) 4-bit bulk prefill as its own template instance: fp16 / 4-bit prefill vs the previous build;
# (2) prefix counts packed in one word (one 4-byte load per token prep) vs three stored addresses
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_ab22.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_ab22.log
for rep in 1 2; do
  for so in gpurun_ab/lib_zb.so gpurun_ab/lib_pq4b.so; do
    cp "$so" paper_2505_22913_b200/lib/libmustafar.so
    for vb in 16 4; do
      echo "$(basename $so) rep$rep $(timeout 300 python tools/prefill_time.py 16 32 8 4096 39 10 32 $vb 2>&1 | tail -1)" | tee -a gpurun_out/ab.txt
    done
  done
done
for w in C4 C2 C4_q4; do bash tools/ab_libs.sh $w gpurun_ab/lib_pq4b.so gpurun_ab/lib_pp2.so; done
