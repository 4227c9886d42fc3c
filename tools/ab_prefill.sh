#!/bin/bash
# dev: A/B prebuilt library variants on the bulk prune+compress (tools/prefill_time.py), ABAB
mkdir -p gpurun_out
for rep in 1 2; do
  for so in "$@"; do
    cp "$so" paper_2505_22913_b200/lib/libmustafar.so
    echo "$(basename $so) rep$rep $(timeout 300 python tools/prefill_time.py 16 32 8 4096 39 2>&1 | tail -1)" | tee -a gpurun_out/ab.txt
  done
done
