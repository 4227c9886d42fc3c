#!/bin/bash
# dev: pre-issue 1 vs 2 on the 4-bit payload
mkdir -p gpurun_out
for w in C4_q4 C2_q4 C5; do bash tools/ab_libs.sh $w gpurun_ab/lib_pre2.so gpurun_ab/lib_pre1.so; done
