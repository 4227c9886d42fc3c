#!/bin/bash
# dev: which token preps load the stored prefix addresses (MSTF_PREFIX_SEL 1 = K, 2 = V, 3 = both)
mkdir -p gpurun_out
for w in C4 C2; do bash tools/ab_libs.sh $w gpurun_ab/lib_sel3.so gpurun_ab/lib_sel1.so gpurun_ab/lib_sel2.so gpurun_ab/lib_base.so; done
