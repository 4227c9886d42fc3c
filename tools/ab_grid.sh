#!/bin/bash
# dev: A/B prebuilt variants on tools/grid_scan.py points (default grid), ABAB
mkdir -p gpurun_out
for rep in 1 2; do
  for so in "$@"; do
    cp "$so" paper_2505_22913_b200/lib/libmustafar.so
    timeout 600 python -c "
import sys; sys.path.insert(0, 'tools')
import grid_scan as g
for b in (1, 2, 16): g.scan(b, grids=())
g.scan(1, T=65536, grids=())
" 2>&1 | sed "s/^/$(basename $so) rep$rep /" | tee -a gpurun_out/ab.txt
  done
done
