#!/bin/bash
# dev: rebuild with each set of extra nvcc flags ("-" = none) and run a scan command
# usage: tools/ab_flags.sh "<scan command>" flags1 flags2 ...
cmd="$1"; shift
for f in "$@"; do
  if [ "$f" = "-" ]; then MSTF_NVCC_EXTRA="" python -m paper_2505_22913_b200.build --force > /dev/null 2>&1;
  else MSTF_NVCC_EXTRA="$f" python -m paper_2505_22913_b200.build --force > /dev/null 2>&1; fi
  TAG="[$f]" bash -c "$cmd"
done
python -m paper_2505_22913_b200.build --force > /dev/null 2>&1
