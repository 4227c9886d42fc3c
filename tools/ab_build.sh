#!/bin/bash
# dev: swap in attention.cu variants (copies saved as tools/ab_attention_<name>.cu, not
# committed), rebuild, run a step scan for each (A/B on one box)
for v in "$@"; do
  cp tools/ab_attention_$v.cu paper_2505_22913_b200/csrc/attention.cu
  python -m paper_2505_22913_b200.build --force > /dev/null 2>&1
  TAG=$v timeout 200 python tools/step_scan.py
done
cp tools/ab_attention_cur.cu paper_2505_22913_b200/csrc/attention.cu
python -m paper_2505_22913_b200.build --force > /dev/null 2>&1
