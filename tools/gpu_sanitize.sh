#!/bin/bash
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
T="tests/test_gpu_parity.py::test_attention_matches_oracle tests/test_gpu_parity.py::test_decode_step_equals_append_then_attention tests/test_gpu_quant.py"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --log-file gpurun_out/san_$tool.log python -m pytest $T -q -x -p no:cacheprovider > gpurun_out/san_${tool}_pytest.log 2>&1
  echo "rc=$?" >> gpurun_out/san_${tool}_pytest.log
done
