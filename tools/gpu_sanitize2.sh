#!/bin/bash
mkdir -p gpurun_out
for w in C4 C2; do bash tools/ab_libs.sh $w gpurun_ab/lib*.so; done
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
T="tests/test_gpu_parity.py::test_attention_matches_oracle tests/test_gpu_parity.py::test_decode_step_equals_append_then_attention tests/test_gpu_quant.py"
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 --log-file gpurun_out/san_racecheck.log python -m pytest $T -q -x -p no:cacheprovider > gpurun_out/san_racecheck_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/san_racecheck_pytest.log
timeout 1200 compute-sanitizer --tool initcheck --print-limit 20 --log-file gpurun_out/san_initcheck.log python -m pytest "tests/test_gpu_parity.py::test_attention_matches_oracle" -q -x -p no:cacheprovider -k "case0 or case3 or case5" > gpurun_out/san_initcheck_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/san_initcheck_pytest.log
