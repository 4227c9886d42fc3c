#!/bin/bash
mkdir -p gpurun_out
python -m paper_2505_22913_b200.build --force > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_seqsplit.py -q -x > gpurun_out/pytest_parity.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_parity.log
for w in C2 C2_b1 C4; do bash tools/ab_libs.sh $w gpurun_ab/lib*.so; done
cp gpurun_ab/libE.so paper_2505_22913_b200/lib/libmustafar.so
for q in 1 2 4; do for a in "1 4096 fused" "16 4096 fused"; do echo "qmin=$q $a $(MSTF_QMIN=$q timeout 300 python tools/trace_attn.py $a 2>&1 | tail -1)" >> gpurun_out/trace.txt; done; done
for q in 2 1; do r=$(MSTF_QMIN=$q timeout 300 python bench.py --steps 10 --warmup 3 --no-dense --no-cpu-baseline --layers 8 --workload C2_b1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['us_per_layer_step'])"); echo "C2_b1 qmin=$q $r" >> gpurun_out/ab.txt; done
