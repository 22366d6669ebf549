#!/bin/bash
# Harness: full GPU check of the tree (tests, bench, launch list, one ncu --set full capture of
# the fp32 engine).  Outputs land in gpurun_out/.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'nseries|gemm|axpby|split|batched|identity|plan_' -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
TIME_D=4096 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32x3 -s 5 -c 1 \
  -o gpurun_out/tf32_full -f python tools/time_f32_gemm.py > gpurun_out/ncu_tf32.log 2>&1
