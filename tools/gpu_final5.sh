#!/bin/bash
# Harness (round 2, session 5): full GPU check -- GPU test suite, bench, ncu launch list of the
# bench step (run plain first), --set full captures of the fp64 engine, the fp32 engine and the
# batched config-4 kernel.  Outputs in gpurun_out/.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-per-plan --no-configs"
$CMD > gpurun_out/plain_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f64 -s 6 -c 1 -o gpurun_out/prof_gemm_f64 -f $CMD > gpurun_out/ncu_full_f64.log 2>&1
TIME_D=4096 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32x3 -s 5 -c 1 -o gpurun_out/prof_tf32 -f python tools/time_f32_gemm.py > gpurun_out/ncu_full_tf32.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:batched_warp -s 3 -c 1 -o gpurun_out/prof_batched -f python tools/time_batched.py > gpurun_out/ncu_full_batched.log 2>&1
echo done > gpurun_out/final_done.txt
