#!/bin/bash
# Run on the GPU box (via gpurun): full bench, then a short bench under ncu (launch list of our
# kernels + one full capture of the FP64 engine and of the FP32 engine).
set -x
python bench.py > gpurun_out/bench.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-per-plan"
$CMD > gpurun_out/plain_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"nseries|gemm|axpby|split|batched|identity" -c 120 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_f64 -s 6 -c 1 -o gpurun_out/prof_gemm_f64 -f $CMD > gpurun_out/ncu_full.log 2>&1
python tools/check_tf32.py 4096 > gpurun_out/plain_tf32.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 1 -c 1 -o gpurun_out/prof_tf32 -f python tools/check_tf32.py 4096 > gpurun_out/ncu_tf32.log 2>&1
echo "profile rc=$?"
