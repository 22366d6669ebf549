#!/bin/bash
# Run on the GPU box (via gpurun): plain short bench, then ncu launch list and one full capture.
set -x
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-per-plan"
$CMD > gpurun_out/plain_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_f64 -s 6 -c 1 -o gpurun_out/prof_gemm_f64 -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "profile rc=$?"
