mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-per-plan --no-configs"
$CMD > gpurun_out/plain_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_f64|gemm_tf32|axpby|split_planes|batched|identity|plan_cluster|count_nonfinite" -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_launches.log
