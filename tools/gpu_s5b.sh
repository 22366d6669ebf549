# session 5: filtered launch list of the bench step, cuBLAS DGEMM at small d, engine GEMM at the same d
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-per-plan --no-configs"
$CMD > gpurun_out/plain_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_f64|gemm_tf32|axpby|split_planes|batched|identity|plan_cluster|count_nonfinite" -c 400 --csv --log-file gpurun_out/launches_f.csv $CMD > gpurun_out/ncu_launches_f.log 2>&1
timeout 300 python tools/cublas_small.py > gpurun_out/cublas_small.txt 2>&1
TILE_D=500,768,1024,1536,2048,4096 timeout 300 python tools/time_f64_sk.py >> gpurun_out/cublas_small.txt 2>&1
