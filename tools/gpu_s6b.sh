#!/bin/bash
# Harness (round 2, session 6): ncu look at cuBLAS's sm_100 DGEMM kernel at d = 4096 (launch shape,
# pipes, stalls) -- its kernel is named Kernel2 -- next to the engine's plain product
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none -k regex:Kernel2 -s 2 -c 1 --page details python tools/cublas_dgemm_once.py > gpurun_out/cublas_ncu_details.txt 2>&1
timeout 300 ncu --set full --clock-control none -k regex:Kernel2 -s 2 -c 1 --page raw --csv python tools/cublas_dgemm_once.py > gpurun_out/cublas_ncu_raw.csv 2>&1
