# full GPU suite after the cvt.rn split change + ncu source capture of the batched kernel
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2c_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2c_tests.log
bash tools/gpu_bw_src.sh
timeout 300 python tools/time_f32_gemm.py > gpurun_out/r2c_f32_gemm.txt 2>&1
