mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 python tools/peak_tcgen05.py 4 > gpurun_out/peak_tcgen05.json 2>&1; echo "peak rc=$?" >> gpurun_out/peak_tcgen05.json
timeout 900 python tools/race_shake.py run > gpurun_out/race_shake.txt 2>&1; echo "shake rc=$?" >> gpurun_out/race_shake.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
