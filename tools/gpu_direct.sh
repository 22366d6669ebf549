# NSERIES_SHARDED_DIRECT: sharded GPU tests, timing of config 5 in 8 blocks (gather vs direct)
mkdir -p gpurun_out
O=gpurun_out/direct.txt
: > $O
timeout 1200 python -m pytest tests/test_gpu_sharded.py -x -q >> $O 2>&1; echo "tests rc=$?" >> $O
timeout 600 python tools/time_sharded.py >> $O 2>&1
TIME_D=8192 timeout 600 python tools/time_sharded.py >> $O 2>&1
