mkdir -p gpurun_out
(timeout 300 python tools/check_sharded_multi.py 1024 9 9; timeout 300 python tools/check_sharded_multi.py 4096 15 15 15; timeout 600 python tools/check_sharded_multi.py) > gpurun_out/check_multi1.txt 2>&1; echo "rc=$?" >> gpurun_out/check_multi1.txt
