# NSERIES_SHARDED_DIRECT incl. the peer-arena path: sharded GPU tests, bench --sharded(-direct) with 1 rank
mkdir -p gpurun_out
O=gpurun_out/direct2.txt
: > $O
timeout 1200 python -m pytest tests/test_gpu_sharded.py -x -q >> $O 2>&1; echo "tests rc=$?" >> $O
timeout 600 python bench.py --sharded --steps 5 --warmup 1 >> $O 2>/dev/null; echo "bench sharded rc=$?" >> $O
timeout 600 python bench.py --sharded --sharded-direct --steps 5 --warmup 1 >> $O 2>/dev/null; echo "bench sharded direct rc=$?" >> $O
