mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "small or cluster or d64 or cfg1 or config1" > gpurun_out/small_tests.log 2>&1; echo "rc=$?" >> gpurun_out/small_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 120 python tools/time_small.py > gpurun_out/time_small.txt 2>&1
