#!/bin/bash
# Harness (round 2, session 5 end): full GPU suite, race shake of the final tree, smoke, bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final6_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/final6_tests.log
timeout 900 python tools/race_shake.py run > gpurun_out/final6_race_shake.txt 2>&1; echo "shake rc=$?" >> gpurun_out/final6_race_shake.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final6_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/final6_bench.json 2> gpurun_out/final6_bench.err; echo "bench rc=$?" >> gpurun_out/final6_bench.err
