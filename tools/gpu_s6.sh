#!/bin/bash
# Harness (round 2, session 6 start): full GPU suite, race shake of the final tree, smoke, bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2s6_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2s6_tests.log
timeout 900 python tools/race_shake.py run > gpurun_out/r2s6_race_shake.txt 2>&1; echo "shake rc=$?" >> gpurun_out/r2s6_race_shake.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2s6_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2s6_bench.json 2> gpurun_out/r2s6_bench.err; echo "bench rc=$?" >> gpurun_out/r2s6_bench.err
