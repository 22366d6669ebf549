#!/bin/bash
# Harness (GPU box): compute-sanitizer over the hand-synchronised kernels.
#   tools/sanitize.sh TOOL [CASE ...]     TOOL in memcheck | racecheck | synccheck | initcheck
# Each case first runs plain (must exit 0), then under the sanitizer; logs in gpurun_out/.
TOOL=${1:-memcheck}; shift
CASES=${*:-"cluster2d warp_f32 cta_f32 cta_f64 splitk_f32 tf32 f64_tiled"}
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out
for c in $CASES; do
  timeout 300 python tools/sanitize_cases.py "$c" > "gpurun_out/san_plain_$c.log" 2>&1
  echo "plain $c rc=$?" >> gpurun_out/san_summary.txt
  EXTRA=""
  [ "$TOOL" = racecheck ] && EXTRA="--racecheck-report all"
  timeout 1200 $CS --tool "$TOOL" $EXTRA --target-processes all --print-limit 50 \
    python tools/sanitize_cases.py "$c" > "gpurun_out/san_${TOOL}_$c.log" 2>&1
  rc=$?
  echo "$TOOL $c rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san_${TOOL}_$c.log | tail -2 | tr '\n' ' ')" \
    >> gpurun_out/san_summary.txt
done
