#!/bin/bash
# A/B (round 2, session 6): intra-CTA split-K fp64 tiles for small d (NSERIES_F64_TILE 10/11/12) vs 32x32 (4)
mkdir -p gpurun_out
O=gpurun_out/ks_ab.txt
: > $O
TILE_REF=1 NSERIES_F64_TILE=4 timeout 120 python tools/time_cfg2_tiles.py >> $O 2>&1
for i in 1 2; do
  for t in 4 10 11 12; do
    NSERIES_F64_TILE=$t timeout 120 python tools/time_cfg2_tiles.py >> $O 2>&1
    NSERIES_F64_TILE=$t TILE_D=512,768,1024,1280,1472 timeout 120 python tools/time_f64_sk.py >> $O 2>&1
  done
done
