mkdir -p gpurun_out
for t in 0 4 5 6 7 3; do NSERIES_F64_TILE=$t TILE_D=500,768,1024,1280,1472,1536 timeout 120 python tools/time_f64_tiles.py; done > gpurun_out/f64_tiles.txt 2>&1
