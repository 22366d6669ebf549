mkdir -p gpurun_out
for t in 0 10 11 12 13 14 15; do NSERIES_F64_TILE=$t TILE_D=500,768,1024,1280,1536 timeout 200 python tools/time_f64_sk.py; done > gpurun_out/f64_t2.txt 2>&1
