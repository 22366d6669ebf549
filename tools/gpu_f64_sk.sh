mkdir -p gpurun_out
for t in 0 8 9 1 3; do NSERIES_F64_TILE=$t TILE_D=500,768,1024,1280,1536,2048,2560,3072,4096 timeout 200 python tools/time_f64_sk.py; done > gpurun_out/f64_sk.txt 2>&1
