mkdir -p gpurun_out
for t in 4 10; do NSERIES_F64_TILE=$t TILE_D=128,192,256,320,384,448,500,576,640,704,768 timeout 200 python tools/time_f64_sk.py; done > gpurun_out/f64_small.txt 2>&1
