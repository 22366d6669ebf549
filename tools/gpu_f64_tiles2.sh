# fp64 engine: further tile shapes (2 CTAs/SM 64x128 / 128x64, BK16 128x128) vs the 128x128x32 default
mkdir -p gpurun_out
O=gpurun_out/f64_tiles2.txt
: > $O
for i in 1 2; do
  for t in 1 5 6 7; do
    NSERIES_LIB=tools/variants/f64_tiles.so NSERIES_F64_TILE=$t TILE_D=2048,3072,4096,8192 timeout 300 python tools/time_f64_sk.py >> $O 2>&1
  done
done
for t in 1 5 6; do echo "plan tile $t" >> $O; NSERIES_LIB=tools/variants/f64_tiles.so NSERIES_F64_TILE=$t timeout 200 python tools/time_f64_plan.py >> $O 2>&1; done
