mkdir -p gpurun_out
(
for lib in tools/variants/orig.so paper_2602_11843_b200/libnseries.so; do
  echo "== $lib"
  for i in 1 2; do NSERIES_LIB=$lib timeout 120 python tools/time_f64_plan.py; done
  for t in 0 1 3; do NSERIES_LIB=$lib NSERIES_F64_TILE=$t TILE_D=1024,2048,4096 timeout 200 python tools/time_f64_sk.py; done
done
NSERIES_DEBUG_LAUNCH=1 NSERIES_F64_TILE=9 TILE_D=500,1024,1536,2048,3072,4096 timeout 200 python tools/time_f64_sk.py
) > gpurun_out/f64_ab.txt 2>&1
