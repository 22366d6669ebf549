# fp64 engine raster band (tile-rows per band) 8 (default) / 16 / 32: DRAM bytes per launch and plan time
mkdir -p gpurun_out
O=gpurun_out/f64_group.txt
: > $O
for i in 1 2; do
  for lib in paper_2602_11843_b200/libnseries.so tools/variants/f64_g16.so tools/variants/f64_g32.so; do
    echo "== $lib" >> $O; NSERIES_LIB=$lib timeout 200 python tools/time_f64_plan.py >> $O 2>&1
  done
done
for lib in paper_2602_11843_b200/libnseries.so tools/variants/f64_g16.so tools/variants/f64_g32.so; do
  echo "== ncu $lib" >> $O
  NSERIES_LIB=$lib timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_f64 -s 18 -c 6 --csv python tools/time_f64_plan.py 2>/dev/null | grep -E "dram__|gpu__time" >> $O
done
