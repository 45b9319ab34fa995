mkdir -p gpurun_out/r24
for v in 0 1 2 3; do
  if [ $v = 0 ]; then L=""; else L=paper_2005_14038_b200/libhetpipe_ld$v.so; fi
  for rep in 1 2; do
    HP_LIB=$L timeout 300 python bench.py --steps 300 --no-e2e --no-cpu-baseline > gpurun_out/r24/ld${v}_$rep.json 2>/dev/null
  done
done
