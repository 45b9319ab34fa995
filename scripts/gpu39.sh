# A/B on one box: previous build vs prefetch off / on for launches with <= 4 (or 2) load streams
mkdir -p gpurun_out/r39
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 300 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r39/$tag.json 2>>gpurun_out/r39/err.log
  echo "$tag $(python -c "import json,sys;d=json.loads(open('gpurun_out/r39/$tag.json').read().strip().splitlines()[-1]);print('%.4e'%d['value'],round(d['ms_per_step'],4),round(d['roofline']['frac'],4),{k:(v['n'],round(v['GBps'])) for k,v in d['launch_mix'].items()})")" >> gpurun_out/r39/summary.txt
}
for rep in 1 2 3; do
  run prev_$rep HP_LIB=paper_2005_14038_b200/libhetpipe_prev.so
  run pf0_$rep HP_PREFETCH=0
  run pf1m4_$rep HP_PREFETCH=1
  run pf1m2_$rep HP_PREFETCH=1 HP_PREFETCH_MAXLOADS=2
  run pf2m4_$rep HP_PREFETCH=2
done
