# A/B on one box: previous build vs separate prefetch instance (off / on, <= 4 or 3 load streams)
mkdir -p gpurun_out/r40
run() { # tag cfgargs env...
  tag=$1; cfg=$2; shift 2
  env "$@" timeout 300 python bench.py $cfg --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r40/$tag.json 2>>gpurun_out/r40/err.log
  echo "$tag $(python -c "import json,sys;d=json.loads(open('gpurun_out/r40/$tag.json').read().strip().splitlines()[-1]);print('%.4e'%d['value'],round(d['ms_per_step'],4),round(d['roofline']['frac'],4),{k:(v['n'],round(v['GBps'])) for k,v in d['launch_mix'].items()})")" >> gpurun_out/r40/summary.txt
}
for rep in 1 2 3; do
  run c2_prev_$rep "--steps 300" HP_LIB=paper_2005_14038_b200/libhetpipe_prev.so
  run c2_pf0_$rep "--steps 300" HP_PREFETCH=0
  run c2_pf1m4_$rep "--steps 300" HP_PREFETCH=1
  run c2_pf1m3_$rep "--steps 300" HP_PREFETCH=1 HP_PREFETCH_MAXLOADS=3
done
for rep in 1 2; do
  run c5_prev_$rep "--config C5 --steps 40" HP_LIB=paper_2005_14038_b200/libhetpipe_prev.so
  run c5_pf0_$rep "--config C5 --steps 40" HP_PREFETCH=0
  run c5_pf1m4_$rep "--config C5 --steps 40" HP_PREFETCH=1
done
