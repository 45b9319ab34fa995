# parity of the CUDA path under the prefetch / dynamic-tile knobs; U=4 for pull launches (perf)
D=gpurun_out/r48; mkdir -p $D
for v in "HP_DYN=0" "HP_PREFETCH=0" "HP_DYN_MINLOADS=1" "HP_TICK_U=4" "HP_PREFETCH=2 HP_PREFETCH_MAXLOADS=16" "HP_DYN_MINLOADS=1 HP_GRID=1"; do
  tag=$(echo $v | tr ' ' '_')
  env $v timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "random_configs or convex_random or update_frequency_random or full_size" > $D/$tag.log 2>&1; echo "$tag=$? $(tail -1 $D/$tag.log)" >> $D/status.txt
done
run() { # tag cfgargs env...
  tag=$1; cfg=$2; shift 2
  env "$@" timeout 300 python bench.py $cfg --warmup 5 --no-e2e --no-cpu-baseline > $D/$tag.json 2>>$D/err.log
  echo "$tag $(python -c "import json,sys;d=json.loads(open('$D/$tag.json').read().strip().splitlines()[-1]);print('%.4e'%d['value'],round(d['ms_per_step'],4),round(d['roofline']['frac'],4),{k:(v['n'],round(v['GBps'])) for k,v in d['launch_mix'].items()})")" >> $D/summary.txt
}
for rep in 1 2; do
  run c2_def_$rep "--steps 300"
  run c2_u4_$rep "--steps 300" HP_TICK_U=4
  run c5_def_$rep "--config C5 --steps 40"
  run c5_u4_$rep "--config C5 --steps 40" HP_TICK_U=4
done
