# Does dynamic tile scheduling pay by launch size? C2 / C3 (60M) vs C4 / C5 (144M) on one B200
D=gpurun_out/r46; mkdir -p $D
run() { # tag cfgargs env...
  tag=$1; cfg=$2; shift 2
  env "$@" timeout 300 python bench.py $cfg --warmup 5 --no-e2e --no-cpu-baseline > $D/$tag.json 2>>$D/err.log
  echo "$tag $(python -c "import json,sys;d=json.loads(open('$D/$tag.json').read().strip().splitlines()[-1]);print('%.4e'%d['value'],round(d['ms_per_step'],4),round(d['roofline']['frac'],4),{k:(v['n'],round(v['GBps'])) for k,v in d['launch_mix'].items()})")" >> $D/summary.txt
}
for rep in 1 2; do
  run c2_dyn0_$rep "--steps 300" HP_DYN=0
  run c2_dyn1_$rep "--steps 300"
  run c4_dyn0_$rep "--config C4 --steps 40" HP_DYN=0
  run c4_dyn1_$rep "--config C4 --steps 40"
  run c3_dyn0_$rep "--config C3 --steps 40" HP_DYN=0
  run c3_dyn1_$rep "--config C3 --steps 40"
  run c5_dyn0_$rep "--config C5 --steps 40" HP_DYN=0
  run c5_dyn1_$rep "--config C5 --steps 40"
done
