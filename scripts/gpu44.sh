# A/B on one box: CTA-claimed dynamic tiles by launch class (HP_DYN, HP_DYN_MINLOADS, HP_DYN_PULLS)
D=gpurun_out/r44; mkdir -p $D
run() { # tag cfgargs env...
  tag=$1; cfg=$2; shift 2
  env "$@" timeout 300 python bench.py $cfg --warmup 5 --no-e2e --no-cpu-baseline > $D/$tag.json 2>>$D/err.log
  echo "$tag $(python -c "import json,sys;d=json.loads(open('$D/$tag.json').read().strip().splitlines()[-1]);print('%.4e'%d['value'],round(d['ms_per_step'],4),round(d['roofline']['frac'],4),{k:(v['n'],round(v['GBps'])) for k,v in d['launch_mix'].items()})")" >> $D/summary.txt
}
timeout 900 python -m pytest tests -m gpu -x -q > $D/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $D/pytest.log)" >> $D/summary.txt
for rep in 1 2 3; do
  run c2_dyn0_$rep "--steps 300" HP_DYN=0
  run c2_m2p1_$rep "--steps 300"
  run c2_m2p0_$rep "--steps 300" HP_DYN_PULLS=0
  run c2_m1p1_$rep "--steps 300" HP_DYN_MINLOADS=1
done
for rep in 1 2; do
  run c5_dyn0_$rep "--config C5 --steps 40" HP_DYN=0
  run c5_m2p1_$rep "--config C5 --steps 40"
  run c5_m2p0_$rep "--config C5 --steps 40" HP_DYN_PULLS=0
done
