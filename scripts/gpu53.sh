# A/B: phase-A applies three sources per step (this build) vs pairs (previous build, HP_LIB)
D=gpurun_out/r53; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $D/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $D/pytest.log)" >> $D/summary.txt
run() { tag=$1; cfg=$2; shift 2
  env "$@" timeout 300 python bench.py $cfg --warmup 5 --no-e2e --no-cpu-baseline > $D/$tag.json 2>>$D/err.log
  echo "$tag $(python -c "import json,sys;d=json.loads(open('$D/$tag.json').read().strip().splitlines()[-1]);print('%.4e'%d['value'],round(d['ms_per_step'],4),round(d['roofline']['frac'],4),{k:(v['n'],round(v['GBps'])) for k,v in d['launch_mix'].items()})")" >> $D/summary.txt
}
for rep in 1 2 3; do
  run c2_prev_$rep "--steps 300" HP_LIB=paper_2005_14038_b200/libhetpipe_prev.so
  run c2_tri_$rep "--steps 300"
done
for rep in 1 2; do
  run c5_prev_$rep "--config C5 --steps 40" HP_LIB=paper_2005_14038_b200/libhetpipe_prev.so
  run c5_tri_$rep "--config C5 --steps 40"
done
