# L2 bulk-prefetch sweep (HP_PREFETCH = rounds ahead) on C2 / C4-shard / C5, then parity with prefetch on
mkdir -p gpurun_out/r38
for pf in 0 1 2 4 0 1 2; do
  HP_PREFETCH=$pf timeout 300 python bench.py --steps 300 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r38/c2_pf$pf.json 2>>gpurun_out/r38/err.log
  echo "c2 pf=$pf $(python -c "import json,sys;d=json.loads(open('gpurun_out/r38/c2_pf$pf.json').read().strip().splitlines()[-1]);print('%.4e'%d['value'],round(d['ms_per_step'],4),round(d['roofline']['frac'],4),{k:(v['n'],round(v['GBps'])) for k,v in d['launch_mix'].items()})")" >> gpurun_out/r38/summary.txt
done
for pf in 0 1 2; do
  HP_PREFETCH=$pf timeout 300 python bench.py --config C5 --steps 40 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r38/c5_pf$pf.json 2>>gpurun_out/r38/err.log
  echo "c5 pf=$pf $(python -c "import json,sys;d=json.loads(open('gpurun_out/r38/c5_pf$pf.json').read().strip().splitlines()[-1]);print('%.4e'%d['value'],round(d['ms_per_step'],4),round(d['roofline']['frac'],4))")" >> gpurun_out/r38/summary.txt
done
HP_PREFETCH=1 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r38/pytest_pf1.log 2>&1; echo "pytest pf1 rc=$?" >> gpurun_out/r38/summary.txt
tail -2 gpurun_out/r38/pytest_pf1.log >> gpurun_out/r38/summary.txt
