# NVLS kernel with dynamic tiles (HP_NVLS_DYN): 2-GPU parity and C5E / HVD A/B
D=gpurun_out/r49; mkdir -p $D
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
HP_MULTI_RANDOM=4 timeout 900 $TR --master-port 29791 tests/gpu_multi_parity.py > $D/multi_g2.log 2>&1; echo "parity=$? $(grep -c OK $D/multi_g2.log) $(tail -1 $D/multi_g2.log)" >> $D/summary.txt
run() { tag=$1; cfg=$2; shift 2
  env "$@" timeout 300 $TR --master-port $((29800 + RANDOM % 100)) bench.py --gpus 2 $cfg --no-e2e --no-cpu-baseline > $D/$tag.json 2>>$D/err.log
  echo "$tag $(python -c "import json,sys;d=json.loads(open('$D/$tag.json').read().strip().splitlines()[-1]);x=d.get('exchange_roofline') or {};print('%.4e'%d['value'],round(d['ms_per_step'],4),x.get('frac'),d['config'].get('lockstep_batches'))")" >> $D/summary.txt
}
for rep in 1 2; do
  run c5e_d0_$rep "--config C5E --span 1 --transport nvls --steps 40" HP_NVLS_DYN=0
  run c5e_d1_$rep "--config C5E --span 1 --transport nvls --steps 40"
  run hvd_d0_$rep "--config HVD --span 1 --transport nvls --steps 40" HP_NVLS_DYN=0
  run hvd_d1_$rep "--config HVD --span 1 --transport nvls --steps 40"
done
