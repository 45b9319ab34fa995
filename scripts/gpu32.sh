mkdir -p gpurun_out/r33
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
HP_NVLS_SPLIT=60 HP_MULTI_RANDOM=4 timeout 900 $TR --master-port 29741 tests/gpu_multi_parity.py > gpurun_out/r33/multi_g4_split60.log 2>&1; echo parity=$? >> gpurun_out/r33/status.txt
for sp in 100 85 70 55 40; do
  HP_NVLS_SPLIT=$sp timeout 300 $TR --master-port 29742 bench.py --gpus 4 --config HVD --span 1 --transport nvls --steps 30 --no-e2e > gpurun_out/r33/hvd_sp$sp.json 2>/dev/null
  HP_NVLS_SPLIT=$sp timeout 300 $TR --master-port 29743 bench.py --gpus 4 --config C5E --span 1 --transport nvls --steps 10 --no-e2e > gpurun_out/r33/c5e_sp$sp.json 2>/dev/null
done
