mkdir -p gpurun_out/r19
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29641 bench.py --gpus 4 --config C3 --span 1 --steps 20 --no-e2e > gpurun_out/r19/c3.json 2>/dev/null
timeout 300 $TR --master-port 29642 bench.py --gpus 4 --config HVD --span 1 --transport nvls --steps 30 --no-e2e > gpurun_out/r19/hvd_nvls.json 2>/dev/null
