mkdir -p gpurun_out/r16
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29621 bench.py --gpus 4 --config C3 --span 1 --steps 20 --no-e2e > gpurun_out/r16/c3.json 2>/dev/null
timeout 300 $TR --master-port 29622 bench.py --gpus 4 --config C5E --span 1 --transport nvls --steps 10 --no-e2e > gpurun_out/r16/c5e_nvls.json 2>/dev/null
timeout 300 $TR --master-port 29623 bench.py --gpus 4 --config C5E --span 1 --transport peer --steps 10 --no-e2e > gpurun_out/r16/c5e_peer.json 2>/dev/null
timeout 300 $TR --master-port 29624 bench.py --gpus 4 --config HVD --span 1 --transport nccl --steps 30 --no-e2e > gpurun_out/r16/hvd_nccl.json 2>/dev/null
timeout 300 $TR --master-port 29625 bench.py --gpus 4 --config HVD --span 1 --transport nvls --steps 30 --no-e2e > gpurun_out/r16/hvd_nvls.json 2>/dev/null
