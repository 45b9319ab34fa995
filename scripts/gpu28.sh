mkdir -p gpurun_out/r29
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
HP_MULTI_RANDOM=16 timeout 1200 $TR --master-port 29701 tests/gpu_multi_parity.py > gpurun_out/r29/multi_g4.log 2>&1; echo parity=$? >> gpurun_out/r29/status.txt
timeout 300 $TR --master-port 29702 bench.py --gpus 4 --config HVD --span 1 --transport nccl --steps 30 --no-e2e > gpurun_out/r29/hvd_nccl.json 2>/dev/null
timeout 300 $TR --master-port 29703 bench.py --gpus 4 --config C5E --span 1 --transport nccl --steps 10 --no-e2e > gpurun_out/r29/c5e_nccl.json 2>/dev/null
