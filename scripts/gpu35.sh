# distributed CONVEX / F: randomized 4-GPU and 2-GPU parity, GPU suite
mkdir -p gpurun_out/r35
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
HP_MULTI_RANDOM=40 HP_MULTI_SEED=11 timeout 1500 $TR --nproc-per-node 4 --master-port 29771 tests/gpu_multi_parity.py > gpurun_out/r35/multi_g4.log 2>&1; echo g4=$? >> gpurun_out/r35/status.txt
HP_MULTI_RANDOM=30 HP_MULTI_SEED=12 timeout 1200 $TR --nproc-per-node 2 --master-port 29772 tests/gpu_multi_parity.py > gpurun_out/r35/multi_g2.log 2>&1; echo g2=$? >> gpurun_out/r35/status.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r35/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/r35/status.txt
