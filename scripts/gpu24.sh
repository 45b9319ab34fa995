mkdir -p gpurun_out/r25
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
HP_MULTI_RANDOM=40 timeout 1200 $TR --master-port 29671 tests/gpu_multi_parity.py > gpurun_out/r25/multi_g4.log 2>&1; echo g4=$? >> gpurun_out/r25/status.txt
HP_MULTI_RANDOM=40 HP_MULTI_SEED=7 HP_PULL_PUSH=0 timeout 1200 $TR --master-port 29672 tests/gpu_multi_parity.py > gpurun_out/r25/multi_g4_reader.log 2>&1; echo g4r=$? >> gpurun_out/r25/status.txt
