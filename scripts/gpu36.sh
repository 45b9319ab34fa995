mkdir -p gpurun_out/r36
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
HP_MULTI_RANDOM=8 timeout 1200 $TR --master-port 29781 tests/gpu_multi_parity.py > gpurun_out/r36/multi_g4.log 2>&1; echo parity=$? >> gpurun_out/r36/status.txt
timeout 600 $TR --master-port 29782 bench.py --gpus 4 --config C3 --span 1 --steps 20 > gpurun_out/r36/c3_e2e.json 2>gpurun_out/r36/c3.err; echo c3=$? >> gpurun_out/r36/status.txt
timeout 600 $TR --master-port 29783 bench.py --gpus 4 --config HVD --span 1 --transport nvls --steps 30 > gpurun_out/r36/hvd_e2e.json 2>gpurun_out/r36/hvd.err; echo hvd=$? >> gpurun_out/r36/status.txt
