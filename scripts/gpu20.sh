mkdir -p gpurun_out/r21
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29651 bench.py --gpus 4 --config C4 --steps 30 > gpurun_out/r21/c4_n4.json 2>gpurun_out/r21/c4.err
