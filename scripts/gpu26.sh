mkdir -p gpurun_out/r27
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for D in 0 4 32; do
  timeout 300 $TR --master-port 29681 bench.py --gpus 4 --config C5 --span 1 --D $D --steps 10 --no-e2e > gpurun_out/r27/c5_n8_D$D.json 2>/dev/null
  timeout 300 $TR --master-port 29682 bench.py --gpus 4 --config C5 --num-vw 4 --span 1 --D $D --steps 10 --no-e2e > gpurun_out/r27/c5_n4_D$D.json 2>/dev/null
done
