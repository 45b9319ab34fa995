mkdir -p gpurun_out/r17
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for u in 1 2 4 8; do
  HP_TICK_U=$u timeout 300 $TR --master-port 29631 bench.py --gpus 4 --config C5E --span 1 --transport peer --steps 10 --no-e2e > gpurun_out/r17/c5e_peer_u$u.json 2>/dev/null
  HP_TICK_U=$u timeout 300 $TR --master-port 29632 bench.py --gpus 4 --config C3 --span 1 --steps 20 --no-e2e > gpurun_out/r17/c3_u$u.json 2>/dev/null
done
