mkdir -p gpurun_out/r15
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for u in 2 4 8; do for xb in 0 296; do
  HP_NVLS_U=$u HP_XBLOCKS=$xb timeout 300 $TR --master-port 29611 bench.py --gpus 4 --config HVD --span 1 --transport nvls --steps 30 --no-e2e > gpurun_out/r15/hvd_u${u}_xb${xb}.json 2>/dev/null
done; done
