mkdir -p gpurun_out/r28
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for D in 0 4 32; do
  timeout 300 $TR --master-port 29691 bench.py --gpus 4 --config C5 --span 1 --D $D --pull lazy --steps 10 --no-e2e > gpurun_out/r28/c5_n8_D${D}_lazy.json 2>/dev/null
done
timeout 300 python bench.py --config C5 --D 32 --pull lazy --steps 30 --no-e2e --no-cpu-baseline > gpurun_out/r28/c5_1gpu_D32_lazy.json 2>/dev/null
timeout 300 python bench.py --config C5 --D 32 --steps 30 --no-e2e --no-cpu-baseline > gpurun_out/r28/c5_1gpu_D32.json 2>/dev/null
