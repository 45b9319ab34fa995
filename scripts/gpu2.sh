# exchange placements on 2 GPUs + multicast probe
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29521 scripts/probe_mc.py > gpurun_out/probe_mc.log 2>&1
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
for c in C3 C5; do
  timeout 600 $TR --master-port 29522 bench.py --gpus 2 --config $c --span 1 --steps 20 > gpurun_out/x_${c}_g2.json 2> gpurun_out/x_${c}_g2.err
done
timeout 600 $TR --master-port 29523 bench.py --gpus 2 --config C4 --steps 20 > gpurun_out/x_C4_g2_edlocal.json 2> gpurun_out/x_C4_g2.err
