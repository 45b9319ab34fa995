mkdir -p gpurun_out/r14
for w in 1 2 4 8 16; do
  timeout 300 python scripts/shard_probe.py --world $w >> gpurun_out/r14/probe.jsonl 2>>gpurun_out/r14/probe.err
  HP_PDL=0 timeout 300 python scripts/shard_probe.py --world $w >> gpurun_out/r14/probe_nopdl.jsonl 2>>gpurun_out/r14/probe.err
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29601 bench.py --gpus 4 --no-e2e > gpurun_out/r14/c2_n4.json 2>/dev/null
