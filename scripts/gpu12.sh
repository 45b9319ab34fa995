# 4 GPUs: multi parity with the owner-side pull, then C3 / C5 / C5E-peer A/B
mkdir -p gpurun_out/r13
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r13/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29591 tests/gpu_multi_parity.py > gpurun_out/r13/multi_parity_g4.log 2>&1; echo parity=$? >> gpurun_out/r13/status.txt
for pp in 1; do
  for c in C3 C5; do
    HP_PULL_PUSH=$pp timeout 300 $TR --master-port 29592 bench.py --gpus 4 --config $c --span 1 --steps 20 --no-e2e > gpurun_out/r13/${c}_pp${pp}.json 2>/dev/null
  done
  HP_PULL_PUSH=$pp timeout 300 $TR --master-port 29593 bench.py --gpus 4 --config C5E --span 1 --transport peer --steps 10 --no-e2e > gpurun_out/r13/C5E_peer_pp${pp}.json 2>/dev/null
  HP_PULL_PUSH=$pp timeout 300 $TR --master-port 29594 bench.py --gpus 4 --config C3 --span 2 --steps 20 --no-e2e > gpurun_out/r13/C3k2_pp${pp}.json 2>/dev/null
done
echo done >> gpurun_out/r13/status.txt
