mkdir -p gpurun_out/r32
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29731 tests/gpu_multi_parity.py > gpurun_out/r32/multi_g4.log 2>&1; echo parity=$? >> gpurun_out/r32/status.txt
for fb in 1 0; do
  HP_FLAG_BARRIER=$fb timeout 300 $TR --master-port 29732 bench.py --gpus 4 --config C3 --span 1 --steps 20 --no-e2e > gpurun_out/r32/c3_fb$fb.json 2>/dev/null
  HP_FLAG_BARRIER=$fb timeout 300 $TR --master-port 29733 bench.py --gpus 4 --config HVD --span 1 --transport nvls --steps 30 --no-e2e > gpurun_out/r32/hvd_fb$fb.json 2>/dev/null
  HP_FLAG_BARRIER=$fb timeout 300 $TR --master-port 29734 bench.py --gpus 4 --config C5 --span 1 --steps 10 --no-e2e > gpurun_out/r32/c5_fb$fb.json 2>/dev/null
done
