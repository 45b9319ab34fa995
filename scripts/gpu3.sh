# lockstep transports on 2 GPUs: parity, then C5E bench per transport
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NG:-2} --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29531 tests/gpu_multi_parity.py > gpurun_out/multi_parity.log 2>&1; echo parity=$? >> gpurun_out/status3.txt
for t in peer nccl nvls; do
  timeout 600 $TR --master-port 29532 bench.py --gpus ${NG:-2} --config C5E --span 1 --transport $t --steps 10 > gpurun_out/c5e_${t}_g${NG:-2}.json 2> gpurun_out/c5e_${t}.err; echo bench_$t=$? >> gpurun_out/status3.txt
done
