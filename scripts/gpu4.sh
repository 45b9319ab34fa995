# 4 GPUs: multi parity, C5E per transport, C3/C5 exchange placements
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29541 tests/gpu_multi_parity.py > gpurun_out/multi_parity_g4.log 2>&1; echo parity=$? >> gpurun_out/status4.txt
for t in peer nccl nvls; do
  timeout 600 $TR --master-port 29542 bench.py --gpus 4 --config C5E --span 1 --transport $t --steps 10 > gpurun_out/c5e_${t}_g4.json 2> gpurun_out/c5e_${t}_g4.err; echo bench_$t=$? >> gpurun_out/status4.txt
done
timeout 600 $TR --master-port 29543 bench.py --gpus 4 --config C3 --span 1 --steps 20 > gpurun_out/c3_g4.json 2> gpurun_out/c3_g4.err
timeout 600 $TR --master-port 29544 bench.py --gpus 4 --config C5 --span 1 --steps 10 > gpurun_out/c5_g4.json 2> gpurun_out/c5_g4.err
nvidia-smi nvlink --help > gpurun_out/nvlink_help.txt 2>&1
nvidia-smi nvlink -gt d -i 0 > gpurun_out/nvlink_gt.txt 2>&1
