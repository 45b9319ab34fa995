# 4 GPUs: multi parity (incl. layer-RR), HVD per transport, C5E layer-RR, C5 layer-RR, C2 pmp timing
mkdir -p gpurun_out/r8
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r8/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29581 tests/gpu_multi_parity.py > gpurun_out/r8/multi_parity_g4.log 2>&1; echo parity=$? >> gpurun_out/r8/status.txt
for t in peer nccl nvls; do
  timeout 300 $TR --master-port 29582 bench.py --gpus 4 --config HVD --span 1 --transport $t --steps 30 --no-e2e > gpurun_out/r8/hvd_${t}_g4.json 2>/dev/null
done
for t in peer nvls; do
  timeout 300 $TR --master-port 29583 bench.py --gpus 4 --config C5E --span 1 --transport $t --ps layer_rr --steps 10 --no-e2e > gpurun_out/r8/c5e_${t}_lrr_g4.json 2>/dev/null
done
timeout 300 $TR --master-port 29584 bench.py --gpus 4 --config C5 --span 1 --ps layer_rr --steps 10 --no-e2e > gpurun_out/r8/c5_lrr_g4.json 2>/dev/null
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --timing pmp --steps 30 --no-e2e --no-cpu-baseline > gpurun_out/r8/c2_pmp_n1.json 2>/dev/null
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --config C3 --timing pmp --steps 30 --no-e2e --no-cpu-baseline > gpurun_out/r8/c3_pmp_n1.json 2>/dev/null
echo done >> gpurun_out/r8/status.txt
