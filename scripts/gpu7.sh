# 2 GPUs: gpu tests, smoke, N=1 and N=2 bench (default contract), C5E per transport
mkdir -p gpurun_out/r7
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r7/smoke.log 2>&1; echo smoke=$? >> gpurun_out/r7/status.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r7/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/r7/status.txt
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/r7/bench_n1.json 2> gpurun_out/r7/bench_n1.err; echo bench1=$? >> gpurun_out/r7/status.txt
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29571 bench.py --gpus 2 > gpurun_out/r7/bench_n2.json 2> gpurun_out/r7/bench_n2.err; echo bench2=$? >> gpurun_out/r7/status.txt
for t in peer nccl nvls; do
  timeout 600 $TR --master-port 29572 bench.py --gpus 2 --config C5E --span 1 --transport $t --steps 10 --no-e2e > gpurun_out/r7/c5e_${t}_g2.json 2>/dev/null
done
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r7/ref.json 2> gpurun_out/r7/ref.err; echo ref=$? >> gpurun_out/r7/status.txt
