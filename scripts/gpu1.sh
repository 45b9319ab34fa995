set -x
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo bench1=$? >> gpurun_out/status.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo bench2=$? >> gpurun_out/status.txt
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo ncu=$? >> gpurun_out/status.txt
