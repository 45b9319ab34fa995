mkdir -p gpurun_out/r30
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r30/smoke.log 2>&1; echo smoke=$? >> gpurun_out/r30/status.txt
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r30/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/r30/status.txt
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29711 bench.py --gpus 4 > gpurun_out/r30/bench_n4.json 2>/dev/null; echo bench4=$? >> gpurun_out/r30/status.txt
timeout 300 $TR --master-port 29712 bench.py --gpus 4 --config C3 --span 1 --steps 20 --no-e2e > gpurun_out/r30/c3.json 2>/dev/null
