# final validation of the round: smoke, GPU suite (multi at 4), default benches, reference arm, ncu list
mkdir -p gpurun_out/final2
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final2/smoke.log 2>&1; echo smoke=$? >> gpurun_out/final2/status.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/final2/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/final2/status.txt
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/final2/bench_n1.json 2> gpurun_out/final2/bench_n1.err; echo bench1=$? >> gpurun_out/final2/status.txt
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference > gpurun_out/final2/ref_n1.json 2>/dev/null; echo ref=$? >> gpurun_out/final2/status.txt
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 2 --master-port 29751 bench.py --gpus 2 > gpurun_out/final2/bench_n2.json 2>/dev/null; echo bench2=$? >> gpurun_out/final2/status.txt
timeout 900 $TR --nproc-per-node 4 --master-port 29752 bench.py --gpus 4 > gpurun_out/final2/bench_n4.json 2>/dev/null; echo bench4=$? >> gpurun_out/final2/status.txt
timeout 900 $TR --nproc-per-node 4 --master-port 29753 bench.py --gpus 4 --impl reference > gpurun_out/final2/ref_n4.json 2>/dev/null; echo ref4=$? >> gpurun_out/final2/status.txt
