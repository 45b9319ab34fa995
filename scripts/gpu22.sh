mkdir -p gpurun_out/r23
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r23/smoke.log 2>&1; echo smoke=$? >> gpurun_out/r23/status.txt
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r23/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/r23/status.txt
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/r23/bench_n1.json 2> gpurun_out/r23/bench_n1.err; echo bench=$? >> gpurun_out/r23/status.txt
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference > gpurun_out/r23/ref.json 2>/dev/null; echo ref=$? >> gpurun_out/r23/status.txt
