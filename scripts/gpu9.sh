# 2 GPUs: full gpu test suite, C2 convex bench, C2 default bench
mkdir -p gpurun_out/r9
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r9/smoke.log 2>&1; echo smoke=$? >> gpurun_out/r9/status.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r9/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/r9/status.txt
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --grad convex --no-e2e > gpurun_out/r9/c2_convex_n1.json 2>gpurun_out/r9/c2_convex.err; echo convex=$? >> gpurun_out/r9/status.txt
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py > gpurun_out/r9/c2_n1.json 2>/dev/null; echo bench=$? >> gpurun_out/r9/status.txt
