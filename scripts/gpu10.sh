# 1 GPU: full gpu suite (single-GPU parts), F and convex benches
mkdir -p gpurun_out/r10
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r10/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/r10/status.txt
timeout 300 python bench.py --update-freq 2 --no-e2e --no-cpu-baseline > gpurun_out/r10/c2_f2.json 2>/dev/null; echo f2=$? >> gpurun_out/r10/status.txt
timeout 300 python bench.py --update-freq 2 --grad convex --no-e2e --no-cpu-baseline > gpurun_out/r10/c2_f2_convex.json 2>/dev/null
