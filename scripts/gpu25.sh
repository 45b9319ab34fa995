mkdir -p gpurun_out/r26
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "update_frequency or full_size" > gpurun_out/r26/pytest.log 2>&1; echo pytest=$? >> gpurun_out/r26/status.txt
timeout 300 python bench.py --update-freq 2 --no-e2e --no-cpu-baseline > gpurun_out/r26/c2_f2.json 2>/dev/null
