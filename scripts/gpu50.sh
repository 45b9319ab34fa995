# 1-GPU check of the final build: smoke, GPU suite (incl. knob parity), bench line
D=gpurun_out/r50; mkdir -p $D
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $D/smoke.log 2>&1; echo smoke=$? >> $D/status.txt
timeout 1500 python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1; echo "pytest=$? $(tail -1 $D/pytest_gpu.log)" >> $D/status.txt
timeout 900 python bench.py > $D/bench_n1.json 2> $D/bench_n1.err; echo bench1=$? >> $D/status.txt
