# final validation (prefetch, dynamic tiles incl. NVLS, apply triples): smoke, GPU suite (multi at 4), benches (1/2/4 GPUs, placements), ncu
D=gpurun_out/r54; mkdir -p $D
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $D/smoke.log 2>&1; echo smoke=$? >> $D/status.txt
timeout 1500 python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1; echo pytest=$? >> $D/status.txt
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $D/bench_n1.json 2> $D/bench_n1.err; echo bench1=$? >> $D/status.txt
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference > $D/ref_n1.json 2>/dev/null; echo ref=$? >> $D/status.txt
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 2 --master-port 29751 bench.py --gpus 2 > $D/bench_n2.json 2>/dev/null; echo bench2=$? >> $D/status.txt
timeout 900 $TR --nproc-per-node 4 --master-port 29752 bench.py --gpus 4 > $D/bench_n4.json 2>/dev/null; echo bench4=$? >> $D/status.txt
timeout 900 $TR --nproc-per-node 4 --master-port 29753 bench.py --gpus 4 --config C4 --no-e2e --no-cpu-baseline --steps 100 > $D/c4_n4.json 2>/dev/null; echo c4=$? >> $D/status.txt
timeout 900 $TR --nproc-per-node 4 --master-port 29754 bench.py --gpus 4 --config C3 --span 1 --no-e2e --no-cpu-baseline --steps 40 > $D/c3_k1_n4.json 2>/dev/null; echo c3k1=$? >> $D/status.txt
timeout 900 $TR --nproc-per-node 4 --master-port 29755 bench.py --gpus 4 --config C3 --span 2 --no-e2e --no-cpu-baseline --steps 40 > $D/c3_k2_n4.json 2>/dev/null; echo c3k2=$? >> $D/status.txt
timeout 900 $TR --nproc-per-node 4 --master-port 29756 bench.py --gpus 4 --config C5 --span 1 --no-e2e --no-cpu-baseline --steps 40 > $D/c5_n4.json 2>/dev/null; echo c5=$? >> $D/status.txt
timeout 900 $TR --nproc-per-node 4 --master-port 29757 bench.py --gpus 4 --config C5E --span 1 --transport nvls --no-e2e --no-cpu-baseline --steps 40 > $D/c5e_nvls_n4.json 2>/dev/null; echo c5e=$? >> $D/status.txt
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > $D/ncu_list.log 2>&1; echo ncu_list=$? >> $D/status.txt
