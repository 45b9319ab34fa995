# parity of the CUDA path under the non-default tuning knobs
mkdir -p gpurun_out/r34
for v in "HP_TICK_U=1" "HP_TICK_U=8" "HP_GRID=1" "HP_PDL=0"; do
  env $v timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "random_configs or convex_random or update_frequency_random or full_size" > gpurun_out/r34/$v.log 2>&1; echo "$v=$?" >> gpurun_out/r34/status.txt
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
HP_XBLOCKS=80 HP_ABLOCKS=216 HP_SPLIT_FOLDS=1 HP_MULTI_RANDOM=8 timeout 900 $TR --master-port 29761 tests/gpu_multi_parity.py > gpurun_out/r34/multi_knobs.log 2>&1; echo multi=$? >> gpurun_out/r34/status.txt
timeout 300 $TR --master-port 29762 bench.py --gpus 4 --no-e2e --steps 50 > gpurun_out/r34/bench_n4.json 2>/dev/null; echo bench=$? >> gpurun_out/r34/status.txt
