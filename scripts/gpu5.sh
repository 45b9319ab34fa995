# 4 GPUs: parity with split folds, then sweep split x exchange grid bound
mkdir -p gpurun_out/sweep2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29551 tests/gpu_multi_parity.py > gpurun_out/multi_parity_g4_split2.log 2>&1; echo parity=$? >> gpurun_out/status6.txt
for sf in 1 0; do for xb in 0 148; do
  for c in "C3 peer" "C5E nvls" "C5E peer"; do set -- $c
    HP_SPLIT_FOLDS=$sf HP_XBLOCKS=$xb timeout 300 $TR --master-port 29552 bench.py --gpus 4 --config $1 --span 1 --transport $2 --steps 10 --no-e2e > gpurun_out/sweep2/${1}_${2}_sf${sf}_xb${xb}.json 2>/dev/null
  done
done; done
echo done >> gpurun_out/status6.txt
