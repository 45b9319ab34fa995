# 4 GPUs: overlap sweep (split folds x grid mode x exchange bound x priorities)
mkdir -p gpurun_out/sweep3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for v in "1 1 0 1" "1 1 148 1" "1 1 296 1" "1 0 148 1" "1 1 148 0" "0 0 0 1" "0 1 0 1"; do set -- $v
  for c in "C3 peer" "C5E nvls" "C5E peer"; do set -- $v $c
    HP_SPLIT_FOLDS=$1 HP_GRID=$2 HP_XBLOCKS=$3 HP_PRIO=$4 timeout 300 $TR --master-port 29552 bench.py --gpus 4 --config $5 --span 1 --transport $6 --steps 10 --no-e2e > gpurun_out/sweep3/${5}_${6}_sf$1_g$2_xb$3_p$4.json 2>/dev/null
  done
done
echo done > gpurun_out/status7.txt
