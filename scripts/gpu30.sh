mkdir -p gpurun_out/r31
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for v in "0 216" "80 216" "80 0" "0 0"; do set -- $v
  for c in C3 C5; do
    HP_XBLOCKS=$1 HP_ABLOCKS=$2 timeout 300 $TR --master-port 29721 bench.py --gpus 4 --config $c --span 1 --steps 20 --no-e2e > gpurun_out/r31/${c}_x$1_a$2.json 2>/dev/null
  done
  HP_XBLOCKS=$1 HP_ABLOCKS=$2 timeout 300 $TR --master-port 29722 bench.py --gpus 4 --config C5E --span 1 --transport peer --steps 10 --no-e2e > gpurun_out/r31/C5E_x$1_a$2.json 2>/dev/null
  HP_XBLOCKS=$1 HP_ABLOCKS=$2 timeout 300 $TR --master-port 29723 bench.py --gpus 4 --config C3 --span 2 --steps 20 --no-e2e > gpurun_out/r31/C3k2_x$1_a$2.json 2>/dev/null
done
