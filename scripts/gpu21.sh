mkdir -p gpurun_out/r22
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for v in "0 0" "80 216" "120 180" "60 236" "148 148" "40 256"; do set -- $v
  HP_XBLOCKS=$1 HP_ABLOCKS=$2 timeout 300 $TR --master-port 29661 bench.py --gpus 4 --config C3 --span 1 --steps 20 --no-e2e > gpurun_out/r22/c3_x$1_a$2.json 2>/dev/null
  HP_XBLOCKS=$1 HP_ABLOCKS=$2 timeout 300 $TR --master-port 29662 bench.py --gpus 4 --config C5 --span 1 --steps 10 --no-e2e > gpurun_out/r22/c5_x$1_a$2.json 2>/dev/null
done
