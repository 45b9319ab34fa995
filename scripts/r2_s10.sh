D=gpurun_out/r2_s10; mkdir -p $D
st() { echo "$1=$2" >> "$D/status.txt"; }
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
NOX="--no-e2e --no-cpu-baseline --no-extras"
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_colocated.py -q -m gpu -k "stress" > $D/stress_p2p.log 2>&1; st stress_p2p $?
CUDA_VISIBLE_DEVICES=0 HP_P2P=0 timeout 600 python -m pytest tests/test_gpu_colocated.py -q -m gpu -k "stress" > $D/stress_bar.log 2>&1; st stress_bar $?
P=29950
run() { P=$((P+1)); name=$1; shift; env $ENVV timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 "$@" > "$D/$name.json" 2>> "$D/err.log"; st "$name" $?; }
for cfg in "C3" "C5E --span 1 --transport nvls"; do
  n=$(echo $cfg | cut -d' ' -f1)
  ENVV="X=0" run ${n}_base --config $cfg $NOX --steps 100
  ENVV="HP_SPLIT_FOLDS=1" run ${n}_split --config $cfg $NOX --steps 100 --timeline $D/tl_${n}_split
  ENVV="HP_SPLIT_FOLDS=1 HP_XBLOCKS=64" run ${n}_split_x64 --config $cfg $NOX --steps 100 --timeline $D/tl_${n}_split_x64
  ENVV="HP_SPLIT_FOLDS=1 HP_XBLOCKS=96" run ${n}_split_x96 --config $cfg $NOX --steps 100
  ENVV="HP_SPLIT_FOLDS=1 HP_XBLOCKS=64 HP_ABLOCKS=232" run ${n}_split_x64_a232 --config $cfg $NOX --steps 100
  ENVV="HP_SPLIT_FOLDS=1 HP_XBLOCKS=64 HP_AGRID=1" run ${n}_split_x64_agrid --config $cfg $NOX --steps 100
  ENVV="HP_SPLIT_FOLDS=1 HP_XBLOCKS=32" run ${n}_split_x32 --config $cfg $NOX --steps 100
done
ENVV="X=0" run c5_base --config C5 --span 1 $NOX --steps 20
ENVV="HP_SPLIT_FOLDS=1 HP_XBLOCKS=96" run c5_split_x96 --config C5 --span 1 $NOX --steps 20
