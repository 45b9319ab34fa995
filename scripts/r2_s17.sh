D=gpurun_out/r2_s17; mkdir -p $D
st() { echo "$1=$2" >> "$D/status.txt"; }
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
NOX="--no-e2e --no-cpu-baseline --no-extras"
P=30200
run() { P=$((P+1)); n=$1; g=$2; shift; shift; env $ENVV timeout 1200 $TR --nproc-per-node $g --master-port $P bench.py --gpus $g "$@" > "$D/$n.json" 2>> "$D/err.log"; st "$n" $?; }
ENVV="X=0" run c3 4 --config C3 $NOX --steps 300
ENVV="HP_APPLY_U=2" run c3_applyu2 4 --config C3 $NOX --steps 300 --timeline $D/tl_c3_applyu2
ENVV="HP_APPLY_U=2 HP_XBLOCKS=128" run c3_applyu2_x128 4 --config C3 $NOX --steps 300
ENVV="X=0" run c5 4 --config C5 --span 1 $NOX --steps 30
ENVV="HP_APPLY_U=2" run c5_applyu2 4 --config C5 --span 1 $NOX --steps 30
ENVV="X=0" run c5_D4 4 --config C5 --span 1 --D 4 $NOX --steps 30
ENVV="X=0" run c5_D4_R3 4 --config C5 --span 1 --D 4 --acc-slots 3 $NOX --steps 30
ENVV="X=0" run c5_D32 4 --config C5 --span 1 --D 32 $NOX --steps 30
ENVV="X=0" run c5_D32_R4 4 --config C5 --span 1 --D 32 --acc-slots 4 $NOX --steps 30
ENVV="HP_APPLY_U=2" run c5e_peer_applyu2 4 --config C5E --span 1 $NOX --steps 30
ENVV="X=0" run c5e_peer 4 --config C5E --span 1 $NOX --steps 30
for s in 11 12 13; do HP_STRESS=$s HP_MULTI_RANDOM=8 timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu > $D/multi_stress_$s.log 2>&1; st multi_stress_$s $?; done
