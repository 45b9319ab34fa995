D=gpurun_out/r2_s19; mkdir -p $D
st() { echo "$1=$2" >> "$D/status.txt"; }
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
NOX="--no-e2e --no-cpu-baseline --no-extras"
P=30400
run() { P=$((P+1)); n=$1; g=$2; shift; shift; env $ENVV timeout 1200 $TR --nproc-per-node $g --master-port $P bench.py --gpus $g "$@" > "$D/$n.json" 2>> "$D/err.log"; st "$n" $?; }
ENVV="X=0" run c3_auto 4 --config C3 $NOX --steps 300
ENVV="HP_XBLOCKS=0" run c3_full 4 --config C3 $NOX --steps 300
ENVV="X=0" run c3k2_auto 4 --config C3 --span 2 $NOX --steps 300
ENVV="HP_XBLOCKS=128" run c3k2_x128 4 --config C3 --span 2 $NOX --steps 300
ENVV="X=0" run c5e_peer_auto 4 --config C5E --span 1 $NOX --steps 30
ENVV="HP_XBLOCKS=0" run c5e_peer_full 4 --config C5E --span 1 $NOX --steps 30
ENVV="X=0" run hvd_peer_auto 4 --config HVD --span 1 $NOX --steps 60
ENVV="HP_XBLOCKS=0" run hvd_peer_full 4 --config HVD --span 1 $NOX --steps 60
ENVV="HP_XBLOCKS=128" run c3_g2_x128 2 --config C3 $NOX --steps 300
ENVV="X=0" run c3_g2_auto 2 --config C3 $NOX --steps 300
for v in 0 1; do CUDA_VISIBLE_DEVICES=0 HP_LEAN_DYN=$v timeout 600 python bench.py --steps 200 --no-e2e --no-cpu-baseline > $D/c2_leandyn$v.json 2>> $D/err.log; st c2_leandyn$v $?; done
CUDA_VISIBLE_DEVICES=0 bash scripts/session.sh knobs r2_knobs > /dev/null 2>&1; st knobs $?
