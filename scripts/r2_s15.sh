D=gpurun_out/r2_s15; mkdir -p $D
st() { echo "$1=$2" >> "$D/status.txt"; }
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
NOX="--no-e2e --no-cpu-baseline --no-extras"
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_colocated.py tests/test_gpu_graph.py -q -m gpu -s > $D/colocated.log 2>&1; st colocated $?
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu > $D/multi.log 2>&1; st multi $?
timeout 600 python scripts/nvlink_peak.py --out $D/nvlink_peak.json > $D/nvlink_peak.log 2>&1; st nvpeak $?
P=30100
run() { P=$((P+1)); n=$1; g=$2; shift; shift; env $ENVV timeout 1200 $TR --nproc-per-node $g --master-port $P bench.py --gpus $g "$@" > "$D/$n.json" 2>> "$D/err.log"; st "$n" $?; }
ENVV="X=0" run default_g4 4
ENVV="X=0" CUDA_VISIBLE_DEVICES=0,1 run default_g2 2
ENVV="X=0" run c3_base 4 --config C3 $NOX --steps 300
ENVV="HP_SPLIT_FOLDS=1 HP_XBLOCKS=96" run c3_split_x96 4 --config C3 $NOX --steps 300
ENVV="HP_SPLIT_FOLDS=1 HP_XBLOCKS=80" run c3_split_x80 4 --config C3 $NOX --steps 300
ENVV="HP_SPLIT_FOLDS=1 HP_XBLOCKS=128" run c3_split_x128 4 --config C3 $NOX --steps 300
ENVV="X=0" run c3_nvls 4 --config C3 --transport nvls $NOX --steps 300
ENVV="HP_SPLIT_FOLDS=1 HP_XBLOCKS=96" run c3_nvls_split_x96 4 --config C3 --transport nvls $NOX --steps 300
ENVV="X=0" run c3k2 4 --config C3 --span 2 $NOX --steps 300
ENVV="X=0" run c4_edlocal 4 --config C4 --span 0 $NOX --steps 60
ENVV="X=0" run c5 4 --config C5 --span 1 $NOX --steps 30
ENVV="X=0" run c5e_nvls 4 --config C5E --span 1 --transport nvls $NOX --steps 30
ENVV="X=0" run hvd_nvls 4 --config HVD --span 1 --transport nvls $NOX --steps 60
ENVV="HP_STRESS=7" run c3_stress_parityrun 4 --config C3 $NOX --steps 20
