D=gpurun_out/r2_s9; mkdir -p $D
st() { echo "$1=$2" >> "$D/status.txt"; }
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
NOX="--no-e2e --no-cpu-baseline --no-extras"
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_colocated.py -q -m gpu > $D/colocated.log 2>&1; st colocated $?
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu > $D/multi.log 2>&1; st multi $?
timeout 600 python scripts/nvlink_peak.py --out $D/nvlink_peak.json > $D/nvlink_peak.log 2>&1; st nvpeak $?
P=29900
run() { P=$((P+1)); name=$1; shift; env $ENVV timeout 900 $TR --nproc-per-node 4 --master-port $P bench.py --gpus 4 "$@" > "$D/$name.json" 2>> "$D/err.log"; st "$name" $?; }
ENVV="X=0" run c3_p2p --config C3 $NOX --steps 200 --timeline $D/tl_c3_p2p
ENVV="HP_P2P=0" run c3_bar --config C3 $NOX --steps 200
ENVV="HP_AGRID=1" run c3_p2p_agrid --config C3 $NOX --steps 200 --timeline $D/tl_c3_agrid
ENVV="HP_XBLOCKS=80" run c3_p2p_x80 --config C3 $NOX --steps 200
ENVV="HP_AGRID=1 HP_XBLOCKS=80" run c3_p2p_agrid_x80 --config C3 $NOX --steps 200
ENVV="X=0" run c3k2_p2p --config C3 --span 2 $NOX --steps 200
ENVV="HP_P2P=0" run c3k2_bar --config C3 --span 2 $NOX --steps 200
ENVV="X=0" run c5_p2p --config C5 --span 1 $NOX --steps 30
ENVV="HP_P2P=0" run c5_bar --config C5 --span 1 $NOX --steps 30
ENVV="HP_AGRID=1" run c5_p2p_agrid --config C5 --span 1 $NOX --steps 30
ENVV="X=0" run c5e_nvls --config C5E --span 1 --transport nvls $NOX --steps 30
ENVV="HP_AGRID=1" run c5e_nvls_agrid --config C5E --span 1 --transport nvls $NOX --steps 30
# single GPU A/B: momentum o4 3 vs 4 CTAs (HP_LIB), lean instance on/off
for lib in libhetpipe.so libhetpipe_ab.so; do
  CUDA_VISIBLE_DEVICES=0 HP_LIB=$PWD/paper_2005_14038_b200/$lib timeout 600 python bench.py --config C5 --steps 20 --no-e2e --no-cpu-baseline > $D/c5_1gpu_$lib.json 2>> $D/err.log; st c5_1gpu_$lib $?
done
for lean in 1 0; do
  CUDA_VISIBLE_DEVICES=0 HP_LEAN=$lean timeout 600 python bench.py --steps 100 --no-e2e --no-cpu-baseline > $D/c2_lean$lean.json 2>> $D/err.log; st c2_lean$lean $?
done
