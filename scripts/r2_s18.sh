D=gpurun_out/r2_s18; mkdir -p $D
st() { echo "$1=$2" >> "$D/status.txt"; }
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
NOX="--no-e2e --no-cpu-baseline --no-extras"
nvidia-smi nvlink -h > $D/nvsmi_help.txt 2>&1
nvidia-smi nvlink -s -i 0 > $D/nvsmi_status.txt 2>&1
nvidia-smi nvlink -gt d -i 0 > $D/nvsmi_gt_before.txt 2>&1
nvidia-smi nvlink -e -i 0 > $D/nvsmi_e.txt 2>&1
P=30300
run() { P=$((P+1)); n=$1; g=$2; shift; shift; env $ENVV timeout 1200 $TR --nproc-per-node $g --master-port $P bench.py --gpus $g "$@" > "$D/$n.json" 2>> "$D/err.log"; st "$n" $?; }
for rep in 1 2; do
ENVV="X=0" run c3_base_$rep 4 --config C3 $NOX --steps 300
ENVV="HP_APPLY_U=2 HP_XBLOCKS=128" run c3_au2x128_$rep 4 --config C3 $NOX --steps 300
ENVV="HP_XBLOCKS=128" run c3_x128_$rep 4 --config C3 $NOX --steps 300
done
nvidia-smi nvlink -gt d -i 0 > $D/nvsmi_gt_after.txt 2>&1
ENVV="X=0" run c5_base 4 --config C5 --span 1 $NOX --steps 30
ENVV="HP_APPLY_U=2 HP_XBLOCKS=128" run c5_au2x128 4 --config C5 --span 1 $NOX --steps 30
ENVV="X=0" run c5e_nvls_base 4 --config C5E --span 1 --transport nvls $NOX --steps 30
ENVV="HP_XBLOCKS=128" run c5e_nvls_x128 4 --config C5E --span 1 --transport nvls $NOX --steps 30
ENVV="HP_APPLY_U=2 HP_XBLOCKS=128" run c3_g2_au2x128 2 --config C3 $NOX --steps 300
ENVV="X=0" run c3_g2_base 2 --config C3 $NOX --steps 300
