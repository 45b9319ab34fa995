#!/usr/bin/env bash
# One parameterised driver for the measurement sessions on a B200 box (it
# replaces round 1's one-off scripts/gpuN.sh files, kept in git history at
# b751f1a). Run from the repo root, e.g.
#   gpurun --timeout 1800 -- 'bash scripts/session.sh validate r02_final'
#   gpurun --gpus 4 --timeout 2400 -- 'bash scripts/session.sh multi r02_g4'
# Every job writes under gpurun_out/<tag>/ and appends "<step>=<rc>" to its
# status.txt; the files worth keeping are copied into profiles/ by hand.
#
# jobs:
#   validate  smoke, pytest -m gpu, bench N=1 (C2) + reference arm, C1 line
#   ncu       ncu launch list of the N=1 bench + one --set full tick-kernel capture
#   ncu_c1    --set full capture of the C1 tick kernels (latency-bound launches)
#   single    single-GPU workloads: C3 / C4 / C5 on one GPU, F=2, CONVEX, PMP timing
#   multi     every visible GPU (N >= 2): nvlink peak, default bench (C3 placement),
#             C2 ED-local, C4 ED-local, C5 (one VW per GPU), C5E / HVD transports,
#             multi-GPU parity
#   overlap   a9 overlap variants (split folds, bounded grids) with per-launch timelines
#   knobs     GPU parity under the non-default tuning knobs (1 GPU)
#   cosched   C3 exchange / completes SM co-scheduling knobs with timelines, N >= 2
#   splitdef  split acc / fold default A/B + multi-GPU parity, N >= 2
#   accov     HP_ACC_OVERLAP A/B (completes-only launches under the exchange), N >= 2
set -u
JOB=${1:?job}
TAG=${2:-$JOB}
D=gpurun_out/$TAG
mkdir -p "$D"
st() { echo "$1=$2" >> "$D/status.txt"; }
NG=$(python -c "import torch; print(torch.cuda.device_count())")
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
NOX="--no-e2e --no-cpu-baseline"

case "$JOB" in
validate)
  python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$D/smoke.log" 2>&1; st smoke $?
  timeout 1500 python -m pytest tests -m gpu -q > "$D/pytest_gpu.log" 2>&1; st pytest $?
  CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > "$D/bench_n1.json" 2> "$D/bench_n1.err"; st bench1 $?
  CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference > "$D/ref_n1.json" 2>/dev/null; st ref $?
  CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --config C1 --no-cpu-baseline > "$D/bench_c1.json" 2> "$D/bench_c1.err"; st c1 $?
  ;;
ncu)
  CMD="python bench.py --steps 3 --warmup 3 $NOX --profile-steps 1"
  CUDA_VISIBLE_DEVICES=0 $CMD > "$D/plain.log" 2>&1; st plain $?
  CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$D/launches.csv" $CMD > "$D/ncu_list.log" 2>&1; st ncu_list $?
  CUDA_VISIBLE_DEVICES=0 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tick_kernel \
    -s 18 -c 6 -o "$D/tick_full" $CMD > "$D/ncu_full.log" 2>&1; st ncu_full $?
  ;;
ncu_c1)
  CMD="python bench.py --config C1 --steps 40 --warmup 5 $NOX --graph 0 --profile-steps 1"
  CUDA_VISIBLE_DEVICES=0 $CMD > "$D/plain.log" 2>&1; st plain $?
  CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tick \
    -s 60 -c 3 -o "$D/c1_full" $CMD > "$D/ncu_full.log" 2>&1; st ncu_full $?
  ;;
single)
  for c in C3 C4 C5; do
    CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --config $c --steps 40 $NOX > "$D/bench_${c}_n1.json" 2>> "$D/err.log"; st "$c" $?
  done
  CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --update-freq 2 --steps 40 $NOX > "$D/bench_c2_f2.json" 2>> "$D/err.log"; st f2 $?
  CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --grad convex --steps 40 $NOX > "$D/bench_c2_convex.json" 2>> "$D/err.log"; st convex $?
  CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --timing pmp --steps 40 $NOX > "$D/bench_c2_pmp.json" 2>> "$D/err.log"; st pmp $?
  ;;
multi)
  [ "$NG" -ge 2 ] || { st multi_needs_2_gpus 1; exit 0; }
  timeout 600 python scripts/nvlink_peak.py --out "$D/nvlink_peak.json" > "$D/nvlink_peak.log" 2>&1; st nvlink_peak $?
  P=29760
  run() { P=$((P+1)); name=$1; shift; timeout 1200 $TR --nproc-per-node "$NG" --master-port $P bench.py --gpus "$NG" "$@" > "$D/$name.json" 2>> "$D/err.log"; st "$name" $?; }
  run bench_default
  run c2_edlocal --config C2 --span 0 $NOX --steps 100
  run c4_edlocal --config C4 --span 0 $NOX --steps 60
  run c3_k1 --config C3 --span 1 $NOX --steps 40
  run c5 --config C5 --span 1 $NOX --steps 20
  run c5e_nvls --config C5E --span 1 --transport nvls $NOX --steps 20
  run c5e_nccl --config C5E --span 1 --transport nccl $NOX --steps 20
  run hvd_nvls --config HVD --span 1 --transport nvls $NOX --steps 40
  timeout 1500 python -m pytest tests/test_gpu_multi.py -q > "$D/pytest_multi.log" 2>&1; st multi_parity $?
  ;;
overlap)
  # a9 overlap experiments on every visible GPU: C3 (default placement) and
  # C5E (NVLS) with split acc / fold launches and bounded grids; per-launch
  # timelines of every rank (bench.py --timeline)
  [ "$NG" -ge 2 ] || { st overlap_needs_2_gpus 1; exit 0; }
  P=29800
  for cfg in "C3" "C5E --transport nvls"; do
    name=$(echo "$cfg" | cut -d' ' -f1)
    for env in "X=0" "HP_SPLIT_FOLDS=1" "HP_XBLOCKS=80 HP_ABLOCKS=216" "HP_SPLIT_FOLDS=1 HP_XBLOCKS=48 HP_ABLOCKS=240" "HP_SPLIT_FOLDS=1 HP_XBLOCKS=80 HP_ABLOCKS=216"; do
      P=$((P+1)); tag=$(echo "$env" | tr ' =' '__')
      env $env timeout 900 $TR --nproc-per-node "$NG" --master-port $P bench.py --gpus "$NG" --config $cfg --span 1 \
        $NOX --steps 30 --profile-steps 6 --no-extras --timeline "$D/tl_${name}_${tag}" > "$D/${name}_${tag}.json" 2>> "$D/err.log"
      st "${name}_${tag}" $?
    done
  done
  ;;
accov)
  # a9: completes-only launches under the exchange (HP_ACC_OVERLAP) A/B on
  # every visible GPU, alternating, plus timelines of the default
  [ "$NG" -ge 2 ] || { st accov_needs_2_gpus 1; exit 0; }
  P=29900
  for cfg in "C3" "C5E --transport nvls" "C5" "C3 --span 2" "C3"; do
    name=$(echo "$cfg" | tr -d ' -')
    for ov in 1 0; do
      P=$((P+1))
      HP_ACC_OVERLAP=$ov timeout 900 $TR --nproc-per-node "$NG" --master-port $P bench.py --gpus "$NG" --config $cfg \
        $NOX --steps 100 --no-extras > "$D/${name}_ov${ov}_$P.json" 2>> "$D/err.log"
      st "${name}_ov${ov}_$P" $?
    done
  done
  P=$((P+1))
  timeout 900 $TR --nproc-per-node "$NG" --master-port $P bench.py --gpus "$NG" $NOX --steps 30 --profile-steps 6 \
    --no-extras --timeline "$D/tl_c3" > "$D/c3_timeline.json" 2>> "$D/err.log"; st tl $?
  CUDA_VISIBLE_DEVICES=0 timeout 1200 python -m pytest tests/test_gpu_colocated.py -q -m gpu > "$D/colocated.log" 2>&1; st colocated $?
  timeout 1500 python -m pytest tests/test_gpu_multi.py -q > "$D/pytest_multi.log" 2>&1; st multi_parity $?
  ;;
cosched)
  # C3 at N GPUs: SM co-scheduling of the owners' exchange with the VW's own
  # completes (grid bounds, non-persistent completes, priorities), timelines;
  # COSCHED_ENVS overrides the list (one entry per variant, '+' joins variables)
  [ "$NG" -ge 2 ] || { st cosched_needs_2_gpus 1; exit 0; }
  P=29950
  for env in ${COSCHED_ENVS:-"X=0" "HP_ABLOCKS=296" "HP_ABLOCKS=148" "HP_AGRID=1" "HP_XBLOCKS=256" "HP_PRIO=0" "X=0"}; do
    P=$((P+1)); tag=$(echo "$env" | tr ' =+@' '____')
    # BENCH_ARGS: a leading '@args@' token of an entry ('@--acc-slots+3@HP_X=1')
    # passes bench arguments ('+' = space)
    bargs=""
    case "$env" in @*@*) bargs=$(echo "$env" | cut -d@ -f2 | tr '+' ' '); env=$(echo "$env" | cut -d@ -f3);; esac
    env $(echo "$env" | tr '+' ' ') timeout 900 $TR --nproc-per-node "$NG" --master-port $P bench.py --gpus "$NG" $NOX --steps 100 \
      --no-extras $bargs --timeline "$D/tl_${tag}_$P" > "$D/c3_${tag}_$P.json" 2>> "$D/err.log"
    st "c3_${tag}_$P" $?
  done
  ;;
splitdef)
  # the split acc / fold default (one VW stage per GPU, SGD, peer): A/B
  # against HP_SPLIT_FOLDS=0, the other one-stage placements, multi-GPU parity
  [ "$NG" -ge 2 ] || { st splitdef_needs_2_gpus 1; exit 0; }
  P=30100
  run() { P=$((P+1)); ev=$1; name=$2; shift 2; env $ev timeout 900 $TR --nproc-per-node "$NG" --master-port $P bench.py --gpus "$NG" "$@" > "$D/$name.json" 2>> "$D/err.log"; st "$name" $?; }
  run X=0 c3_default $NOX --steps 300
  run HP_SPLIT_FOLDS=0 c3_fused $NOX --steps 300
  run X=0 c3_default2 $NOX --steps 300
  run X=0 c5e_peer --config C5E --span 1 --transport peer $NOX --steps 40
  run HP_SPLIT_FOLDS=0 c5e_peer_fused --config C5E --span 1 --transport peer $NOX --steps 40
  run X=0 hvd_peer --config HVD --span 1 --transport peer $NOX --steps 40
  run HP_SPLIT_FOLDS=0 hvd_peer_fused --config HVD --span 1 --transport peer $NOX --steps 40
  run X=0 c5e_nvls --config C5E --span 1 --transport nvls $NOX --steps 40
  timeout 1500 python -m pytest tests/test_gpu_multi.py -q > "$D/pytest_multi.log" 2>&1; st multi_parity $?
  CUDA_VISIBLE_DEVICES=0 timeout 1200 python -m pytest tests/test_gpu_colocated.py -q -m gpu > "$D/colocated.log" 2>&1; st colocated $?
  ;;
knobs)
  for kv in "HP_TICK_U=1" "HP_GRID=1" "HP_PDL=0" "HP_DYN=0" "HP_PREFETCH=0" "HP_DYN_MIN_N=0" \
            "HP_LEAN=0" "HP_APPLY_U=2" "HP_TICK_BATCH=0"; do
    env $kv timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -q -m gpu > "$D/parity_${kv}.log" 2>&1; st "$kv" $?
  done
  for kv in "HP_P2P=0" "HP_AGRID=1" "HP_APPLY_U=2 HP_XBLOCKS=128" "HP_SPLIT_FOLDS=1 HP_XBLOCKS=96"; do
    tag=$(echo "$kv" | tr ' =' '__')
    env $kv timeout 900 python -m pytest tests/test_gpu_colocated.py -q -m gpu > "$D/colocated_${tag}.log" 2>&1; st "colocated_$tag" $?
  done
  ;;
*)
  echo "unknown job $JOB" >&2; exit 2 ;;
esac
