mkdir -p gpurun_out/r20
for w in 1 4 8; do timeout 300 python scripts/shard_probe.py --config C4 --world $w --steps 30 >> gpurun_out/r20/c4_probe.jsonl 2>>gpurun_out/r20/err.log; done
