# 1 GPU: ncu launch list + one --set full capture of the tick kernel (C2, FLOAT)
mkdir -p gpurun_out/r11
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --profile-steps 1"
$CMD > gpurun_out/r11/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r11/launches.csv $CMD > gpurun_out/r11/ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tick_kernel -s 18 -c 6 -o gpurun_out/r11/prof $CMD > gpurun_out/r11/ncu_full.log 2>&1
echo rc=$? > gpurun_out/r11/status.txt
