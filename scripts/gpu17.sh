mkdir -p gpurun_out/r18
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r18/plain.log 2>&1 && \
timeout 900 compute-sanitizer --tool memcheck --leak-check no python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r18/memcheck.log 2>&1
echo rc=$? > gpurun_out/r18/status.txt
