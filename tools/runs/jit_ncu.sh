python tools/prof_run.py 262144 0 4 > gpurun_out/jit_pre.log 2>&1 && \
timeout 600 ncu --set full --clock-control none -k regex:detnet_sparse_jit -s 1 -c 1 -o gpurun_out/jit_k4j python tools/prof_run.py 262144 0 4 > gpurun_out/jit_ncu.log 2>&1
echo rc $?
