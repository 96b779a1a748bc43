timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_invariants_gpu.py -x -q -k "sparse or masked or invariant" > gpurun_out/jit_tests.log 2>&1; echo "tests $?" >> gpurun_out/jit_tests.log
for g in 64 96; do DETNET_JIT_GREG=$g PROF_TIME=1 timeout 300 python tools/prof_run.py 1048576 0 4 > gpurun_out/jit_prof_g$g.log 2>&1; done
echo done
