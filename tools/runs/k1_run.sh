timeout 600 python -m pytest tests/test_preprocess_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/k1_tests.log 2>&1; echo "tests $?" >> gpurun_out/k1_tests.log
for r in 1 2; do for c in 2 4; do echo "c$c: $(PROF_TIME=1 timeout 120 python tools/prof_run.py 1048576 0 $c 2>&1 | tail -1)"; done; done > gpurun_out/k1_time.log 2>&1
