export DETNET_H16_2T=1
timeout 300 python tools/prof_run.py 4096 0 2 > gpurun_out/t2_small.log 2>&1; echo "small rc $?" >> gpurun_out/t2_small.log
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_invariants_gpu.py tests/test_h16_gpu.py -x -q > gpurun_out/t2_tests.log 2>&1; echo "tests $?" >> gpurun_out/t2_tests.log
unset DETNET_H16_2T
for c in 2 3; do for v in 0 1; do echo "2T=$v c$c: $(DETNET_H16_2T=$v PROF_TIME=1 timeout 120 python tools/prof_run.py 1048576 0 $c 2>&1 | tail -2 | tr '\n' ' ')"; done; done > gpurun_out/t2_time.log 2>&1
