for n in 4096 37888 151552 1048576; do echo "n=$n: $(DETNET_H16_2T=1 timeout 120 python tools/prof_run.py $n 0 2 2>&1 | tail -1)"; done > gpurun_out/t2_dbg2.log 2>&1
for c in 2 3; do for v in 0 1; do echo "2T=$v c$c: $(DETNET_H16_2T=$v PROF_TIME=1 timeout 120 python tools/prof_run.py 1048576 0 $c 2>&1 | tail -2 | tr '\n' ' ')"; done; done > gpurun_out/t2_time.log 2>&1
