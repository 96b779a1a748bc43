export DETNET_JIT_CACHE=off
for sc in 0 1; do for g in 16 64; do echo "scout=$sc greg=$g: $(DETNET_JIT_SCOUT=$sc DETNET_JIT_GREG=$g PROF_TIME=1 timeout 200 python tools/prof_run.py 1048576 0 4 2>&1 | tail -2 | tr '\n' ' ')"; done; done
