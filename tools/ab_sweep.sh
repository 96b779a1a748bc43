# A/B of library variants inside the power-capped config-2 sweep (bench.py, device-resident, 20 steps)
mkdir -p gpurun_out/s6
for v in "$@"; do
  if [ "$v" = base ]; then unset DETNET_LIB; else export DETNET_LIB=build/$v/libdetnet_b200.so; fi
  timeout 300 python bench.py --config 2 --only --no-cpu --no-e2e --no-parity 2>/dev/null | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step'],2), 'ms/step  stack', round(d['roofline']['avg_launch_ms'],3), 'ms', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
