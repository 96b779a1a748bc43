mkdir -p gpurun_out/s6
DETNET_BENCH_SHARE_GPU=1 timeout 800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu > gpurun_out/s6/n2.json 2> gpurun_out/s6/n2.err
echo rc=$?
tail -c 600 gpurun_out/s6/n2.err
python - <<EOF
import json
d=json.loads(open("gpurun_out/s6/n2.json").read().strip().splitlines()[-1])
print(d["n_gpus"], d["value"], d["config"]["parallelism"], d.get("parity",{}).get("parity"))
for k,c in d["configs"].items(): print(k, c["value"], c.get("n_gpus"), c["config"].get("parallelism"))
EOF
