#!/bin/bash
# Round profile capture on one B200 (run under gpurun from the repo root).
# Each ncu pass runs only after the same command has exited 0 without ncu.
# Outputs land in gpurun_out/prof/; tools/summarize_profiles.py turns them
# into the text summaries committed under profiles/.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
# 1. benches (no profiler): the default run (config 2 + nested configs 1, 3, 4, 5),
#    then each config alone
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for c in 1 2 3 4 5; do
  timeout 600 python bench.py --config $c --only > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err
done
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
# 2. launch list of the default bench command (per-launch durations, cold, serialised)
if timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $OUT/plain.json 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $OUT/ncu_launch.log 2>&1
fi
# 2b. launch list of one training step (config 5)
if timeout 600 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu > $OUT/plain_c5.json 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file $OUT/launches_c5.csv python bench.py --config 5 --steps 1 --warmup 3 --no-cpu > $OUT/ncu_launch_c5.log 2>&1
fi
# 3. one full capture per hot kernel (2^18 detections, config-2 workload):
#    the split-FP16 stack (default), K1, and the 3xTF32 stack (path 2) for comparison
if timeout 300 python tools/prof_run.py 262144 > $OUT/prof_run.log 2>&1; then
  for k in k_stack_h16 k_prep_stream; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o $OUT/$k python tools/prof_run.py 262144 > $OUT/ncu_$k.log 2>&1
  done
fi
if timeout 300 python tools/prof_run.py 262144 2 > $OUT/prof_run_tf32.log 2>&1; then
  timeout 900 ncu --set full --clock-control none -k regex:k_stack_tc -s 1 -c 1 \
    -o $OUT/k_stack_tc python tools/prof_run.py 262144 2 > $OUT/ncu_k_stack_tc.log 2>&1
fi
# 4. the compacted (config-3) stack kernel
if timeout 300 python tools/prof_run.py 262144 0 3 > $OUT/prof_run3.log 2>&1; then
  timeout 900 ncu --set full --clock-control none -k regex:k_stack_h16 -s 1 -c 1 \
    -o $OUT/k_stack_h16_64 python tools/prof_run.py 262144 0 3 > $OUT/ncu_h16_64.log 2>&1
fi
# 5. the model-specialised sparse kernel (config 4, JIT-compiled at model creation)
if timeout 300 python tools/prof_run.py 262144 0 4 > $OUT/prof_run4.log 2>&1; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:detnet_sparse_jit -s 1 -c 1 \
    -o $OUT/detnet_sparse_jit python tools/prof_run.py 262144 0 4 > $OUT/ncu_jit.log 2>&1
fi
# 6. SURVEY 8f measurements: ZF/ML baselines, pruning planner, incremental trainer
timeout 900 python tools/bench_baselines.py > $OUT/baselines.json 2> $OUT/baselines.err
timeout 900 python tools/bench_prune.py > $OUT/prune.json 2> $OUT/prune.err
timeout 1200 python tools/bench_incremental.py > $OUT/incremental.json 2> $OUT/incremental.err
echo done
