"""SURVEY 8f row 4 measurement: ZF / ML detector baselines on the device
(detnet_batch_baseline_errors, host FP64 samples in, counts out -- the
transfer is inside the timing) vs the reference's batch_baseline_errors
(OpenMP, all host cores) on the same samples. One JSON line per case."""
import json
import os

# the in-process reference (OpenMP) must not spin its workers while the GPU
# side is timed on the same host cores (read when libgomp loads)
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2003_09446_b200 as eng  # noqa: E402
from oracle.oracle import Oracle, RefLib  # noqa: E402


def timed(f, reps):
    """Median of per-call wall times (a few ms each: a mean over 5 calls moved
    4x between runs on a busy host), after one warm-up call."""
    f()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = f()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return ts[len(ts) // 2], out


def main():
    orc, ref, ctx = Oracle(), RefLib(), eng.Context(0)
    cases = [("zf", 0, 20, 30, 1 << 16), ("ml", 1, 8, 16, 1 << 14), ("ml", 1, 12, 16, 1 << 11)]
    for name, kind, K, N, n in cases:
        H, x, y, _ = orc.generate_batch(orc.rng(3, 0), N, K, n, 0.0, 12.0)
        tg, (eg, sg) = timed(lambda: ctx.baseline_errors(kind, H, y, x), 21)
        tr, (st, er, sr) = timed(lambda: ref.baseline_errors(kind, H, y, x), 3)
        assert st == 0 and (eg, sg) == (er, sr), (eg, er)
        print(json.dumps({"baseline": name, "K": K, "N": N, "samples": n,
                          "b200_detections_per_s": n / tg, "reference_detections_per_s": n / tr,
                          "reference_cores": ref.worker_count(), "speedup": tr / tg,
                          "errors": eg, "symbols": sg, "identical_counts": True}))
        sys.stdout.flush()


if __name__ == "__main__":
    main()
