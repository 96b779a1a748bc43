#!/usr/bin/env python3
"""Config-5 training runs of the reference (O64) and of the FP32 restatement
(O32) from identical seeds (TEST INFRASTRUCTURE: runs the checkers only).

Shape: L=40, K=20, N=30, batch 5000, plain loss + group LASSO lambda1=1e-4
(the reference's column groups, kind sparse_group with lambda2=0), Adam lr0
1e-3, decay 0.97/1000, 100 steps; batches keyed like training.cpp:39,63-64
(train stream 2 of Rng(dseed), one generate_batch per step, H and y scaled by
1/sqrt(N) and rounded to FP32), validation set = 2000 samples of stream 3 at
12 dB. Weights: Xavier-uniform from Rng(pseed) (workload.xavier_params).

Writes
  tests/golden/train_ref_k20_l40.json : the reference's own trajectory per seed
      (per-step data loss and objective, final validation loss, sha256 of the
      final FP64 params) -- the FP64 GPU mode must reproduce it bit for bit;
  profiles/r2_train_spread.json : O32-vs-O64 final validation-loss spread --
      FP32's intrinsic distance from the FP64 reference after 100 steps, the
      calibration for the FP32 GPU default's bound.
"""
import argparse
import ctypes as C
import hashlib
import importlib.util
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import Model, Oracle, RefLib  # noqa: E402

K, N, Z, V = 20, 30, 160, 40


def workload():
    spec = importlib.util.spec_from_file_location(
        "detnet_workload", os.path.join(ROOT, "paper_2003_09446_b200", "workload.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def batches(orc, dseed, steps, batch):
    """Yields the FP32-rounded (as float64) training batches of one run."""
    train = orc.lib.or_stream(C.byref(orc.rng(dseed, 0)), 2)
    for _ in range(steps):
        H, x, y, _ = orc.generate_batch(train, N, K, batch, 7.0, 14.0)
        H = (H / np.sqrt(N)).astype(np.float32).astype(np.float64)
        y = (y / np.sqrt(N)).astype(np.float32).astype(np.float64)
        yield H, y, x


def val_set(orc, dseed, count=2000):
    val = orc.lib.or_stream(C.byref(orc.rng(dseed, 0)), 3)
    H, x, y, _ = orc.generate_batch(val, N, K, count, 12.0, 12.0)
    return ((H / np.sqrt(N)).astype(np.float32).astype(np.float64),
            (y / np.sqrt(N)).astype(np.float32).astype(np.float64), x)


def run(orc, ref, pseed, dseed, L, steps, batch, o32=True):
    params = workload().xavier_params(K, L, seed=pseed)
    m64 = Model(K, N, Z, V, L, params.copy())
    m32 = Model(K, N, Z, V, L, params.copy())
    mo = [np.zeros_like(params) for _ in range(4)]
    s64 = s32 = 0
    Hv, yv, xv = val_set(orc, dseed)
    out = {"pseed": pseed, "dseed": dseed, "layers": L, "steps": steps, "batch": batch,
           "val_loss_init": ref.batch_evaluate(m64, Hv, yv, xv)["data_loss"],
           "data_loss": [], "objective": [], "data_loss_o32": []}
    t0 = time.time()
    for H, y, x in batches(orc, dseed, steps, batch):
        g = ref.batch_gradient(m64, H, y, x, kind=2, lam1=1e-4)
        out["objective"].append(g["data_loss"] + ref.regularizer(m64, kind=2, lam1=1e-4))
        out["data_loss"].append(g["data_loss"])
        s64 = ref.adam_step(m64, g["grads"], mo[0], mo[1], s64, lr0=1e-3)
        if o32:
            g32 = orc.batch_gradient_f32(m32, H, y, x, kind=2, lam1=1e-4)
            out["data_loss_o32"].append(g32["data_loss"])
            s32 = orc.adam_step(m32, g32["grads"], mo[2], mo[3], s32, lr0=1e-3)
    out["val_loss_final"] = ref.batch_evaluate(m64, Hv, yv, xv)["data_loss"]
    out["params_sha256"] = hashlib.sha256(np.ascontiguousarray(m64.params).tobytes()).hexdigest()
    if o32:
        out["val_loss_final_o32"] = ref.batch_evaluate(m32, Hv, yv, xv)["data_loss"]
    out["seconds"] = time.time() - t0
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", default="9:1,9:2,10:1,11:3,12:4")
    ap.add_argument("--golden-seeds", type=int, default=3, help="first S seeds go to the golden")
    ap.add_argument("--layers", type=int, default=40)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--batch", type=int, default=5000)
    ap.add_argument("--golden", default=os.path.join(ROOT, "tests", "golden", "train_ref_k20_l40.json"))
    ap.add_argument("--spread", default=os.path.join(ROOT, "profiles", "r2_train_spread.json"))
    args = ap.parse_args()
    orc, ref = Oracle(), RefLib()
    runs = []
    for sp in args.seeds.split(","):
        p, d = (int(v) for v in sp.split(":"))
        r = run(orc, ref, p, d, args.layers, args.steps, args.batch)
        rel = abs(r["val_loss_final_o32"] - r["val_loss_final"]) / r["val_loss_final"]
        print(f"seed {p}:{d}: val {r['val_loss_init']:.6f} -> {r['val_loss_final']:.6f} (O64), "
              f"{r['val_loss_final_o32']:.6f} (O32), rel {rel:.3e}, {r['seconds']:.0f} s", flush=True)
        r["final_rel_o32"] = rel
        runs.append(r)
        golden = {"what": "reference (unfold_ref, FP64) config-5 training trajectories; "
                          "tools/train_reference_runs.py", "workers": ref.worker_count(),
                  "runs": [{k: v for k, v in q.items() if not k.endswith("o32") and k != "seconds"}
                           for q in runs[:args.golden_seeds]]}
        json.dump(golden, open(args.golden, "w"), indent=1)
        rels = [q["final_rel_o32"] for q in runs]
        spread = {"what": "O32 (FP32 restatement) vs O64 (the reference) after the same 100 "
                          "config-5 training steps: final validation-loss relative difference",
                  "runs": [{"pseed": q["pseed"], "dseed": q["dseed"], "final_rel": q["final_rel_o32"],
                            "val_o64": q["val_loss_final"], "val_o32": q["val_loss_final_o32"],
                            "step_rel": [abs(a - b) / b for a, b in zip(q["data_loss_o32"], q["data_loss"])]}
                           for q in runs],
                  "median": float(np.median(rels)), "max": float(np.max(rels))}
        json.dump(spread, open(args.spread, "w"), indent=1)


if __name__ == "__main__":
    main()
