"""SURVEY 8f row 2 measurement: the reference's train_incremental running on
the B200 seam, the device-resident detnet_train_incremental, and the
reference on its own OpenMP kernels (same box, same arguments). Prints one JSON line per schedule; wall-clock includes context
creation, generation, validation and checkpoint round trip (the whole
controller), and the marginal per-optimizer-step time from two run lengths."""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B = os.path.join(ROOT, "oracle", "_ref", "incremental_b200")
R = os.path.join(ROOT, "oracle", "_ref", "incremental_ref")


def run(binary, args):
    with tempfile.TemporaryDirectory() as td:
        out = subprocess.run([binary, *map(str, args), os.path.join(td, "ck.json")],
                             capture_output=True, text=True, timeout=1800)
    if out.returncode:
        raise SystemExit(out.stderr + out.stdout)
    return json.loads(out.stdout)


_CTX = None


def run_device(args):
    """detnet_train_incremental with incremental_main.cpp's configuration."""
    global _CTX
    sys.path.insert(0, ROOT)
    from paper_2003_09446_b200 import Context
    K, N, s0, ts, mx, nb, bs, val, seed = args
    if _CTX is None:  # one context: its training workspace is allocated once (warm-up)
        _CTX = Context(0)
    c = _CTX
    recs, res, _ = c.train_incremental(K, N, s0, ts, mx, nb, bs, val, seed, halt_epsilon=0.0,
                                       val_snr_db=10.0, snr_lo_db=7.0, snr_hi_db=14.0, lr0=1e-3,
                                       kind=2, lam1=1e-4)
    # the controller's own per-step wall clocks (batches, Adam, validation, each
    # waited for on the host): context and model creation are not step time
    return {"seconds": sum(r["wall_ms"] for r in recs) / 1e3, "optimizer_steps": res["optimizer_steps"],
            "steps": recs}


def main():
    # (label, K, N, start, t_step, max_layers, batches_short, batches_long, batch, val)
    cases = [("whole-network L=40 (config-5 dims)", 20, 30, 40, 10, 40, 4, 12, 5000, 2000),
             ("incremental 10->40 by 10", 20, 30, 10, 10, 40, 2, 6, 5000, 2000)]
    # warm-up: module load, workspace, and every depth the schedules visit
    for _, K, N, s0, ts, mx, b1, _, bs, val in cases:
        run_device([K, N, s0, ts, mx, b1, bs, val, 1])
    for label, K, N, s0, ts, mx, b1, b2, bs, val in cases:
        res = {}
        for name, binary in (("b200", B), ("device", None), ("reference", R)):
            # the engine legs run 3x the batches: their steps are short next to
            # the fixed costs (process / context start, model creation)
            mult = 1 if name == "reference" else 3
            if binary is None:
                a, c = (run_device([K, N, s0, ts, mx, mult * bb, bs, val, 3]) for bb in (b1, b2))
            else:
                a = run(binary, [K, N, s0, ts, mx, mult * b1, bs, val, 3])
                c = run(binary, [K, N, s0, ts, mx, mult * b2, bs, val, 3])
            per_step = (c["seconds"] - a["seconds"]) / (c["optimizer_steps"] - a["optimizer_steps"])
            res[name] = {"seconds_long": c["seconds"], "optimizer_steps_long": c["optimizer_steps"],
                         "marginal_ms_per_optimizer_step": per_step * 1e3,
                         "samples_per_s_marginal": bs / per_step,
                         "final_val_loss": c["steps"][-1]["val_loss"],
                         "final_val_ber": c["steps"][-1]["val_ber"]}
        print(json.dumps({"case": label, "batch": bs, "cores_reference": os.cpu_count(), **res,
                          "speedup_marginal_seam": res["reference"]["marginal_ms_per_optimizer_step"] /
                          res["b200"]["marginal_ms_per_optimizer_step"],
                          "speedup_marginal_device": res["reference"]["marginal_ms_per_optimizer_step"] /
                          res["device"]["marginal_ms_per_optimizer_step"]}))
        sys.stdout.flush()


if __name__ == "__main__":
    main()
