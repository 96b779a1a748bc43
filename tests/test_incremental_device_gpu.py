"""SURVEY 8f row 2, device-resident: detnet_train_incremental runs the
reference's incremental-depth schedule (train_incremental, training.cpp:22-141)
entirely on the engine -- on-device batches with the reference's keying,
parameters and Adam moments in HBM, a fresh Adam state per step, validation,
halting, freeze + append with the reference's init draws -- against the
reference's own trainer on its own CPU kernels (oracle/_ref/incremental_ref,
same configuration). The on-device generator matches the host one to FP32
rounding (x bits exact), so the trajectories agree to the FP32 tolerances
of tests/test_incremental_gpu.py."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN_R = os.path.join(ROOT, "oracle", "_ref", "incremental_ref")


def _ref(args, tmp_path):
    if not os.path.exists(BIN_R):
        pytest.skip("incremental_ref not built (needs the reference tree at build time)")
    out = subprocess.run([BIN_R, *map(str, args), str(tmp_path / "r.json")], capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stderr + out.stdout
    return json.loads(out.stdout)


@pytest.mark.parametrize("K,N,start,tstep,maxl,batches,bsize,val,seed,rtol,btol", [
    (4, 8, 2, 1, 4, 30, 200, 1000, 5, 1e-5, 1e-3),
    (20, 30, 2, 1, 4, 20, 1000, 2000, 7, 2e-2, 1e-2),
])
def test_device_incremental_matches_reference(tmp_path, K, N, start, tstep, maxl, batches, bsize,
                                              val, seed, rtol, btol):
    from paper_2003_09446_b200 import Context
    r = _ref([K, N, start, tstep, maxl, batches, bsize, val, seed], tmp_path)
    c = Context(0)
    # incremental_main.cpp's configuration: halt_epsilon 0 (grow to max_layers),
    # validation at 10 dB, training SNR U[7, 14] dB, lr0 1e-3, group LASSO 1e-4
    recs, res, params = c.train_incremental(K, N, start, tstep, maxl, batches, bsize, val, seed,
                                            halt_epsilon=0.0, val_snr_db=10.0, snr_lo_db=7.0,
                                            snr_hi_db=14.0, lr0=1e-3, kind=2, lam1=1e-4)
    assert res["halt"] == r["halt"] == "max_layers"
    assert res["optimizer_steps"] == r["optimizer_steps"]
    assert [s["layers"] for s in recs] == [s["layers"] for s in r["steps"]]
    assert params.shape[0] == maxl and res["frozen_prefix"] == maxl - tstep
    for a, b in zip(recs, r["steps"]):
        assert abs(a["val_loss"] - b["val_loss"]) <= rtol * abs(b["val_loss"]), (a, b)
        assert abs(a["train_loss"] - b["train_loss"]) <= rtol * abs(b["train_loss"]), (a, b)
        assert abs(a["val_ber"] - b["val_ber"]) <= btol, (a, b)
    print(f"K={K}: device {res['seconds']:.3f} s vs reference {r['seconds']:.3f} s "
          f"({r['seconds'] / res['seconds']:.1f}x); steps {[round(s['val_loss'], 6) for s in recs]}")
