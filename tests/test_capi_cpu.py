"""CPU-only checks of the product boundary: the C-ABI library loads, exports
every entry point include/detnet_b200.h declares, refuses to run without a
GPU (no CPU fallback), and its host-side helpers (Rng keying, workload
builders) agree with the oracle."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "detnet_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(detnet_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    from paper_2003_09446_b200.detnet import LIB_PATH
    lib = C.CDLL(LIB_PATH)
    names = _declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a():
    from paper_2003_09446_b200.detnet import LIB_PATH
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2003_09446_b200 as p
    with pytest.raises(p.CudaError):
        p.Context(0)


def test_rng_helpers_match_oracle(oracle):
    import paper_2003_09446_b200 as p
    r = oracle.rng(77, 5)
    assert p.rng_seed(77, 5) == r.s
    assert p.rng_stream(r.s, 0x45564131 + 3) == oracle.lib.or_stream(C.byref(r), 0x45564131 + 3).s
    child, adv = p.rng_split(r.s)
    rr = oracle.rng(77, 5)
    c2 = oracle.lib.or_split(C.byref(rr))
    assert child == c2.s and adv == rr.s


def test_workload_xavier_matches_oracle(oracle):
    from oracle.oracle import xavier_model
    from paper_2003_09446_b200.workload import xavier_params
    m = xavier_model(oracle, n_tx=4, n_rx=8, depth=3, seed=9)
    assert np.array_equal(xavier_params(4, 3, seed=9), m.params)
    m20 = xavier_model(oracle, n_tx=20, n_rx=30, depth=2, seed=9)
    p20 = xavier_params(20, 2, seed=9)
    assert np.array_equal(p20, m20.params)
    # Xavier bound a = sqrt(6/(fan_in+fan_out)): 0.1519 for W1 at K=20
    from paper_2003_09446_b200.workload import record_layout
    sl, _ = record_layout(20, 160, 40)
    assert abs(np.abs(p20[0, sl["W1"]]).max() - np.sqrt(6 / 260)) < 1e-3


def test_group_masks_census(oracle):
    """Config 3 masks give the 556,400-FLOP census."""
    from oracle.oracle import Model
    from paper_2003_09446_b200.workload import group_masks, xavier_params
    p = xavier_params(20, 40, seed=9)
    mk = group_masks(20, 40, seed=31)
    m = Model(20, 30, 160, 40, 40, p, masks=mk)
    assert oracle.flops_per_detection(m) == 556_400
