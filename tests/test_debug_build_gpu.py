"""The debug build (make EXTRA=-DDETNET_DEBUG_ASSERT -> build/debug/, built by
__graft_entry__.build()): device-side bounds checks on the index math of
every kernel family, trapping on a violation -- the stand-in for
compute-sanitizer, which this GPU pool does not offer. One pass over every
kernel family (evaluation on the SIMT / 3xTF32 / split-FP16 / sparse paths,
dense, compacted and sparse-group models; FP32 and FP64 gradients and
training steps; a device group) must run clean and give the same results as
the product library (tools/debug_check.py)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEBUG_LIB = os.path.join(ROOT, "build", "debug", "libdetnet_b200.so")


@pytest.mark.skipif(not os.path.exists(DEBUG_LIB), reason="debug library not built")
def test_debug_assert_build_runs_clean_and_matches():
    outs = []
    for lib in (DEBUG_LIB, None):
        env = dict(os.environ)
        env.pop("DETNET_LIB", None)
        if lib:
            env["DETNET_LIB"] = lib
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "debug_check.py")],
                           env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        assert "DETNET_DASSERT" not in r.stdout + r.stderr
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs[0] == outs[1]
