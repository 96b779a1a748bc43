"""Box probe: host cores, GPU properties and the TF32 / FP32 roofline denominators.

Runs on a gpurun box; writes gpurun_out/probe_box.json. The TF32 figure is the
denominator for the 3xTF32 layer-stack roofline (TF32 peak / 3), measured the
same way MEASURED_PEAKS.json measures bf16 (torch.matmul 8192^3, best of 10).
"""
import json
import os
import subprocess
import time

import torch


def gemm_tflops(dtype, n=8192, reps=10, tf32=False):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return 2 * n ** 3 / best / 1e12


def main():
    out = {}
    out["nproc"] = os.cpu_count()
    out["sched_affinity"] = len(os.sched_getaffinity(0))
    try:
        out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout[:2000]
    except Exception as e:  # pragma: no cover
        out["lscpu"] = str(e)
    p = torch.cuda.get_device_properties(0)
    out["gpu"] = {"name": p.name, "sms": p.multi_processor_count, "mem": p.total_memory,
                  "smem_per_block_optin": getattr(p, "shared_memory_per_block_optin", None),
                  "l2": getattr(p, "L2_cache_size", None)}
    out["tf32_tflops"] = gemm_tflops(torch.float32, tf32=True)
    out["fp32_tflops_cublas"] = gemm_tflops(torch.float32, tf32=False, reps=3)
    out["bf16_tflops"] = gemm_tflops(torch.bfloat16)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/probe_box.json", "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "lscpu"}))


if __name__ == "__main__":
    main()
