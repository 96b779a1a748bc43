"""Turns the ncu reports written by tools/capture_profiles.sh into the text
summaries kept under profiles/ (run here, after gpurun merged gpurun_out/)."""
import csv, io, os, subprocess, sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
    "lts__t_sector_hit_rate.pct", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def main(src, dst, title):
    lines = [f"# {title}", "# ncu --set full --clock-control none; per-launch values (cold-cache, serialised)", ""]
    for rep in sorted(os.listdir(src)):
        if not rep.endswith(".ncu-rep"):
            continue
        recs, units = raw(os.path.join(src, rep))
        for r in recs:
            lines.append(f"== {r.get('Kernel Name', '?')[:90]}  ({rep})")
            for m in METRICS:
                if m in r:
                    lines.append(f"  {m} = {r[m]} {units.get(m, '')}")
            lines.append("")
    open(dst, "w").write("\n".join(lines))
    print("\n".join(lines))
    # DRAM bytes per detection of the stack kernels (bench.py's roofline.traffic)
    traffic = {}
    for rep in sorted(os.listdir(src)):
        if rep.startswith(("k_stack", "detnet_sparse_jit")) and rep.endswith(".ncu-rep"):
            recs, units = raw(os.path.join(src, rep))
            for r in recs:
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                b = sum(float(r[m]) * scale.get(units.get(m, "byte"), 1)
                        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
                traffic[rep[:-8]] = {"dram_bytes_per_launch": b, "detections_per_launch": 262144,
                                     "dram_bytes_per_detection": b / 262144}
    if traffic:
        import json
        json.dump(traffic, open(os.path.join(os.path.dirname(dst), "traffic.json"), "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "profile summary")
