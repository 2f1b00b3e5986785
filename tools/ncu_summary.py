"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py <launches.csv> <full.ncu-rep> <images> <tag>

(<images>: images per launch of the --set full capture; NCU_LAUNCH_CMD names
the command of the launch list when it differs from the default.)

Writes profiles/<tag>_launches.md (per-kernel share of the step from the
`gpu__time_duration` launch list), profiles/<tag>_ncu_full.md (key counters and
stall reasons per kernel from the `--set full` capture) and
profiles/kernel_traffic.json (DRAM bytes per launch per image, read by
bench.py for the roofline `traffic` field).
"""

import collections
import csv
import io
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_%",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_%",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_%",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_%",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_%",
    "launch__registers_per_thread": "regs",
    "smsp__inst_executed.sum": "warp_inst",
}

SHORT = {
    "place_assemble_kernel": "place_assemble_kernel",
    "place_ranges_kernel": "place_ranges_kernel",
    "gdt_x_kernel": "gdt_x_kernel",
    "gdt_y_kernel": "gdt_y_kernel",
    "corr_tc_kernel": "corr_tc_kernel",
    "corr_kernel": "corr_kernel",
    "project_kernel": "project_kernel",
    "project_mma_kernel": "project_mma_kernel",
}


def short(name):
    for k in SHORT:
        if k in name:
            base = name.split("(")[0].replace("void ", "").replace("dpm::", "")
            return base
    return name.split("(")[0][:60]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if r[mi] == "gpu__time_duration.sum":
            agg[short(r[ki])].append(float(r[vi].replace(",", "")))
    return agg


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6,
             "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    out = []
    for r in rows[2:]:
        rec = {"kernel": short(r[ki])}
        for m, k in KEYS.items():
            if m in h:
                try:
                    v = float(r[h.index(m)].replace(",", ""))
                except ValueError:
                    continue
                # durations -> us, bytes -> MB
                rec[k] = v * scale.get(units[h.index(m)], 1.0)
        stalls = []
        for i, m in enumerate(h):
            if m.startswith("smsp__pcsamp_warps_issue_stalled") and not m.endswith("not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")),
                                   m.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        rec["stalls"] = [(n, round(100 * v / tot, 1)) for v, n in sorted(stalls, reverse=True)[:6]]
        out.append(rec)
    return out


def main(launch_csv, rep, images, tag):
    images = int(images)
    prof = os.path.join(REPO, "profiles")
    la = launches(launch_csv)
    ours = {k: v for k, v in la.items() if "probe" not in k and "at::" not in k and "elementwise" not in k}
    per_step = {k: sum(v) / max(1, len(v)) for k, v in ours.items()}
    tot = sum(per_step.values())
    with open(os.path.join(prof, f"{tag}_launches.md"), "w") as fh:
        fh.write(f"# {tag}: ncu launch list (gpu__time_duration, --clock-control none)\n\n")
        cmd = os.environ.get("NCU_LAUNCH_CMD",
                             f"bench.py --images {images} --steps 2 --warmup 3 --no-cpu")
        fh.write(f"Command: `{cmd}` under ncu "
                 "(cold-cache, serialised launches: compare shares, not absolutes).\n\n")
        fh.write("| kernel | launches | mean time / launch (us) | share of step |\n|---|---|---|---|\n")
        for k, v in sorted(per_step.items(), key=lambda kv: -kv[1]):
            fh.write(f"| `{k}` | {len(ours[k])} | {v / 1e3:.1f} | {100 * v / tot:.1f}% |\n")
    fu = full(rep)
    traffic = {}
    with open(os.path.join(prof, f"{tag}_ncu_full.md"), "w") as fh:
        fh.write(f"# {tag}: ncu --set full summary ({images} images per launch)\n\n")
        fh.write("| kernel | time (us) | DRAM read+write (MB) | per image (MB) | tensor pipe % | "
                 "FMA pipe % | FP64 pipe % | issue active % | occupancy % | regs | top stalls |\n")
        fh.write("|---|---|---|---|---|---|---|---|---|---|---|\n")
        seen = set()
        for rec in fu:
            dram = rec.get("dram_read", 0) + rec.get("dram_write", 0)
            name = rec["kernel"]
            if name in seen:  # the capture's -c may wrap into the next run: one launch each
                continue
            seen.add(name)
            # ncu reports bytes in the unit of the column (MB in --csv raw for these metrics)
            # one entry per kernel family (template instantiations summed: a
            # step launches each family's instantiations once)
            fam = name.split("<")[0]
            if "at::" not in name and "elementwise" not in name:
                traffic[fam] = traffic.get(fam, 0.0) + dram * 1e6 / images
            fh.write(f"| `{name}` | {rec.get('duration', 0):.1f} | {dram:.1f} | "
                     f"{dram / images:.2f} | {rec.get('tensor_pipe_%', 0):.1f} | "
                     f"{rec.get('fma_pipe_%', 0):.1f} | {rec.get('fp64_pipe_%', 0):.1f} | "
                     f"{rec.get('issue_active_%', 0):.1f} | {rec.get('occupancy_%', 0):.1f} | "
                     f"{rec.get('regs', 0):.0f} | "
                     + ", ".join(f"{n} {p}%" for n, p in rec["stalls"][:4]) + " |\n")
    with open(os.path.join(prof, "kernel_traffic.json"), "w") as fh:
        json.dump({"unit": "dram bytes per launch per image (multiply by images)",
                   "source": f"profiles/{tag}_ncu_full.md", "per_image": traffic}, fh, indent=1)
    print(open(os.path.join(prof, f"{tag}_launches.md")).read())
    print(open(os.path.join(prof, f"{tag}_ncu_full.md")).read())


if __name__ == "__main__":
    main(*sys.argv[1:5])
