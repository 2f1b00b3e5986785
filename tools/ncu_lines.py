"""Attribute an ncu capture's per-instruction counts to CUDA source lines.

    python tools/ncu_lines.py <report.ncu-rep> <kernel regex> <object.o> <mangled kernel> [top]

NCU_LINES_SKIP=k takes the (k+1)-th matching launch.  NCU_LINES_SORT=stall ranks the lines by stall samples instead of instructions.

Joins the SASS page of the report (executed instructions and stall samples
per instruction) with `nvdisasm --print-line-info` of the kernel in the
object file (same build), by offset from the function start.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main():
    rep, kre, obj, fn = sys.argv[1:5]
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kre}", "--launch-skip", os.environ.get("NCU_LINES_SKIP", "0"),
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    seen, data = set(), []
    for r in rows[2:]:
        if len(r) == len(hdr) and r[0].startswith("0x") and r[0] not in seen:
            seen.add(r[0])
            data.append(r)
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        dis = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(d, cub)],
                             capture_output=True, text=True).stdout.split("\n")
    start = [i for i, l in enumerate(dis) if l.startswith(".text." + fn)][0]
    off2loc, cur = {}, None
    for l in dis[start + 1:]:
        if l.startswith("//---------------------") and ".text." in l:
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+", l)
        if m and cur:
            off2loc[int(m.group(1), 16)] = cur
    base = int(data[0][0], 16)
    ie = hdr.index("Instructions Executed")
    ws = hdr.index("Warp Stall Sampling (All Samples)")
    ins, st = collections.Counter(), collections.Counter()
    for r in data:
        k = off2loc.get(int(r[0], 16) - base, "?")
        ins[k] += int(r[ie])
        st[k] += int(r[ws])
    ti, ts = sum(ins.values()), sum(st.values())
    print(f"instructions {ti}, stall samples {ts}")
    srcs = {}
    order = st if os.environ.get("NCU_LINES_SORT") == "stall" else ins
    for k, _ in order.most_common(top):
        n = ins[k]
        f, _, ln = k.partition(":")
        if f not in srcs:
            path = os.path.join(os.path.dirname(obj), "..", "..", "paper_1707_03268_b200", "csrc", f)
            srcs[f] = open(path).read().split("\n") if os.path.exists(path) else []
        text = srcs[f][int(ln) - 1].strip()[:64] if ln.isdigit() and srcs[f] else ""
        print(f"{k:22s} {n / ti * 100:5.1f}% instr {st[k] / ts * 100:5.1f}% stall  {text}")


if __name__ == "__main__":
    main()
