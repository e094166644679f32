"""Attribute ncu per-instruction SASS counters to source lines.

    python tools/sass_lines.py gpurun_out/sass_c2_cosine.csv <kernel-substring> [cubin-name]
Disassembles the matching kernel from the in-tree libsemidist_b200.so with line
info (nvdisasm -g) and sums 'Warp Stall Sampling (All Samples)' and
'Instructions Executed' per source line.
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def line_map(kernel_sub, cubin_name):
    so = os.path.join(ROOT, "paper_2104_06357_b200", "libsemidist_b200.so")
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", cubin_name, so], cwd=d, check=True, capture_output=True)
    cub = os.path.join(d, [f for f in os.listdir(d) if f.endswith(".cubin")][0])
    txt = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    amap, cur_fn, cur_line = {}, None, None
    for ln in txt.splitlines():
        m = re.match(r"^\.text\.(\S+):", ln)
        if m:
            cur_fn = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur_fn and kernel_sub in cur_fn:
            amap.setdefault(cur_fn, {})[int(m.group(1), 16)] = cur_line
    return amap


def main():
    path, ksub = sys.argv[1], sys.argv[2]
    cubin = sys.argv[3] if len(sys.argv) > 3 else "isect_f32.sm_100a.cubin"
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr_i]
    iA, iS, iI = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    data = [r for r in rows[hdr_i + 1:] if len(r) > iI and r[iA].startswith("0x") or (len(r) > iI and r[iA].isdigit())]
    amap = line_map(ksub, cubin)
    # pick the disassembled function with the same instruction count
    n = len(data)
    fn = min(amap, key=lambda f: abs(len(amap[f]) - n))
    am = amap[fn]
    samp, inst = collections.Counter(), collections.Counter()
    a0 = int(data[0][iA], 16) if data[0][iA].startswith("0x") else int(data[0][iA])
    for r in data:
        a = (int(r[iA], 16) if r[iA].startswith("0x") else int(r[iA])) - a0
        key = am.get(a, "?")
        samp[key] += float(r[iS] or 0)
        inst[key] += float(r[iI] or 0)
    ts, ti = sum(samp.values()), sum(inst.values())
    print(f"function {fn} ({len(am)} sass vs {n} profiled); samples {ts:.0f}, warp inst {ti:.3g}")
    for k, v in sorted(samp.items(), key=lambda kv: -kv[1])[:40]:
        print(f"{k:28s} samples {100 * v / ts:5.1f}%  inst {100 * inst[k] / ti:5.1f}%")


if __name__ == "__main__":
    main()
