"""Summarise gpurun_out/ ncu artefacts into profiles/ (tracked).

    python tools/summarize_ncu.py <tag>
writes profiles/<tag>_launches.txt (per-kernel share of the step from the
gpu__time_duration launch list), profiles/<tag>_isect_ncu.txt (key metrics and
stall reasons of the fused kernel from the --set full capture) and
profiles/ncu_isect_traffic.json (DRAM bytes per launch, read by bench.py).
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def launches(tag):
    rows = [r for r in csv.reader(open(os.path.join(OUT, "launches.csv"))) if len(r) > 10]
    h, data = rows[0], rows[1:]
    iN, iV, iU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        v = float(r[iV].replace(",", ""))
        v = v * 1e3 if r[iU] == "ms" else (v / 1e3 if r[iU] in ("ns", "nsecond") else v)
        name = r[iN].split("(")[0]
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    lines = ["# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)",
             "# command: python bench.py --steps 3 --warmup 3 --no-cpu --extra   (index build included once)",
             f"{'share':>6} {'avg_us':>10} {'count':>5}  kernel"]
    for n, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{v / s * 100:5.1f}% {v / cnt[n]:10.1f} {cnt[n]:5d}  {n}")
    open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")
    return tot, cnt


def full(tag):
    rep = os.path.join(OUT, "prof_isect.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, units, v = r[0], r[1], r[2]
    m = dict(zip(h, v))
    u = dict(zip(h, units))

    def num(k):
        return float(m[k].replace(",", "")) if k in m and m[k] not in ("", "n/a") else None

    def to_bytes(k):
        x = num(k)
        if x is None:
            return None
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
        return x * scale.get(u.get(k, "byte"), 1)

    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
            "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__block_size",
            "launch__grid_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "smsp__thread_inst_executed_per_inst_executed.ratio"]
    lines = [f"# ncu --set full --clock-control none, kernel {r[2][h.index('Kernel Name')] if 'Kernel Name' in h else ''}",
             "# command: python bench.py --steps 1 --warmup 1 --no-cpu --extra  (C2 cosine, 10k x 162,541, fp32)"]
    for k in keys:
        if k in m:
            lines.append(f"{k} = {m[k]} {u.get(k, '')}")
    stalls = [(k, num(k)) for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    tot = sum(x for _, x in stalls if x)
    lines.append("# warp stall sampling (share of samples)")
    for k, x in sorted(stalls, key=lambda t: -(t[1] or 0))[:10]:
        lines.append(f"  {k.split('stalled_')[1]:24s} {x / tot * 100:5.1f}%")
    open(os.path.join(PROF, f"{tag}_isect_ncu.txt"), "w").write("\n".join(lines) + "\n")
    traffic = (to_bytes("dram__bytes_read.sum") or 0) + (to_bytes("dram__bytes_write.sum") or 0)
    json.dump({"kernel": "isect_kernel<float, cosine>", "dram_bytes_per_launch": traffic,
               "dram_read_bytes": to_bytes("dram__bytes_read.sum"), "dram_write_bytes": to_bytes("dram__bytes_write.sum"),
               "source": f"profiles/{tag}_isect_ncu.txt"},
              open(os.path.join(PROF, "ncu_isect_traffic.json"), "w"), indent=1)
    return traffic


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    launches(tag)
    print("traffic bytes/launch", full(tag))
    for f in ("bench.json", "bench_ref.json"):
        if os.path.exists(os.path.join(OUT, f)):
            open(os.path.join(PROF, f"{tag}_{f}"), "w").write(open(os.path.join(OUT, f)).read())
