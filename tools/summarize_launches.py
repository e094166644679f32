"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum launch list.

    python tools/summarize_launches.py gpurun_out/launches_x.csv
"""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h, data = rows[0], rows[1:]
    iN, iV, iU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        v = float(r[iV].replace(",", ""))
        v = v * 1e3 if r[iU] in ("ms", "msecond") else (v / 1e3 if r[iU] in ("ns", "nsecond") else v)
        name = r[iN].split("(")[0][:90]
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    print(f"{'share':>6} {'avg_us':>10} {'count':>5}  kernel")
    for n, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v / s * 100:5.1f}% {v / cnt[n]:10.1f} {cnt[n]:5d}  {n}")


if __name__ == "__main__":
    main(sys.argv[1])
