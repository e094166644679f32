"""Copy the round's GPU evidence (gpurun_out/, scratch) into profiles/ (tracked).

    python tools/summarize_evidence.py r01c
writes profiles/<tag>_bench_<workload>.json, <tag>_bench_ref.json,
<tag>_launches.txt, <tag>_ncu_<kernel>.txt (key metrics + stall reasons from
the ncu --set full text exports) and profiles/ncu_isect_traffic.json (DRAM
bytes per launch of the fused kernel, read by bench.py for roofline.traffic).
"""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def run(*args):
    return subprocess.run([sys.executable, *args], capture_output=True, text=True, cwd=ROOT).stdout


def main(tag):
    for f in glob.glob(os.path.join(OUT, "bench_*.json")):
        lines = [l for l in open(f).read().splitlines() if l.startswith("{")]
        if lines:
            name = os.path.basename(f)
            open(os.path.join(PROF, f"{tag}_{name}"), "w").write(lines[-1] + "\n")
    if os.path.exists(os.path.join(OUT, "launches.csv")):
        txt = run("tools/summarize_launches.py", os.path.join(OUT, "launches.csv"))
        hdr = ("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)\n"
               "# command: python bench.py --steps 3 --warmup 3 --no-cpu --no-extra  (index build included once)\n")
        open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write(hdr + txt)
    for f in sorted(glob.glob(os.path.join(OUT, "raw_*.csv"))):
        kern = os.path.basename(f)[len("raw_"):-len(".csv")]
        txt = run("tools/ncu_raw.py", f)
        hdr = (f"# ncu --set full --clock-control none --import-source on, one launch ({kern})\n"
               "# command: python bench.py --workload c2 --metric cosine --steps 1 --warmup 1 --no-cpu --no-extra\n")
        open(os.path.join(PROF, f"{tag}_ncu_{kern}.txt"), "w").write(hdr + txt)
        if kern.endswith("isect_kernel"):
            vals = {}
            for line in txt.splitlines():
                k, _, v = line.partition(" = ")
                vals[k.strip()] = v.strip()

            def gb(k):
                num, unit = vals[k].split()[:2]
                return float(num.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
            rd, wr = gb("dram__bytes_read.sum"), gb("dram__bytes_write.sum")
            json.dump({"kernel": "isect_kernel<float, cosine>", "workload": "c2", "dram_bytes_per_launch": rd + wr,
                       "dram_read_bytes": rd, "dram_write_bytes": wr,
                       "source": f"profiles/{tag}_ncu_{kern}.txt"},
                      open(os.path.join(PROF, "ncu_isect_traffic.json"), "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1])
