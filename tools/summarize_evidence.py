"""Copy a round's GPU evidence (gpurun_out/, scratch) into profiles/ (tracked).

    python tools/summarize_evidence.py r02a

writes profiles/<tag>_bench_<workload>.json, <tag>_bench_ref.json,
<tag>_launches.txt, <tag>_ncu_<workload>_<metric>_<dtype>_<kernel>.txt (key
metrics + stall reasons of one launch, each file headed by the exact command
that produced it) and merges the sweep kernel's DRAM bytes per launch into
profiles/ncu_traffic.json keyed "<workload>/<metric>/<f32|f64>" — the
`roofline.traffic` bench.py reports for the same workload, metric and dtype.
"""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def run(*args):
    return subprocess.run([sys.executable, *args], capture_output=True, text=True, cwd=ROOT).stdout


def main(tag):
    for f in glob.glob(os.path.join(OUT, "bench_*.json")):
        lines = [l for l in open(f).read().splitlines() if l.startswith("{")]
        if lines:
            open(os.path.join(PROF, f"{tag}_{os.path.basename(f)}"), "w").write(lines[-1] + "\n")
    if os.path.exists(os.path.join(OUT, "launches.csv")):
        txt = run("tools/summarize_launches.py", os.path.join(OUT, "launches.csv"))
        hdr = ("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)\n"
               "# command: python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --no-check\n"
               "# (index build and lazily built index parts included once)\n")
        open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write(hdr + txt)
    traffic_path = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for f in sorted(glob.glob(os.path.join(OUT, "raw_*.csv"))):
        name = os.path.basename(f)[len("raw_"):-len(".csv")]      # <wl>_<metric>_<dtype>_<kernel>
        wl, metric, dt, kernel = name.split("_", 3)
        txt = run("tools/ncu_raw.py", f)
        if not txt.strip():
            continue
        hdr = (f"# ncu -f --set full --clock-control none --import-source on -k regex:{kernel} -s 1 -c 1 (one launch)\n"
               f"# command: python bench.py --workload {wl} --metric {metric} --dtype {dt} --steps 1 --warmup 1 "
               f"--no-cpu --no-extra --no-check\n")
        out = os.path.join(PROF, f"{tag}_ncu_{name}.txt")
        open(out, "w").write(hdr + txt)
        if kernel != "isect_kernel":
            continue
        vals = {}
        for line in txt.splitlines():
            k, _, v = line.partition(" = ")
            vals[k.strip()] = v.strip()

        def nbytes(k):
            num, unit = vals[k].split()[:2]
            return float(num.replace(",", "")) * UNITS[unit]
        rd, wr = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
        traffic[f"{wl}/{metric}/{'f32' if dt == 'float32' else 'f64'}"] = {
            "kernel": vals.get("Kernel Name", kernel), "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd,
            "dram_write_bytes": wr, "duration": vals.get("gpu__time_duration.sum"),
            "source": os.path.relpath(out, ROOT)}
    json.dump(traffic, open(traffic_path, "w"), indent=1, sort_keys=True)
    for f in glob.glob(os.path.join(OUT, "sanitize_*.log")):
        tool = os.path.basename(f)[len("sanitize_"):-len(".log")]
        lines = open(f).read().splitlines()
        keep = [l for l in lines if l.startswith("ok ") or "SUMMARY" in l]
        hdr = f"# compute-sanitizer --tool {tool} (tools/sanitize.sh -> python tools/sanitize_cases.py)\n"
        open(os.path.join(PROF, f"{tag}_sanitize_{tool}.txt"), "w").write(hdr + "\n".join(keep) + "\n")
    for name in ("hbm_probe.json", "timeline_c2_cosine.txt", "timeline_c2_manhattan.txt",
                 "timeline_c2_cosine_q1250.txt", "timeline_c5_cosine.txt"):
        f = os.path.join(OUT, name)
        if os.path.exists(f):
            open(os.path.join(PROF, f"{tag}_{name}"), "w").write(open(f).read())


if __name__ == "__main__":
    main(sys.argv[1])
