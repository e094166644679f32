"""Key metrics + stall reasons from an ncu --page raw --csv export.

    python tools/ncu_raw.py gpurun_out/raw_c2_cosine_hgather.csv
"""
import csv
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio"]


def main(path):
    rows = list(csv.reader(open(path)))
    h, units, vals = rows[0], rows[1], rows[2]
    m = dict(zip(h, vals))
    u = dict(zip(h, units))
    for k in KEYS:
        if k in m:
            print(f"{k} = {m[k]} {u.get(k, '')}")
    st = [(k, float(m[k].replace(',', ''))) for k in h
          if k.startswith("smsp__average_warp_latency_issue_stalled_") or
          (k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"))]
    tot = sum(v for _, v in st) or 1
    print("# stall sampling (share)")
    for k, v in sorted(st, key=lambda kv: -kv[1])[:10]:
        print(f"  {k.split('stalled_')[-1]:28s} {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
