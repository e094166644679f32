"""HBM ceilings for the sweep's traffic pattern: write-only (fill), read-only
(sum) and copy bandwidth on 6.5 GB buffers (the C2 output size), CUDA-event
timed, median of 10.  The sweep kernel writes its output and reads little,
so its roofline is the write-only figure, not the copy figure.

    python tools/hbm_probe.py
"""
import json

import torch


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / 1e3)
    out.sort()
    return out[len(out) // 2]


def main():
    n = 6_500_000_000 // 4
    a = torch.empty(n, dtype=torch.float32, device="cuda")
    b = torch.empty(n, dtype=torch.float32, device="cuda")
    nbytes = n * 4
    res = {}
    res["write_fill_gbs"] = nbytes / timed(lambda: a.fill_(1.0)) / 1e9
    res["write_memset_gbs"] = nbytes / timed(lambda: a.zero_()) / 1e9
    res["copy_gbs_read_plus_write"] = 2 * nbytes / timed(lambda: b.copy_(a)) / 1e9
    res["read_sum_gbs"] = nbytes / timed(lambda: a.sum()) / 1e9
    print(json.dumps({k: round(v, 1) for k, v in res.items()}))


if __name__ == "__main__":
    main()
