"""PCIe duplex check: pinned H2D and D2H alone and concurrently (two streams).

Prints one JSON line per case with GB/s per direction; used to decide how
far e2e calls can overlap (bench.py --e2e-inflight).
"""
import json
import time

import torch

GB = 1 << 30


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t


def main():
    n = 4 * GB
    h_src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def h2d():
        with torch.cuda.stream(s1):
            d_a.copy_(h_src, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_dst.copy_(d_b, non_blocking=True)

    for _ in range(2):
        timed(h2d)
        timed(d2h)
    t_h2d = timed(h2d)
    t_d2h = timed(d2h)
    t_both = timed(lambda: (h2d(), d2h()))
    print(json.dumps({"h2d_gbs": n / t_h2d / 1e9, "d2h_gbs": n / t_d2h / 1e9,
                      "both_ms": 1e3 * t_both, "serial_ms": 1e3 * (t_h2d + t_d2h),
                      "duplex_gbs_each": n / t_both / 1e9}))


if __name__ == "__main__":
    main()
