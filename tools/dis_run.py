"""DIS gradients at a generic Omega on G_mol(100, N) for K odd-Y candidates
(profiling driver: python tools/dis_run.py [N] [K])."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    N = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
    K = int(float(sys.argv[2])) if len(sys.argv) > 2 else 10_000
    from bench_aux import odd_y_candidates
    from paper_2603_08883_b200 import iqcc, native
    native.init(0)
    n = 100
    d = iqcc.DeviceSum.generate_mol(n, N, 3)
    rs = np.random.default_rng(9)
    om = iqcc.QmfState(rs.uniform(-3, 3, n), rs.uniform(-3, 3, n))
    cands = odd_y_candidates(n, K, 4)
    d.gradients(om, cands[:256])
    t0 = time.perf_counter()
    g = d.gradients(om, cands)
    dt = time.perf_counter() - t0
    print(f"dis {N} x {K}: {dt:.3f} s, {N * K / dt:.3e} pairs/s, checksum {np.abs(g).sum():.12e}", flush=True)


if __name__ == "__main__":
    main()
