"""expect_sum / qmf_energy_gradient on G_mol(124, N) at a generic Omega
(profiling driver: python tools/energy_run.py [N] [reps])."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    N = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    from paper_2603_08883_b200 import iqcc, native
    native.init(0)
    n = 124
    d = iqcc.DeviceSum.generate_mol(n, N, 2)
    rs = np.random.default_rng(5)
    om = iqcc.QmfState(rs.uniform(-3, 3, n), rs.uniform(-3, 3, n))
    for name, fn in (("expect", lambda: d.expect(om)), ("qmf_grad", lambda: d.qmf_energy_gradient(om))):
        fn()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        print(name, f"{1e3 * (time.perf_counter() - t0) / reps:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
