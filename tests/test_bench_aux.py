"""CPU checks of bench_aux.py's synthetic inputs: the
G_uniform generator yields a canonically sorted, duplicate-free sum (the
checker re-sorts it into the same rows), and the DIS candidates have the
odd-#Y, weight-4 shape dis_candidates produces (iqcc/dis.hpp:89-116)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_g_uniform_is_canonical():
    import bench_aux
    from oracle.oracle import Oracle
    h = bench_aux.g_uniform(64, 4000, 1)
    port = Oracle("port")
    rows = np.ascontiguousarray(h.rows, np.uint64)
    coeffs = np.ascontiguousarray(h.coeffs, np.complex128)
    want, _ = port.from_terms(64, rows, coeffs, drop=0.0, check=False).export()
    assert np.array_equal(want, rows)
    assert len(h) > 3900


def test_dis_candidates_shape():
    import bench_aux
    c = bench_aux.odd_y_candidates(100, 64, 4)
    for row in c:
        x = int(row[0]) | (int(row[1]) << 64)
        z = int(row[2]) | (int(row[3]) << 64)
        assert bin(x).count("1") == 4
        assert z & ~x == 0 and bin(z).count("1") % 2 == 1
    # groups of 8 candidates share one support
    for g in range(0, 64, 8):
        assert len({(int(r[0]), int(r[1])) for r in c[g:g + 8]}) == 1
