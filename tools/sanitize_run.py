"""Small dressing workloads for compute-sanitizer (memcheck / racecheck /
synccheck) and the IQCC_DEBUG bounds checks: G_mol(124, 2e5) through a
compressed dress_sequence (merge, rank, carry, partition, select kernels),
a 200-qubit sequence (4 device blocks), the pipelined merge variant, the
device PartitionedSum (exchange + gather), and the energy/gradient kernels.
Each case is checked against the CPU checker so a sanitizer run also proves
the results unchanged.  Usage: python tools/sanitize_run.py [--small]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def entanglers(n, k, seed):
    rs = np.random.default_rng(seed)
    B = (n + 63) // 64
    out = []
    for _ in range(k):
        row = np.zeros(2 * B, np.uint64)
        qs = rs.choice(n, 3, replace=False)
        for j, q in enumerate(qs):
            row[q // 64] |= np.uint64(1 << int(q % 64))
            if j == 1:
                row[B + q // 64] |= np.uint64(1 << int(q % 64))
        out.append((row, float(rs.uniform(-0.2, 0.2))))
    return out


def main():
    small = "--small" in sys.argv
    from oracle.oracle import Oracle
    from paper_2603_08883_b200 import iqcc, native
    native.init(0)
    port = Oracle("port")
    terms = 20_000 if small else 200_000
    for n, M, steps in ((124, terms, 4), (200, terms // 4, 3)):
        ents = entanglers(n, steps, n)
        h = port.gen_mol(n, M, 2)
        want, _ = port.dress_sequence(h, np.stack([e[0] for e in ents]), [e[1] for e in ents], 1e-10, M)
        d = iqcc.DeviceSum.generate_mol(n, M, 2)
        d.dress_sequence(iqcc.Ansatz([iqcc.PauliWord(n, e[0]) for e in ents], [e[1] for e in ents]), 1e-10, M)
        got = d.download()
        wr, wc = want.export()
        assert np.array_equal(got.rows, wr) and np.array_equal(got.coeffs, wc), f"sequence {n}"
        th = np.random.default_rng(3).uniform(-3, 3, n)
        e, g = d.qmf_energy_gradient(iqcc.QmfState(th, th))
        e2 = d.expect(iqcc.QmfState(th, th))
        assert abs(e - e2) <= 1e-10 * max(1.0, abs(e))
        print(f"ok sequence n={n} terms={len(got)}", flush=True)
    # device PartitionedSum: 8 shards on one GPU, exchange + gather
    h = port.gen_mol(64, terms // 2, 4)
    r, c = h.export()
    bits, _ = port.choose_partition_bits(h, 3)
    pm = iqcc.PartitionMap(64, [int(b) for b in bits], [p % 4 for p in range(8)], 4)
    ph = iqcc.distribute(iqcc.PauliSum(64, r, c), pm)
    row = np.zeros(2, np.uint64)
    b0 = int(bits[0])
    row[0 if b0 < 64 else 1] |= np.uint64(1 << (b0 % 64))
    row[0] |= np.uint64(1 << ((b0 + 7) % 64))
    ph.dress(iqcc.DressOp(iqcc.PauliWord(64, row), 0.3), 1e-9, terms)
    want, _ = port.dress_sequence(h, row[None, :], [0.3], 1e-9, terms)
    got = ph.gather()
    wr, wc = want.export()
    assert np.array_equal(got.rows, wr) and np.array_equal(got.coeffs, wc), "psum"
    print("ok psum", len(got), flush=True)
    print("SANITIZE RUN OK", flush=True)


if __name__ == "__main__":
    main()
