"""GPU parity for the energy / gradient / DIS rows:
expect_sum, qmf_energy_gradient, gradient, dis_candidates and
choose_partition_bits against the CPU checker, restating tests/test_qmf.cpp
and tests/test_dis.cpp.  Tolerances: the exact modes (per-term expect_word
values, IQCC_DIS_EXACT gradients, dis_candidates) are summed in the
reference's order and compared bit-exactly; the nibble-table DIS gradients
within 1e-13; energies and QMF gradients are sums in a different order,
compared at 1e-10 relative (north_star's fp64 tolerance)."""
import math
import os

import numpy as np
import pytest

from helpers import load_golden

pytestmark = pytest.mark.gpu

REL = 1e-10


def host(eng, osum):
    r, c = osum.export()
    return eng.PauliSum(osum.n_qubits, r, c)


def close(a, b, rel=REL):
    return abs(a - b) <= rel * max(1.0, abs(b))


def test_expect_word_axes(eng):  # test_qmf.cpp:21-27
    om = eng.QmfState.zeros(1)
    h = eng.PauliSum(1)
    h.append(eng.PauliWord.from_string("Z"), 1.0)
    assert eng.expect_sum(om, h) == 1.0
    om.theta[0] = math.pi / 2
    hx = eng.PauliSum(1)
    hx.append(eng.PauliWord.from_string("X"), 1.0)
    assert eng.expect_sum(om, hx) == pytest.approx(1.0)


def test_expect_sum_random(eng, port):
    rng = port.rng(201)
    for t in range(40):
        n = 2 + t % 30
        h = rng.sum(n, 200)
        th, ph = rng.qmf(n)
        got = eng.expect_sum(eng.QmfState(th, ph), host(eng, h))
        assert close(got, port.expect_sum(th, ph, h))

def test_expect_word_values(eng, port, monkeypatch):
    """One-term sums: the nibble-table product (default) agrees with
    expect_word to 1e-14; the lockstep mode (IQCC_EXPECT_EXACT=1) is bit-exact."""
    rng = port.rng(203)
    cases = []
    for t in range(100):
        n = 1 + t % 200
        w = rng.word(n)
        cases.append((n, w, rng.qmf(n)))
    for n, w, (th, ph) in cases:
        h = port.sum(n, w[None, :], [1.0])
        want = port.expect_word(n, th, ph, w)
        assert abs(eng.expect_sum(eng.QmfState(th, ph), host(eng, h)) - want) <= 1e-13 * max(1e-300, abs(want))
    monkeypatch.setenv("IQCC_EXPECT_EXACT", "1")
    for n, w, (th, ph) in cases:
        h = port.sum(n, w[None, :], [1.0])
        assert eng.expect_sum(eng.QmfState(th, ph), host(eng, h)) == port.expect_word(n, th, ph, w)


def test_h2_hf_energy(eng):  # test_qmf.cpp:54-66
    g = load_golden("c1_h2_sto3g.npz")
    h = eng.PauliSum(4, g["rows0"], g["coeffs0"])
    e = eng.expect_sum(eng.hf_reference([True, True, False, False]), h)
    assert e == pytest.approx(-1.11615145, abs=1e-6)
    assert close(e, float(g["e_hf"]), 1e-14)


@pytest.mark.parametrize("n", [6, 40, 124, 200])
def test_qmf_energy_gradient(eng, port, n):
    rng = port.rng(211 + n)
    h = rng.sum(n, 3000)
    th, ph = rng.qmf(n)
    e, g = eng.qmf_energy_gradient(host(eng, h), eng.QmfState(th, ph))
    er, gr = port.qmf_energy_gradient(h, th, ph)
    assert close(e, er)
    scale = max(1.0, np.abs(gr).max())
    assert np.abs(g - gr).max() <= REL * scale


@pytest.mark.parametrize("mode", ["bitsliced", "bins"])
def test_qmf_gradient_near_poles(eng, port, monkeypatch, mode):
    """|sin theta| ~ 1e-8 (a QMF state next to the HF poles): the c*P*(f'/f)
    rearrangement must still match the reference's prefix/suffix products
    (iqcc/qmf.hpp:94-148), on a Hamiltonian and on its G_mol-like shape;
    both kernels (the bit-sliced default and the per-qubit bins)."""
    if mode == "bins":
        monkeypatch.setenv("IQCC_QMF_GRAD_BINS", "1")
    rng = port.rng(223)
    for n, h in ((12, rng.sum(12, 800)), (124, port.gen_mol(124, 20000, 7))):
        th, ph = rng.qmf(n)
        occ = np.arange(n) < n // 3
        th = np.where(occ, np.pi - 1e-8 * (1 + np.arange(n) % 3), 1e-8 * (1 + np.arange(n) % 5))
        th[::7] += 0.3  # and some generic angles
        e, g = eng.qmf_energy_gradient(host(eng, h), eng.QmfState(th, ph))
        er, gr = port.qmf_energy_gradient(h, th, ph)
        assert close(e, er)
        assert np.abs(g - gr).max() <= REL * max(1.0, np.abs(gr).max())


@pytest.mark.parametrize("n", [64, 124, 200])
def test_qmf_gradient_gmol_kernels_agree(eng, port, monkeypatch, n):
    """The bit-sliced kernel against the reference at G_mol shapes (sparse x
    planes, the benchmark's shape) and against the per-qubit-bin kernel."""
    h = port.gen_mol(n, 30000, 3)
    th, ph = port.rng(227).qmf(n)
    d = eng.DeviceSum.upload(host(eng, h))
    e1, g1 = d.qmf_energy_gradient(eng.QmfState(th, ph))
    er, gr = port.qmf_energy_gradient(h, th, ph)
    assert close(e1, er) and np.abs(g1 - gr).max() <= REL * max(1.0, np.abs(gr).max())
    monkeypatch.setenv("IQCC_QMF_GRAD_BINS", "1")
    e2, g2 = d.qmf_energy_gradient(eng.QmfState(th, ph))
    assert close(e2, er) and np.abs(g2 - gr).max() <= REL * max(1.0, np.abs(gr).max())


def test_qmf_gradient_finite_difference(eng, port):  # test_qmf.cpp:68-87
    rng = port.rng(211)
    for _ in range(5):
        h = rng.sum(6, 60)
        th, ph = rng.qmf(6)
        _, g = eng.qmf_energy_gradient(host(eng, h), eng.QmfState(th, ph))
        step = 1e-5
        for j in range(12):
            lo_t, hi_t = th.copy(), th.copy()
            lo_p, hi_p = ph.copy(), ph.copy()
            if j < 6:
                lo_t[j] -= step
                hi_t[j] += step
            else:
                lo_p[j - 6] -= step
                hi_p[j - 6] += step
            fd = (port.expect_sum(hi_t, hi_p, h) - port.expect_sum(lo_t, lo_p, h)) / (2 * step)
            assert abs(g[j] - fd) / max(1.0, abs(fd), abs(g[j])) < 1e-6


def test_gradient_known_answer(eng):  # test_dis.cpp:108-114
    h = eng.PauliSum(1)
    h.append(eng.PauliWord.from_string("X"), 1.0)
    assert eng.gradient(h, eng.QmfState.zeros(1), eng.PauliWord.from_string("Y")) == pytest.approx(1.0)


@pytest.mark.parametrize("n", [5, 64, 124, 200])
def test_gradient_bit_exact(eng, port, monkeypatch, n):
    """DIS gradients at a generic Omega: the factor-ratio kernel (default)
    and the nibble-table kernel (IQCC_DIS_NIB=1) within 1e-13 of the
    reference, the ascending-qubit kernel (IQCC_DIS_EXACT=1) bit for bit."""
    rng = port.rng(419 + n)
    h = rng.sum(n, 2000)
    th, ph = rng.qmf(n)
    d = eng.DeviceSum.upload(host(eng, h))
    cands = np.stack([rng.word(n, False) for _ in range(64)])
    want = np.array([port.gradient(h, th, ph, c) for c in cands])
    g = d.gradients(eng.QmfState(th, ph), cands)
    assert np.abs(g - want).max() <= 1e-13 * max(1.0, np.abs(want).max())
    monkeypatch.setenv("IQCC_DIS_NIB", "1")
    g = d.gradients(eng.QmfState(th, ph), cands)
    assert np.abs(g - want).max() <= 1e-13 * max(1.0, np.abs(want).max())
    monkeypatch.delenv("IQCC_DIS_NIB")
    monkeypatch.setenv("IQCC_DIS_EXACT", "1")
    g = d.gradients(eng.QmfState(th, ph), cands)
    for k in range(len(cands)):
        assert g[k] == want[k]


def test_dis_candidates_random(eng, port):  # test_dis.cpp:231-263 shapes
    rng = port.rng(443)
    for t in range(12):
        n = 4 + t % 5
        h = rng.sum(n, 80)
        th, ph = rng.qmf(n)
        occ = np.where(np.arange(n) % 2 == 0, math.pi, 0.0)
        for thx in (th, occ):
            for k, seed in ((4, None), (100, None), (100, 7)):
                want_rows, want_g = port.dis_candidates(h, thx, ph, k, seed=seed)
                got = eng.dis_candidates(host(eng, h), eng.QmfState(thx, ph), k,
                                         eng.DisOptions(tie_break_seed=seed))
                assert len(got) == len(want_g)
                for p, wr, wg in zip(got, want_rows, want_g):
                    assert np.array_equal(p.word.row, wr) and p.gradient == wg


@pytest.mark.parametrize("name", ["c1_h2_sto3g.npz", "c1_h2_ccpvdz.npz"])
def test_dis_at_hf_golden(eng, name):
    g = load_golden(name)
    n, ne = int(g["n_qubits"]), int(g["n_electrons"])
    h = eng.PauliSum(n, g["rows0"], g["coeffs0"])
    picks = eng.dis_candidates(h, eng.hf_reference([j < ne for j in range(n)]), 1 << 20)
    assert len(picks) == len(g["dis_g"])
    for p, wr, wg in zip(picks, g["dis_rows"], g["dis_g"]):
        assert np.array_equal(p.word.row, wr) and p.gradient == wg


def test_choose_partition_bits(eng, port):  # test_partition.cpp:79-134
    rng = port.rng(607)
    for t in range(6):
        h = rng.sum(8, 150)
        for m in (1, 2, 3):
            bits, imb = eng.choose_partition_bits(host(eng, h), m)
            wb, wi = port.choose_partition_bits(h, m)
            assert bits == list(wb) and imb == pytest.approx(wi, rel=1e-15)
    hm = port.gen_mol(124, 50000, 2)
    d = eng.DeviceSum.generate_mol(124, 50000, 2)
    for m in (1, 2, 3):
        bits, imb = eng.choose_partition_bits(d, m)
        wb, wi = port.choose_partition_bits(hm, m)
        assert bits == list(wb) and imb == pytest.approx(wi, rel=1e-15)


@pytest.mark.parametrize("n,terms,K", [(6, 60, 3), (20, 800, 4), (64, 3000, 5)])
def test_qcc_energy_and_gradient(eng, port, n, terms, K):  # optimizer.hpp:19-77 (test_optimizer.cpp shapes)
    rng = port.rng(613 + n)
    h = rng.sum(n, terms)
    th, ph = rng.qmf(n)
    gens = np.stack([rng.word(n, False) for _ in range(K)])
    taus = [0.31, -0.17, 0.09, 0.23, -0.41][:K]
    ans = eng.Ansatz([eng.PauliWord(n, g) for g in gens], taus)
    om = eng.QmfState(th, ph)
    e = eng.qcc_energy(host(eng, h), om, ans)
    assert close(e, port.qcc_energy(h, th, ph, gens, taus))
    g = eng.qcc_gradient(host(eng, h), om, ans)
    gr = port.qcc_gradient(h, th, ph, gens, taus)
    assert np.abs(g - gr).max() <= REL * max(1.0, np.abs(gr).max())


def test_qcc_gradient_at_zero_is_dis_gradient(eng):
    # optimizer.hpp:50-53: at tau = 0 component k is the DIS screening
    # gradient of generator k (test_optimizer.cpp)
    g = load_golden("c1_h2_ccpvdz.npz")
    n, ne = int(g["n_qubits"]), int(g["n_electrons"])
    h = eng.PauliSum(n, g["rows0"], g["coeffs0"])
    hf = eng.hf_reference([q < ne for q in range(n)])
    picks = eng.dis_candidates(h, hf, 3)
    ans = eng.Ansatz([p.word for p in picks], [0.0] * len(picks))
    grad = eng.qcc_gradient(h, hf, ans)
    for k, p in enumerate(picks):
        assert close(grad[k], p.gradient, 1e-10) or abs(grad[k] - p.gradient) < 1e-12


def _bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def _kernels_equal(ker, ref_tuple):
    hk = np.stack([ker.h_kernel.real.ravel(), ker.h_kernel.imag.ravel()], 1)
    nk = np.stack([ker.n_kernel.real.ravel(), ker.n_kernel.imag.ravel()], 1)
    return (np.array_equal(_bits(hk), _bits(ref_tuple[4][0])) and
            np.array_equal(_bits(nk), _bits(ref_tuple[4][1])))


@pytest.mark.parametrize("seed,n,terms,N,k", [(757, 4, 25, 4, 4), (761, 3, 30, 4, 4), (701, 20, 400, 4, 2),
                                              (703, 64, 1500, 5, 2), (705, 124, 800, 3, 3),
                                              (707, 200, 3000, 6, 2)])
def test_poly_kernels_bit_exact(eng, port, seed, n, terms, N, k):
    # build_poly_kernels (iqcc/optimizer.hpp:340-368): one chunk covers the
    # sum (<= 4096 terms), so every kernel element is bit-identical
    rng = port.rng(seed)
    h = rng.sum(n, terms)
    th, ph = rng.qmf(n)
    ents = np.stack([rng.word(n, False) for _ in range(N)])
    om = eng.QmfState(th, ph)
    ex = eng.build_poly([eng.PauliWord(n, e) for e in ents], om, k)
    ker = eng.build_poly_kernels(host(eng, h), om, ex)
    assert _kernels_equal(ker, port.poly_kernels(h, th, ph, ents, k))


def test_poly_kernels_at_poles_bit_exact(eng, port):
    # sandwich's pole path (optimizer.hpp:295-326) on H2 cc-pVDZ at HF
    g = load_golden("c1_h2_ccpvdz.npz")
    n, ne = int(g["n_qubits"]), int(g["n_electrons"])
    h = port.sum(n, g["rows0"], g["coeffs0"])
    th = np.array([math.pi if j < ne else 0.0 for j in range(n)])
    ph = np.zeros(n)
    rows, _ = port.dis_candidates(h, th, ph, 6)
    om = eng.QmfState(th, ph)
    ex = eng.build_poly([eng.PauliWord(n, r) for r in rows], om, 3)
    ker = eng.build_poly_kernels(host(eng, h), om, ex)
    assert _kernels_equal(ker, port.poly_kernels(h, th, ph, rows, 3))
    e0, nrm = eng.poly_energy_from_kernels(ex, ker, [0.0] * len(rows))
    assert close(e0, port.expect_sum(th, ph, h), 1e-12) and nrm == pytest.approx(1.0, abs=1e-12)


def test_poly_kernels_chunked_large(eng, port):
    # 124 qubits, 60000 G_mol terms: the store is split into chunks summed in
    # order, so elements agree to fp64 reassociation (1e-12 of the row scale)
    n = 124
    hm = port.gen_mol(n, 60000, 3)
    d = eng.DeviceSum.generate_mol(n, 60000, 3)
    rng = port.rng(709)
    th, ph = rng.qmf(n)
    rs = np.random.default_rng(709)  # weight-4 odd-#Y entanglers (dis.hpp:89-116 shape)
    rows = []
    for _ in range(4):
        w = ["I"] * n
        for j, q in enumerate(rs.choice(n, 4, replace=False)):
            w[q] = "Y" if j == 0 else "X"
        rows.append(eng.PauliWord.from_string("".join(w)).row)
    rows = np.stack(rows)
    om = eng.QmfState(th, ph)
    ex = eng.build_poly([eng.PauliWord(n, r) for r in rows], om, 2)
    ker = d.poly_kernels(om, ex)
    _, _, hc, nc, raw = port.poly_kernels(hm, th, ph, rows, 2)
    scale = max(1e-300, np.abs(hc).max())
    assert np.abs(ker.h_kernel - hc).max() <= 1e-12 * scale
    assert np.array_equal(_bits(np.stack([ker.n_kernel.real.ravel(), ker.n_kernel.imag.ravel()], 1)), _bits(raw[1]))
    # exact mode: one chunk, bit-identical to the reference at this size too
    import os
    os.environ["IQCC_POLY_EXACT"] = "1"
    try:
        kx = d.poly_kernels(om, ex)
    finally:
        del os.environ["IQCC_POLY_EXACT"]
    assert _kernels_equal(kx, port.poly_kernels(hm, th, ph, rows, 2))


def test_poly_energy_full_order_is_qcc_energy(eng, port):
    # tests/test_optimizer.cpp:203-216: the untruncated expansion reproduces
    # qcc_energy (both computed on the device)
    rng = port.rng(761)
    for trial in range(6):
        n = 3 + trial % 2
        h = rng.sum(n, 30)
        th, ph = rng.qmf(n)
        ents = [eng.PauliWord(n, rng.word(n, False)) for _ in range(4)]
        taus = [0.3 * (trial + 1), -0.2, 0.45, 0.1]
        om = eng.QmfState(th, ph)
        ex = eng.build_poly(ents, om, 4)
        ker = eng.build_poly_kernels(host(eng, h), om, ex)
        e, _ = eng.poly_energy_from_kernels(ex, ker, taus)
        exact = eng.qcc_energy(host(eng, h), om, eng.Ansatz(ents, taus))
        assert abs(e - exact) <= 1e-12 * max(1.0, abs(exact))


def test_poly_kernels_edge_cases(eng, port):
    # order 0 (t = 1: h_kernel = <H>, n_kernel = 1), an empty sum (h_kernel 0),
    # and the pole path at 200 qubits (B = 4 blocks)
    rng = port.rng(719)
    n = 12
    h = rng.sum(n, 80)
    th, ph = rng.qmf(n)
    ents = np.stack([rng.word(n, False) for _ in range(3)])
    om = eng.QmfState(th, ph)
    ex0 = eng.build_poly([eng.PauliWord(n, e) for e in ents], om, 0)
    ker = eng.build_poly_kernels(host(eng, h), om, ex0)
    assert ker.t == 1 and _kernels_equal(ker, port.poly_kernels(h, th, ph, ents, 0))
    ex = eng.build_poly([eng.PauliWord(n, e) for e in ents], om, 2)
    kz = eng.build_poly_kernels(eng.PauliSum(n), om, ex)
    assert not np.any(kz.h_kernel) and np.array_equal(kz.n_kernel, ker_n(eng, port, n, th, ph, ents))
    with pytest.raises(ValueError):
        eng.build_poly([eng.PauliWord(n)], om, 1)  # identity entangler
    n = 200
    hm = port.gen_mol(n, 3000, 4)
    d = eng.DeviceSum.generate_mol(n, 3000, 4)
    th = np.array([math.pi if q % 4 == 0 else 0.0 for q in range(n)])
    ph = np.zeros(n)
    rows, _ = port.dis_candidates(hm, th, ph, 4)
    om = eng.QmfState(th, ph)
    ex = eng.build_poly([eng.PauliWord(n, r) for r in rows], om, 2)
    assert _kernels_equal(d.poly_kernels(om, ex), port.poly_kernels(hm, th, ph, rows, 2))


def ker_n(eng, port, n, th, ph, ents):
    z = port.sum(n, np.zeros((0, 2 * eng.blocks_for(n)), np.uint64), np.zeros(0, np.complex128))
    return port.poly_kernels(z, th, ph, ents, 2)[3]


def test_c4_shape_gradients_bit_exact(eng, port, monkeypatch):
    """SURVEY.md §8(d) C4 shape: G_mol(100 qubits, seed 3) against odd-Y
    candidates (seed 4) at a generic Omega and, flip-group restricted, at HF
    poles.  Gradients are summed in canonical order like the reference's
    gradient / group_gradient (dis.hpp:39-52, 121-132): bit-exact.  1e6 terms
    here (the checker's pace); bench_aux runs the config's 1e7 x 1e5."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench_aux import odd_y_candidates
    n, terms = 100, 1_000_000
    h = port.gen_mol(n, terms, 3)
    d = eng.DeviceSum.generate_mol(n, terms, 3)
    cands = odd_y_candidates(n, 64, 4)
    rs = np.random.default_rng(9)
    th, ph = rs.uniform(-3, 3, n), rs.uniform(-3, 3, n)
    sel = [0, 1, 9, 17, 40, 63]
    want = {k: port.gradient(h, th, ph, cands[k]) for k in sel}
    g = d.gradients(eng.QmfState(th, ph), cands)  # factor ratios (default)
    for k in sel:
        assert abs(g[k] - want[k]) <= 1e-13 * max(1.0, abs(want[k])), k
    monkeypatch.setenv("IQCC_DIS_EXACT", "1")  # ascending-qubit products: bit-exact
    g = d.gradients(eng.QmfState(th, ph), cands)
    for k in sel:
        assert g[k] == want[k], k
    monkeypatch.delenv("IQCC_DIS_EXACT")
    thp = np.where(np.arange(n) < n // 4, np.pi, 0.0)
    gp = d.gradients(eng.QmfState(thp, np.zeros(n)), cands, flip_group_only=True)
    for k in sel:  # exact at the poles (every other term's contribution vanishes)
        assert abs(gp[k] - port.gradient(h, thp, np.zeros(n), cands[k])) <= 1e-12 * max(1.0, abs(gp[k]))
