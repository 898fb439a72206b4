"""GPU parity of the Pauli text I/O and the FCIDUMP -> Jordan-Wigner ingest
(iqcc/io.hpp:31-101, 154-276) against the unmodified reference's outputs
(tests/golden/io.npz and the fixture files, made by make_golden.py)."""
import os

import numpy as np
import pytest

from helpers import GOLDEN, digest, load_golden

pytestmark = pytest.mark.gpu


def same(got, rows, coeffs):
    return got.rows.shape == rows.shape and np.array_equal(got.rows, rows) and np.array_equal(got.coeffs, coeffs)


def test_parse_reference_written_file(eng):
    g = load_golden("io.npz")
    h = eng.parse_pauli_file(os.path.join(GOLDEN, "io_sum10.txt"))
    assert len(h) == g["n_sum10"]
    assert digest(h.rows, h.coeffs) == g["sha_sum10"] == g["sha_sum10_parsed"]


def test_parse_comments_blank_lines_duplicates(eng):
    g = load_golden("io.npz")
    h = eng.parse_pauli_file(os.path.join(GOLDEN, "io_dups.txt"))
    assert same(h, g["rows_dups"], g["coeffs_dups"])


def test_write_round_trip_is_bit_exact(eng, port, tmp_path):
    """write_pauli_file then parse_pauli_file gives back the same sum bit for
    bit (full-precision decimals), and the text equals what the reference's
    "%.17g <letters>" format produces (Python's %-formatting is correctly
    rounded like glibc printf)."""
    for n, terms, seed in ((10, 300, 71), (124, 200_000, 2), (200, 30_000, 5)):
        h = port.gen_mol(n, terms, seed) if n > 10 else port.rng(seed).sum(n, terms)
        r, c = h.export()
        d = eng.DeviceSum.upload(eng.PauliSum(n, r, c))
        path = str(tmp_path / f"h{n}.txt")
        eng.write_pauli_file(d, path)
        back = eng.parse_pauli_file(path)
        assert same(back, r, c)
        if n <= 124:
            lines = open(path).read().splitlines()
            assert lines[0] == f"# qubits: {n}"
            for i in (0, 1, len(r) // 2, len(r) - 1):
                assert lines[1 + i] == "%.17g %s" % (c[i].real, eng.PauliSum(n, r, c).word(i).to_string())


@pytest.mark.parametrize("body,msg", [
    ("0.5 XXZ\n0.1 XZ\n", ":2: inconsistent string length (expected 3)"),
    ("0.5 XQZ\n", ":1: invalid Pauli letter 'Q'"),
    ("abc XXZ\n", ":1: bad coefficient 'abc'"),
    ("0.5 XXZ extra\n", ":1: trailing content 'extra'"),
    ("inf XXZ\n", ":1: non-finite coefficient"),
    ("0.5\n", ":1: expected `<coefficient> <letters>`"),
])
def test_parse_errors_match_reference(eng, tmp_path, body, msg):
    path = tmp_path / "bad.txt"
    path.write_text(body)
    with pytest.raises(RuntimeError) as e:
        eng.parse_pauli_file(str(path))
    assert str(e.value) == str(path) + msg


def test_empty_files(eng, tmp_path):
    p = tmp_path / "empty.txt"
    p.write_text("# nothing\n")
    with pytest.raises(RuntimeError, match="no terms and no `# qubits:` header"):
        eng.parse_pauli_file(str(p))
    p.write_text("# qubits: 7\n")
    h = eng.parse_pauli_file(str(p))
    assert len(h) == 0 and h.n_qubits == 7
    with pytest.raises(RuntimeError, match="cannot open"):
        eng.parse_pauli_file(str(tmp_path / "missing.txt"))


@pytest.mark.parametrize("name", ["fcidump_4", "fcidump_6"])
def test_jordan_wigner_matches_reference(eng, name):
    """Same Pauli words and term count as the reference's
    jordan_wigner(read_fcidump); coefficients within 1e-12 relative (equal
    words are combined in emission order; the reference's std::sort leaves
    that order unspecified)."""
    g = load_golden("io.npz")
    h, ne = eng.jordan_wigner_fcidump(os.path.join(GOLDEN, f"{name}.txt"))
    assert ne == g[f"nelec_{name}"]
    r, c = g[f"rows_{name}"], g[f"coeffs_{name}"]
    assert h.rows.shape == r.shape and np.array_equal(h.rows, r)
    scale = np.abs(c).max()
    assert np.abs(h.coeffs - c).max() <= 1e-12 * scale
    # and the JW sum is a working device input: dress it, energies agree
    om = eng.QmfState(np.where(np.arange(h.n_qubits) < ne, np.pi, 0.0), np.zeros(h.n_qubits))
    e_dev = eng.expect_sum(om, h)
    e_ref = eng.expect_sum(om, eng.PauliSum(h.n_qubits, r, c))
    assert abs(e_dev - e_ref) <= 1e-12 * max(1.0, abs(e_ref))


def test_fcidump_errors(eng, tmp_path):
    p = tmp_path / "bad.fcidump"
    p.write_text(" &FCI NELEC=2,\n &END\n")
    with pytest.raises(RuntimeError, match="missing NORB"):
        eng.jordan_wigner_fcidump(str(p))
    p.write_text(" &FCI NORB=2,NELEC=2,\n &END\n0.5 3 1 0 0\n")
    with pytest.raises(RuntimeError, match="orbital index out of range"):
        eng.jordan_wigner_fcidump(str(p))
