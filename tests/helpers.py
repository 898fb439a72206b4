"""Test helpers: converters between the checker (oracle/) and the engine's
host containers, and an independent dense numpy oracle for small n (the
role Eigen plays in the reference tests, tests/helpers.hpp:19-72)."""
import hashlib
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

_I = np.eye(2, dtype=complex)
_X = np.array([[0, 1], [1, 0]], dtype=complex)
_Y = np.array([[0, -1j], [1j, 0]], dtype=complex)
_Z = np.array([[1, 0], [0, -1]], dtype=complex)
_LET = {"I": _I, "X": _X, "Y": _Y, "Z": _Z}


def blocks_for(n):
    return 1 if n == 0 else (n + 63) // 64


def letters(row, n):
    B = blocks_for(n)
    out = []
    for j in range(n):
        x = (int(row[j // 64]) >> (j % 64)) & 1
        z = (int(row[B + j // 64]) >> (j % 64)) & 1
        out.append("IXZY"[x | (z << 1)])
    return "".join(out)


def word_matrix(row, n):
    """Qubit 0 is the least significant basis bit (tests/helpers.hpp:44-49)."""
    m = np.eye(1, dtype=complex)
    s = letters(row, n)
    for j in range(n - 1, -1, -1):
        m = np.kron(m, _LET[s[j]])
    return m


def sum_matrix(rows, coeffs, n):
    d = 1 << n
    m = np.zeros((d, d), dtype=complex)
    for r, c in zip(rows, coeffs):
        m += c * word_matrix(r, n)
    return m


def dense_dressed(rows, coeffs, n, gen, tau):
    """e^{i tau/2 P} H e^{-i tau/2 P} (tests/test_dressing.cpp:15-22)."""
    p = word_matrix(gen, n)
    u = np.cos(tau / 2) * np.eye(1 << n) + 1j * np.sin(tau / 2) * p
    return u @ sum_matrix(rows, coeffs, n) @ u.conj().T


def to_host(osum):
    """Checker sum -> (n, rows, coeffs)."""
    r, c = osum.export()
    return osum.n_qubits, r, c


def digest(rows, coeffs):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(rows, np.uint64).tobytes())
    # values, not bit patterns: -0.0 and +0.0 (e.g. imaginary parts produced
    # by the reference's complex arithmetic) compare equal, as in PauliSum ==
    h.update((np.ascontiguousarray(coeffs, np.complex128).view(np.float64) + 0.0).tobytes())
    return h.hexdigest()


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


def same(a_rows, a_coeffs, b_rows, b_coeffs):
    return (a_rows.shape == b_rows.shape and np.array_equal(a_rows, b_rows)
            and np.array_equal(a_coeffs, b_coeffs))
