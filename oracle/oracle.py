"""ctypes front-end for the CPU checkers in oracle/ (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's CPU arm import this
module.  It wraps either flavour of oracle_api.h:

* ``Oracle("port")``      -> oracle/liboracle.so, our restatement
  (iqcc_oracle.cpp) of the reference algorithms;
* ``Oracle("reference")`` -> oracle/_ref/libiqcc_ref.so, the unmodified
  reference headers compiled here (absent on machines without
  /root/reference; ``Oracle.available("reference")`` says so).

Sums cross the boundary in the reference storage layout
(iqcc/pauli.hpp:373-377): rows ``uint64[M, 2B]`` (x blocks then z blocks),
coefficients ``complex128[M]``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {
    "port": os.path.join(HERE, "liboracle.so"),
    "reference": os.path.join(HERE, "_ref", "libiqcc_ref.so"),
}

_u64p = C.POINTER(C.c_uint64)
_f64p = C.POINTER(C.c_double)
_szp = C.POINTER(C.c_size_t)
_vp = C.c_void_p


def blocks_for(n: int) -> int:
    return 1 if n == 0 else (n + 63) // 64


def build(flavor: str = "port") -> None:
    """(Re)build a checker with oracle/Makefile (gcc; no GPU needed)."""
    target = PATHS[flavor]
    rule = target if flavor == "port" else "ref"
    subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile"), rule], check=True,
                   cwd=os.path.dirname(HERE))


def _p(a, t):
    return a.ctypes.data_as(t)


class OracleError(Exception):
    pass


class Oracle:
    _cache: dict = {}

    @staticmethod
    def available(flavor: str) -> bool:
        return os.path.exists(PATHS[flavor])

    def __new__(cls, flavor: str = "port"):
        if flavor in cls._cache:
            return cls._cache[flavor]
        path = PATHS[flavor]
        if not os.path.exists(path):
            if flavor == "port":
                build("port")
            else:
                raise FileNotFoundError(f"{path} not built (needs /root/reference)")
        self = super().__new__(cls)
        self.flavor = flavor
        self.lib = lib = C.CDLL(path)
        sig = {
            "orc_last_error": (C.c_char_p, []),
            "orc_last_error_kind": (C.c_int, []),
            "orc_flavor": (C.c_char_p, []),
            "orc_sum_new": (_vp, [C.c_size_t, _u64p, _f64p, C.c_size_t]),
            "orc_from_terms": (_vp, [C.c_size_t, _u64p, _f64p, C.c_size_t, C.c_double, C.c_int, C.c_double]),
            "orc_sum_free": (None, [_vp]),
            "orc_sum_size": (C.c_size_t, [_vp]),
            "orc_sum_qubits": (C.c_size_t, [_vp]),
            "orc_sum_export": (None, [_vp, _u64p, _f64p]),
            "orc_sum_is_canonical": (C.c_int, [_vp]),
            "orc_canonical_compare": (C.c_int, [C.c_size_t, _u64p, _u64p]),
            "orc_commutes": (C.c_int, [C.c_size_t, _u64p, _u64p]),
            "orc_multiply": (C.c_int, [C.c_size_t, _u64p, _u64p, _u64p]),
            "orc_merge_sums": (_vp, [_vp, _vp, C.c_double, C.c_int, C.c_double]),
            "orc_compress": (_vp, [_vp, C.c_double, C.c_size_t, _szp, _f64p]),
            "orc_dress_single": (_vp, [_vp, _u64p, C.c_double, C.c_double, C.c_int, C.c_double]),
            "orc_sortless_dress": (_vp, [_vp, _u64p, C.c_double, C.c_double, _szp, _szp]),
            "orc_dress_sequence": (_vp, [_vp, C.c_size_t, _u64p, _f64p, C.c_double, C.c_size_t, C.c_double,
                                        _szp, _f64p]),
            "orc_growth_split": (None, [_vp, _u64p, _szp, _szp]),
            "orc_expect_word": (C.c_double, [C.c_size_t, _f64p, _f64p, _u64p]),
            "orc_expect_sum": (C.c_double, [_f64p, _f64p, _vp]),
            "orc_qmf_energy_gradient": (C.c_double, [_vp, _f64p, _f64p, _f64p]),
            "orc_qcc_energy": (C.c_double, [_vp, _f64p, _f64p, C.c_size_t, _u64p, _f64p]),
            "orc_qcc_gradient": (C.c_int, [_vp, _f64p, _f64p, C.c_size_t, _u64p, _f64p, _f64p]),
            "orc_poly_kernels": (C.c_int, [_vp, _f64p, _f64p, C.c_size_t, _u64p, C.c_size_t, C.c_size_t,
                                            _szp, _u64p, C.POINTER(C.c_int), _f64p, _f64p]),
            "orc_gradient": (C.c_double, [_vp, _f64p, _f64p, _u64p]),
            "orc_dis_candidates": (C.c_size_t, [_vp, _f64p, _f64p, C.c_size_t, C.c_double, C.c_size_t,
                                                C.c_int, C.c_uint64, _u64p, _f64p, C.c_size_t]),
            "orc_flip_groups": (C.c_size_t, [_vp, _szp, C.c_size_t]),
            "orc_choose_partition_bits": (C.c_double, [_vp, C.c_size_t, _szp]),
            "orc_parallel_dress": (_vp, [_vp, C.c_size_t, _szp, _szp, C.c_size_t, _u64p, C.c_double,
                                         C.c_double, C.c_size_t, C.c_int, _szp, _szp, C.c_size_t,
                                         _szp, _szp]),
            "orc_parallel_expect": (C.c_double, [_vp, C.c_size_t, _szp, _szp, C.c_size_t, _f64p, _f64p]),
            "orc_rebalance": (C.c_int, [_vp, C.c_size_t, _szp, _szp, C.c_size_t, C.c_double]),
            "orc_rng_new": (_vp, [C.c_uint64]),
            "orc_rng_free": (None, [_vp]),
            "orc_rng_next": (C.c_uint64, [_vp]),
            "orc_rng_uniform": (C.c_double, [_vp, C.c_double, C.c_double]),
            "orc_random_word": (None, [_vp, C.c_size_t, C.c_int, _u64p]),
            "orc_random_sum": (_vp, [_vp, C.c_size_t, C.c_size_t]),
            "orc_random_qmf": (None, [_vp, C.c_size_t, _f64p, _f64p]),
            "orc_gen_mol": (_vp, [C.c_size_t, C.c_size_t, C.c_uint64]),
            "orc_time_dress_sequence": (C.c_double, [_vp, C.c_size_t, _u64p, _f64p, C.c_double,
                                                     C.c_size_t, C.c_size_t, C.c_int, _szp, _szp,
                                                     C.POINTER(_vp)]),
        }
        if flavor == "reference":
            sig.update({
                "orc_ref_jordan_wigner_fcidump": (_vp, [C.c_char_p, _szp]),
                "orc_ref_ground_energy": (C.c_double, [_vp]),
                "orc_ref_parse_pauli_file": (_vp, [C.c_char_p]),
                "orc_ref_write_pauli_file": (C.c_int, [_vp, C.c_char_p]),
                "orc_ref_iqcc_iteration": (_vp, [_vp, _f64p, _f64p, C.c_size_t, C.c_double, C.c_size_t,
                                                 _u64p, _f64p, _szp, _f64p]),
            })
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        cls._cache[flavor] = self
        return self

    # ---------------------------------------------------------------- helpers
    def _raise(self):
        msg = self.lib.orc_last_error().decode()
        kind = self.lib.orc_last_error_kind()
        raise (ValueError if kind == 1 else RuntimeError)(msg)

    def _wrap(self, handle) -> "OSum":
        if not handle:
            self._raise()
        return OSum(self, handle)

    def sum(self, n_qubits: int, rows, coeff) -> "OSum":
        rows = np.ascontiguousarray(rows, dtype=np.uint64).reshape(-1, 2 * blocks_for(n_qubits))
        cf = np.ascontiguousarray(np.asarray(coeff, dtype=np.complex128)).view(np.float64)
        M = rows.shape[0]
        return self._wrap(self.lib.orc_sum_new(n_qubits, _p(rows, _u64p), _p(cf, _f64p), M))

    def from_terms(self, n_qubits, rows, coeff, drop=1e-12, check=True, tol=1e-10) -> "OSum":
        rows = np.ascontiguousarray(rows, dtype=np.uint64).reshape(-1, 2 * blocks_for(n_qubits))
        cf = np.ascontiguousarray(np.asarray(coeff, dtype=np.complex128)).view(np.float64)
        return self._wrap(self.lib.orc_from_terms(n_qubits, _p(rows, _u64p), _p(cf, _f64p),
                                                  rows.shape[0], drop, int(check), tol))

    @staticmethod
    def _row(w):
        return np.ascontiguousarray(w, dtype=np.uint64)

    def dress_single(self, h, gen, tau, drop=1e-12, check=True, tol=1e-10):
        g = self._row(gen)
        return self._wrap(self.lib.orc_dress_single(h.handle, _p(g, _u64p), tau, drop, int(check), tol))

    def sortless_dress(self, h, gen, tau, drop=1e-12):
        g = self._row(gen)
        nb, ns = C.c_size_t(0), C.c_size_t(0)
        out = self._wrap(self.lib.orc_sortless_dress(h.handle, _p(g, _u64p), tau, drop, C.byref(nb), C.byref(ns)))
        return out, {"n_buckets": nb.value, "new_stream_sorts": ns.value}

    def dress_sequence(self, h, gens, taus, eps, max_terms=2**64 - 1, drop=1e-12):
        g = np.ascontiguousarray(gens, dtype=np.uint64)
        t = np.ascontiguousarray(taus, dtype=np.float64)
        dt, dw = C.c_size_t(0), C.c_double(0.0)
        out = self._wrap(self.lib.orc_dress_sequence(h.handle, len(t), _p(g, _u64p), _p(t, _f64p), eps,
                                                     max_terms, drop, C.byref(dt), C.byref(dw)))
        return out, {"dropped_terms": dt.value, "dropped_weight": dw.value}

    def compress(self, h, eps, max_terms):
        dt, dw = C.c_size_t(0), C.c_double(0.0)
        out = self._wrap(self.lib.orc_compress(h.handle, eps, max_terms, C.byref(dt), C.byref(dw)))
        return out, {"dropped_terms": dt.value, "dropped_weight": dw.value}

    def merge_sums(self, a, b, drop=1e-12, check=True, tol=1e-10):
        return self._wrap(self.lib.orc_merge_sums(a.handle, b.handle, drop, int(check), tol))

    def growth_split(self, h, gen):
        g = self._row(gen)
        nc, na = C.c_size_t(0), C.c_size_t(0)
        self.lib.orc_growth_split(h.handle, _p(g, _u64p), C.byref(nc), C.byref(na))
        return nc.value, na.value

    def canonical_compare(self, n, a, b):
        a, b = self._row(a), self._row(b)
        return self.lib.orc_canonical_compare(n, _p(a, _u64p), _p(b, _u64p))

    def commutes(self, n, a, b):
        a, b = self._row(a), self._row(b)
        return bool(self.lib.orc_commutes(n, _p(a, _u64p), _p(b, _u64p)))

    def multiply(self, n, a, b):
        a, b = self._row(a), self._row(b)
        out = np.zeros_like(a)
        t = self.lib.orc_multiply(n, _p(a, _u64p), _p(b, _u64p), _p(out, _u64p))
        return t, out

    def expect_word(self, n, theta, phi, w):
        th, ph, w = np.ascontiguousarray(theta, np.float64), np.ascontiguousarray(phi, np.float64), self._row(w)
        return self.lib.orc_expect_word(n, _p(th, _f64p), _p(ph, _f64p), _p(w, _u64p))

    def expect_sum(self, theta, phi, h):
        th, ph = np.ascontiguousarray(theta, np.float64), np.ascontiguousarray(phi, np.float64)
        return self.lib.orc_expect_sum(_p(th, _f64p), _p(ph, _f64p), h.handle)

    def qmf_energy_gradient(self, h, theta, phi):
        th, ph = np.ascontiguousarray(theta, np.float64), np.ascontiguousarray(phi, np.float64)
        g = np.zeros(2 * h.n_qubits, np.float64)
        e = self.lib.orc_qmf_energy_gradient(h.handle, _p(th, _f64p), _p(ph, _f64p), _p(g, _f64p))
        return e, g

    def qcc_energy(self, h, theta, phi, gens, taus):
        """qcc_energy (iqcc/optimizer.hpp:19-25)."""
        th, ph = np.ascontiguousarray(theta, np.float64), np.ascontiguousarray(phi, np.float64)
        g = np.ascontiguousarray(gens, np.uint64)
        t = np.ascontiguousarray(taus, np.float64)
        return self.lib.orc_qcc_energy(h.handle, _p(th, _f64p), _p(ph, _f64p), len(t), _p(g, _u64p),
                                       _p(t, _f64p))

    def poly_kernels(self, h, theta, phi, ents, k):
        """build_poly + build_poly_kernels (iqcc/optimizer.hpp:219-368).
        Returns (words [t][2B], phases [t], h_kernel [t][t] complex, n_kernel)."""
        th, ph = np.ascontiguousarray(theta, np.float64), np.ascontiguousarray(phi, np.float64)
        B2 = 2 * ((h.n_qubits + 63) // 64 or 1)
        e = np.ascontiguousarray(np.asarray(ents, np.uint64).reshape(-1, B2))
        N = e.shape[0]
        cap, binom = 0, 1
        for j in range(min(k, N) + 1):
            cap += binom
            binom = binom * (N - j) // (j + 1)
        cap = max(cap, 1)
        words = np.zeros((cap, B2), np.uint64)
        phs = np.zeros(cap, np.int32)
        hk = np.zeros((cap * cap, 2), np.float64)
        nk = np.zeros((cap * cap, 2), np.float64)
        t = C.c_size_t(0)
        rc = self.lib.orc_poly_kernels(h.handle, _p(th, _f64p), _p(ph, _f64p), N, _p(e, _u64p), k, cap,
                                       C.byref(t), _p(words, _u64p), phs.ctypes.data_as(C.POINTER(C.c_int)),
                                       _p(hk, _f64p), _p(nk, _f64p))
        if rc != 0:
            raise RuntimeError(self.lib.orc_last_error().decode())
        t = t.value
        hc = hk[: t * t].copy().view(np.complex128).reshape(t, t)  # signed zeros kept
        nc = nk[: t * t].copy().view(np.complex128).reshape(t, t)
        return words[:t], phs[:t], hc, nc, (hk[: t * t].copy(), nk[: t * t].copy())

    def qcc_gradient(self, h, theta, phi, gens, taus):
        """qcc_gradient (iqcc/optimizer.hpp:54-77)."""
        th, ph = np.ascontiguousarray(theta, np.float64), np.ascontiguousarray(phi, np.float64)
        g = np.ascontiguousarray(gens, np.uint64)
        t = np.ascontiguousarray(taus, np.float64)
        out = np.zeros(max(1, len(t)), np.float64)
        rc = self.lib.orc_qcc_gradient(h.handle, _p(th, _f64p), _p(ph, _f64p), len(t), _p(g, _u64p),
                                       _p(t, _f64p), _p(out, _f64p))
        if rc != 0:
            raise RuntimeError(self.lib.orc_last_error().decode())
        return out[: len(t)]

    def gradient(self, h, theta, phi, p):
        th, ph, p = np.ascontiguousarray(theta, np.float64), np.ascontiguousarray(phi, np.float64), self._row(p)
        return self.lib.orc_gradient(h.handle, _p(th, _f64p), _p(ph, _f64p), _p(p, _u64p))

    def dis_candidates(self, h, theta, phi, top_k, thr=1e-8, cap=128, seed=None):
        th, ph = np.ascontiguousarray(theta, np.float64), np.ascontiguousarray(phi, np.float64)
        W = 2 * blocks_for(h.n_qubits)
        cap_out = max(1, min(top_k, max(1, h.size)))
        rows = np.zeros((cap_out, W), np.uint64)
        g = np.zeros(cap_out, np.float64)
        n = self.lib.orc_dis_candidates(h.handle, _p(th, _f64p), _p(ph, _f64p), top_k, thr, cap,
                                        int(seed is not None), seed or 0, _p(rows, _u64p), _p(g, _f64p),
                                        cap_out)
        if n == 2**64 - 1:
            self._raise()
        return rows[:n], g[:n]

    def flip_groups(self, h):
        out = np.zeros(max(1, h.size), np.uintp)
        n = self.lib.orc_flip_groups(h.handle, _p(out, _szp), out.size)
        return out[:n].astype(np.int64)

    def choose_partition_bits(self, h, m):
        bits = np.zeros(max(1, m), np.uintp)
        imb = self.lib.orc_choose_partition_bits(h.handle, m, _p(bits, _szp))
        if imb < 0:
            self._raise()
        return bits[:m].astype(np.int64), imb

    def parallel_dress(self, h, bits, owner, n_workers, gen, tau, eps, max_terms=2**64 - 1, threaded=False):
        m = len(bits)
        b = np.ascontiguousarray(bits, np.uintp)
        o = np.ascontiguousarray(owner, np.uintp)
        g = self._row(gen)
        sizes = np.zeros(1 << m, np.uintp)
        log = np.zeros((max(1, 1 << m), 4), np.uintp)
        nlog, mask = C.c_size_t(0), C.c_size_t(0)
        out = self._wrap(self.lib.orc_parallel_dress(h.handle, m, _p(b, _szp), _p(o, _szp), n_workers,
                                                     _p(g, _u64p), tau, eps, max_terms, int(threaded),
                                                     _p(sizes, _szp), _p(log, _szp), log.shape[0],
                                                     C.byref(nlog), C.byref(mask)))
        return out, sizes.astype(np.int64), log[: nlog.value].astype(np.int64), mask.value

    def parallel_expect(self, h, bits, owner, n_workers, theta, phi):
        b = np.ascontiguousarray(bits, np.uintp)
        o = np.ascontiguousarray(owner, np.uintp)
        th, ph = np.ascontiguousarray(theta, np.float64), np.ascontiguousarray(phi, np.float64)
        return self.lib.orc_parallel_expect(h.handle, len(bits), _p(b, _szp), _p(o, _szp), n_workers,
                                            _p(th, _f64p), _p(ph, _f64p))

    def rebalance(self, h, bits, owner, n_workers, threshold):
        b = np.ascontiguousarray(bits, np.uintp)
        o = np.ascontiguousarray(owner, np.uintp).copy()
        if self.lib.orc_rebalance(h.handle, len(bits), _p(b, _szp), _p(o, _szp), n_workers, threshold) != 0:
            self._raise()
        return o.astype(np.int64)

    def rng(self, seed: int) -> "ORng":
        return ORng(self, seed)

    def gen_mol(self, n, count, seed):
        return self._wrap(self.lib.orc_gen_mol(n, count, seed))

    def time_dress_sequence(self, h, gens, taus, eps, max_terms, m_bits=0, threads=0, want_out=False):
        """Returns (seconds, summed input terms, final size[, final sum])."""
        g = np.ascontiguousarray(gens, dtype=np.uint64)
        t = np.ascontiguousarray(taus, dtype=np.float64)
        tin, fin = C.c_size_t(0), C.c_size_t(0)
        out = _vp(None)
        secs = self.lib.orc_time_dress_sequence(h.handle, len(t), _p(g, _u64p), _p(t, _f64p), eps, max_terms,
                                                m_bits, threads, C.byref(tin), C.byref(fin),
                                                C.byref(out) if want_out else None)
        if want_out:
            return secs, tin.value, fin.value, self._wrap(out.value)
        return secs, tin.value, fin.value

    # reference-only extras -------------------------------------------------
    def jordan_wigner_fcidump(self, path):
        ne = C.c_size_t(0)
        h = self._wrap(self.lib.orc_ref_jordan_wigner_fcidump(path.encode(), C.byref(ne)))
        return h, ne.value

    def parse_pauli_file(self, path):
        return self._wrap(self.lib.orc_ref_parse_pauli_file(path.encode()))

    def write_pauli_file(self, h, path):
        if self.lib.orc_ref_write_pauli_file(h.handle, path.encode()) != 0:
            self._raise()

    def ground_energy(self, h):
        return self.lib.orc_ref_ground_energy(h.handle)

    def iqcc_iteration(self, h, theta, phi, k, eps=0.0, max_terms=2**64 - 1):
        th, ph = np.ascontiguousarray(theta, np.float64), np.ascontiguousarray(phi, np.float64)
        W = 2 * blocks_for(h.n_qubits)
        gens = np.zeros((max(1, k), W), np.uint64)
        taus = np.zeros(max(1, k), np.float64)
        npk, e = C.c_size_t(0), C.c_double(0.0)
        out = self._wrap(self.lib.orc_ref_iqcc_iteration(h.handle, _p(th, _f64p), _p(ph, _f64p), k, eps,
                                                         max_terms, _p(gens, _u64p), _p(taus, _f64p),
                                                         C.byref(npk), C.byref(e)))
        return out, gens[: npk.value], taus[: npk.value], e.value


class OSum:
    """Owning handle to a checker-side PauliSum."""

    def __init__(self, orc: Oracle, handle):
        self.orc, self.handle = orc, handle
        self.n_qubits = orc.lib.orc_sum_qubits(handle)
        self.size = orc.lib.orc_sum_size(handle)

    def __del__(self):
        try:
            self.orc.lib.orc_sum_free(self.handle)
        except Exception:
            pass

    def __len__(self):
        return self.size

    def export(self):
        W = 2 * blocks_for(self.n_qubits)
        rows = np.zeros((self.size, W), np.uint64)
        cf = np.zeros(self.size, np.complex128)
        self.orc.lib.orc_sum_export(self.handle, _p(rows, _u64p), _p(cf.view(np.float64), _f64p))
        return rows, cf

    def is_canonical(self):
        return bool(self.orc.lib.orc_sum_is_canonical(self.handle))


class ORng:
    """std::mt19937_64 living in the checker library (same libstdc++
    distributions as the reference test helpers)."""

    def __init__(self, orc: Oracle, seed: int):
        self.orc = orc
        self.handle = orc.lib.orc_rng_new(seed)

    def __del__(self):
        try:
            self.orc.lib.orc_rng_free(self.handle)
        except Exception:
            pass

    def uniform(self, lo, hi):
        return self.orc.lib.orc_rng_uniform(self.handle, lo, hi)

    def next(self):
        return self.orc.lib.orc_rng_next(self.handle)

    def word(self, n, allow_identity=True):
        out = np.zeros(2 * blocks_for(n), np.uint64)
        self.orc.lib.orc_random_word(self.handle, n, int(allow_identity), _p(out, _u64p))
        return out

    def sum(self, n, max_terms) -> OSum:
        return self.orc._wrap(self.orc.lib.orc_random_sum(self.handle, n, max_terms))

    def qmf(self, n):
        th, ph = np.zeros(n), np.zeros(n)
        self.orc.lib.orc_random_qmf(self.handle, n, _p(th, _f64p), _p(ph, _f64p))
        return th, ph
