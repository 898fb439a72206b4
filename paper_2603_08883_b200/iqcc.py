"""Python mirror of the reference's ``namespace iqcc`` API for the hot path,
backed by the B200 engine (C-ABI in include/iqcc_b200.h).

Names, argument meaning and error behaviour follow the reference headers
(``/root/reference/proj/include/iqcc/*.hpp``): ``ValueError`` stands for
``std::invalid_argument`` and ``RuntimeError`` for ``std::runtime_error``.
Host containers use the reference storage layout (iqcc/pauli.hpp:373-377):
rows ``uint64[M, 2B]`` (x blocks then z blocks, bit j%64 of block j//64 is
qubit j) and ``complex128`` coefficients.  Everything numeric runs on the GPU;
the host only computes ``cos/sin`` of amplitudes and Bloch angles with libm
(``math.cos``/``math.sin`` are glibc's, like ``std::cos``/``std::sin`` in the
reference), so device results are bit-identical to the reference's.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import native
from .native import check, lib

U64_MAX = 2**64 - 1


def blocks_for(n_qubits: int) -> int:
    """iqcc/pauli.hpp:21-23."""
    return 1 if n_qubits == 0 else (n_qubits + 63) // 64


def _addr(a: np.ndarray) -> int:
    return a.ctypes.data


# ---------------------------------------------------------------- words
class PauliWord:
    """A Pauli word as one reference row (x blocks then z blocks)."""

    __slots__ = ("n_qubits", "row")

    def __init__(self, n_qubits: int, row=None):
        self.n_qubits = n_qubits
        B = blocks_for(n_qubits)
        self.row = np.zeros(2 * B, np.uint64) if row is None else np.array(row, dtype=np.uint64).reshape(2 * B)

    @staticmethod
    def from_string(letters: str) -> "PauliWord":
        """PauliWord::from_string, iqcc/pauli.hpp:50-65."""
        w = PauliWord(len(letters))
        B = blocks_for(len(letters))
        for j, ch in enumerate(letters):
            bit = np.uint64(1 << (j % 64))
            if ch == "I":
                continue
            if ch not in "XYZ":
                raise ValueError(f"invalid Pauli letter '{ch}'")
            if ch in "XY":
                w.row[j // 64] |= bit
            if ch in "ZY":
                w.row[B + j // 64] |= bit
        return w

    def letter(self, j: int) -> str:
        B = blocks_for(self.n_qubits)
        x = (int(self.row[j // 64]) >> (j % 64)) & 1
        z = (int(self.row[B + j // 64]) >> (j % 64)) & 1
        return "IXZY"[x | (z << 1)]

    def to_string(self) -> str:
        return "".join(self.letter(j) for j in range(self.n_qubits))

    def is_identity(self) -> bool:
        return not self.row.any()

    def __eq__(self, other) -> bool:
        return isinstance(other, PauliWord) and self.n_qubits == other.n_qubits and np.array_equal(self.row, other.row)

    def __repr__(self) -> str:
        return f"PauliWord('{self.to_string()}')"


def multiply(p: PauliWord, q: PauliWord):
    """multiply_into (iqcc/pauli.hpp:202-215): returns (p xor q, t) with
    p*q = i^t (p xor q), t reduced mod 4."""
    B = blocks_for(p.n_qubits)
    t = 0
    for b in range(B):
        px, pz, qx, qz = (int(v) for v in (p.row[b], p.row[B + b], q.row[b], q.row[B + b]))
        rx, rz = px ^ qx, pz ^ qz
        t += (px & pz).bit_count() + (qx & qz).bit_count() - (rx & rz).bit_count() + 2 * (pz & qx).bit_count()
    return PauliWord(p.n_qubits, p.row ^ q.row), t % 4

def _complex_of(pairs: np.ndarray) -> np.ndarray:
    """(re, im) rows -> complex128 with both parts' bits (signed zeros) kept."""
    return np.ascontiguousarray(pairs, np.float64).reshape(-1, 2).view(np.complex128).reshape(-1).copy()

# ------------------------------------------------------------ containers
class PauliSum:
    """Host PauliSum in the reference layout (canonical, duplicate free)."""

    def __init__(self, n_qubits: int, rows=None, coeffs=None):
        self.n_qubits = n_qubits
        W = 2 * blocks_for(n_qubits)
        self.rows = np.zeros((0, W), np.uint64) if rows is None else np.ascontiguousarray(rows, np.uint64).reshape(-1, W)
        self.coeffs = (np.zeros(0, np.complex128) if coeffs is None
                       else np.ascontiguousarray(np.asarray(coeffs, dtype=np.complex128)).reshape(-1))
        if self.rows.shape[0] != self.coeffs.shape[0]:
            raise ValueError("rows / coeffs length mismatch")

    def __len__(self) -> int:
        return self.coeffs.shape[0]

    def size(self) -> int:
        return len(self)

    def word(self, i: int) -> PauliWord:
        return PauliWord(self.n_qubits, self.rows[i])

    def coeff(self, i: int) -> complex:
        return complex(self.coeffs[i])

    def append(self, w: PauliWord, c) -> None:
        """PauliSum::append (caller keeps canonical order)."""
        self.rows = np.vstack([self.rows, w.row[None, :]])
        self.coeffs = np.append(self.coeffs, np.complex128(c))

    def __eq__(self, other) -> bool:
        return (isinstance(other, PauliSum) and self.n_qubits == other.n_qubits
                and np.array_equal(self.rows, other.rows) and np.array_equal(self.coeffs, other.coeffs))

    def to_device(self) -> "DeviceSum":
        return DeviceSum.upload(self)


@dataclass
class DressOp:
    """iqcc/dressing.hpp:15-18."""
    generator: PauliWord
    amplitude: float = 0.0


@dataclass
class Ansatz:
    """iqcc/dressing.hpp:22-31."""
    entanglers: list = field(default_factory=list)
    tau: list = field(default_factory=list)

    def push(self, p: PauliWord, amplitude: float) -> None:
        self.entanglers.append(p)
        self.tau.append(float(amplitude))

    def size(self) -> int:
        return len(self.entanglers)


@dataclass
class MergeOptions:
    """iqcc/pauli.hpp:236-240 (the device path has no imaginary parts, so
    the hermiticity check can never fire; kept for signature parity)."""
    drop_threshold: float = 1e-12
    check_hermitian: bool = True
    hermitian_tol: float = 1e-10


@dataclass
class CompressStats:
    """iqcc/pauli.hpp:417-420."""
    dropped_terms: int = 0
    dropped_weight: float = 0.0


@dataclass
class GrowthSplit:
    n_commuting: int = 0
    n_anticommuting: int = 0

    def bound(self) -> int:
        return self.n_commuting + 2 * self.n_anticommuting


@dataclass
class QmfState:
    """iqcc/qmf.hpp:14-31."""
    theta: np.ndarray
    phi: np.ndarray

    @staticmethod
    def zeros(n: int) -> "QmfState":
        return QmfState(np.zeros(n), np.zeros(n))

    def n_qubits(self) -> int:
        return len(self.theta)

    def at_poles(self, tol: float = 1e-12) -> bool:
        return all(abs(math.sin(float(t))) <= tol for t in self.theta)


def hf_reference(occupations: Sequence[bool]) -> QmfState:
    """iqcc/qmf.hpp:34-39."""
    th = np.array([math.pi if o else 0.0 for o in occupations], np.float64)
    return QmfState(th, np.zeros(len(occupations)))


@dataclass
class DisOptions:
    """iqcc/dis.hpp:60-70."""
    screen_threshold: float = 1e-8
    per_group_cap: int = 128
    tie_break_seed: Optional[int] = None


@dataclass
class RankedGenerator:
    word: PauliWord
    gradient: float


def qmf_factor_table(omega: QmfState) -> np.ndarray:
    """Per-qubit (X, Z, Y) expectations, evaluated exactly as qmf_factor
    (iqcc/qmf.hpp:56-61) with glibc sin/cos."""
    n = omega.n_qubits()
    t = np.zeros((n, 3), np.float64)
    for j in range(n):
        th, ph = float(omega.theta[j]), float(omega.phi[j])
        t[j, 0] = math.sin(th) * math.cos(ph)
        t[j, 1] = math.cos(th)
        t[j, 2] = math.sin(th) * math.sin(ph)
    return t


def qmf_deriv_table(omega: QmfState) -> np.ndarray:
    """Per-qubit (dth_X, dph_X, dth_Z, dph_Z, dth_Y, dph_Y) as in
    qmf_energy_gradient (iqcc/qmf.hpp:130-143)."""
    n = omega.n_qubits()
    t = np.zeros((n, 6), np.float64)
    for j in range(n):
        th, ph = float(omega.theta[j]), float(omega.phi[j])
        st, ct, sp, cp = math.sin(th), math.cos(th), math.sin(ph), math.cos(ph)
        t[j] = (ct * cp, -st * sp, -st, 0.0, ct * sp, st * cp)
    return t


# --------------------------------------------------------- device handle
class DeviceSum:
    """A PauliSum resident in B200 HBM (one shard when partitioned)."""

    def __init__(self, handle: int, n_qubits: int):
        self.handle = handle
        self.n_qubits = n_qubits

    @staticmethod
    def upload(h: PauliSum) -> "DeviceSum":
        native.init()
        out = C.c_void_p()
        rows = np.ascontiguousarray(h.rows, np.uint64)
        cf = np.ascontiguousarray(h.coeffs, np.complex128)
        check(lib.iqcc_gpu_sum_create(h.n_qubits, _addr(rows), _addr(cf), len(h), C.byref(out)))
        return DeviceSum(out.value, h.n_qubits)

    @staticmethod
    def generate_mol(n_qubits: int, n_terms: int, seed: int) -> "DeviceSum":
        native.init()
        out = C.c_void_p()
        check(lib.iqcc_gpu_sum_generate_mol(n_qubits, n_terms, seed, C.byref(out)))
        return DeviceSum(out.value, n_qubits)

    def clone(self) -> "DeviceSum":
        out = C.c_void_p()
        check(lib.iqcc_gpu_sum_clone(self.handle, C.byref(out)))
        return DeviceSum(out.value, self.n_qubits)

    def __del__(self):
        try:
            if self.handle:
                lib.iqcc_gpu_sum_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def size(self) -> int:
        n = C.c_size_t()
        check(lib.iqcc_gpu_sum_size(self.handle, C.byref(n)))
        return n.value

    def __len__(self) -> int:
        return self.size()

    def download(self, rows: np.ndarray | None = None, coeffs: np.ndarray | None = None) -> PauliSum:
        n = self.size()
        W = 2 * blocks_for(self.n_qubits)
        if rows is None:
            rows = np.empty((max(n, 1), W), np.uint64)
            coeffs = np.empty(max(n, 1), np.complex128)
        got = C.c_size_t()
        check(lib.iqcc_gpu_sum_download(self.handle, _addr(rows), _addr(coeffs), rows.shape[0], C.byref(got)))
        return PauliSum(self.n_qubits, rows[: got.value], coeffs[: got.value])

    # ---- hot path, in place
    def dress(self, gen: PauliWord, tau: float, drop_threshold: float = 1e-12) -> DressStats:
        g = np.ascontiguousarray(gen.row, np.uint64)
        st = native.DressStats()
        check(lib.iqcc_gpu_dress(self.handle, _addr(g), math.cos(tau), math.sin(tau), drop_threshold, C.byref(st)))
        return st

    def compress(self, eps: float, max_terms: int = U64_MAX, stats: CompressStats | None = None) -> None:
        cs = native.CompressStatsC()
        check(lib.iqcc_gpu_compress(self.handle, eps, max_terms, C.byref(cs)))
        if stats is not None:
            stats.dropped_terms += cs.dropped_terms
            stats.dropped_weight += cs.dropped_weight

    def dress_sequence(self, ansatz: Ansatz, eps: float, max_terms: int = U64_MAX,
                       stats: CompressStats | None = None, opts: MergeOptions | None = None) -> int:
        """In place dress_sequence; returns the summed logical input size of
        the K dressing steps (the bench metric's unit of work).  opts: the
        MergeOptions every step merges with (dressing.hpp:319)."""
        drop = (opts or MergeOptions()).drop_threshold
        K = ansatz.size()
        W = 2 * blocks_for(self.n_qubits)
        gens = np.zeros((max(K, 1), W), np.uint64)
        for k, p in enumerate(ansatz.entanglers):
            gens[k] = p.row
        cs_ = np.array([math.cos(t) for t in ansatz.tau] or [1.0])
        sn_ = np.array([math.sin(t) for t in ansatz.tau] or [0.0])
        st = native.CompressStatsC()
        tin = C.c_size_t(0)
        check(lib.iqcc_gpu_dress_sequence(self.handle, K, _addr(gens), _addr(cs_), _addr(sn_), eps, max_terms,
                                          drop, C.byref(st) if stats is not None else None, C.byref(tin)))
        if stats is not None:
            stats.dropped_terms += st.dropped_terms
            stats.dropped_weight += st.dropped_weight
        return tin.value

    def download_pinned(self) -> PauliSum:
        """Download into page-locked host memory (fast DMA; bench e2e input)."""
        rows, coeffs = pinned_buffers(self.n_qubits, self.size())
        return self.download(rows, coeffs)

    def growth_split(self, p: PauliWord) -> GrowthSplit:
        g = np.ascontiguousarray(p.row, np.uint64)
        nc, na = C.c_size_t(), C.c_size_t()
        check(lib.iqcc_gpu_growth_split(self.handle, _addr(g), C.byref(nc), C.byref(na)))
        return GrowthSplit(nc.value, na.value)

    def expect(self, omega: QmfState) -> float:
        t = qmf_factor_table(omega)
        e = C.c_double()
        check(lib.iqcc_gpu_expect(self.handle, _addr(t), C.byref(e)))
        return e.value

    def qmf_energy_gradient(self, omega: QmfState):
        t, d = qmf_factor_table(omega), qmf_deriv_table(omega)
        g = np.zeros(2 * self.n_qubits, np.float64)
        e = C.c_double()
        check(lib.iqcc_gpu_qmf_energy_gradient(self.handle, _addr(t), _addr(d), C.byref(e), _addr(g)))
        return e.value, g

    def _ansatz_arrays(self, ansatz: "Ansatz"):
        K = ansatz.size()
        W = 2 * blocks_for(self.n_qubits)
        gens = np.zeros((max(K, 1), W), np.uint64)
        for k, p in enumerate(ansatz.entanglers):
            gens[k] = p.row
        cs_ = np.array([math.cos(t) for t in ansatz.tau] or [1.0])
        sn_ = np.array([math.sin(t) for t in ansatz.tau] or [0.0])
        return K, gens, cs_, sn_

    def qcc_energy(self, omega: QmfState, ansatz: "Ansatz") -> float:
        """qcc_energy (iqcc/optimizer.hpp:19-25) on a device copy; the sum is unchanged."""
        K, gens, cs_, sn_ = self._ansatz_arrays(ansatz)
        t = qmf_factor_table(omega)
        e = C.c_double()
        check(lib.iqcc_gpu_qcc_energy(self.handle, K, _addr(gens), _addr(cs_), _addr(sn_), _addr(t), C.byref(e)))
        return e.value

    def qcc_gradient(self, omega: QmfState, ansatz: "Ansatz") -> np.ndarray:
        """qcc_gradient (iqcc/optimizer.hpp:54-77): dE/dtau_k for every entangler."""
        K, gens, cs_, sn_ = self._ansatz_arrays(ansatz)
        t = qmf_factor_table(omega)
        g = np.zeros(max(K, 1), np.float64)
        check(lib.iqcc_gpu_qcc_gradient(self.handle, K, _addr(gens), _addr(cs_), _addr(sn_), _addr(t), _addr(g)))
        return g[:K]

    def gradients(self, omega: QmfState, cands: np.ndarray, flip_group_only: bool = False) -> np.ndarray:
        t = qmf_factor_table(omega)
        c = np.ascontiguousarray(cands, np.uint64).reshape(-1, 2 * blocks_for(self.n_qubits))
        g = np.zeros(max(1, c.shape[0]), np.float64)
        check(lib.iqcc_gpu_gradients(self.handle, _addr(t), _addr(c), c.shape[0], int(flip_group_only), _addr(g)))
        return g[: c.shape[0]]


    def poly_kernels(self, omega: QmfState, ex: "PolyExpansion", partitioned: bool = False) -> "PolyKernels":
        """build_poly_kernels (iqcc/optimizer.hpp:340-368) against this sum
        (partitioned: the PartitionedSum overload, :371-422, a collective)."""
        t = len(ex.subsets)
        words = np.ascontiguousarray(np.stack([s.word.row for s in ex.subsets]) if t else
                                     np.zeros((1, 2 * blocks_for(self.n_qubits)), np.uint64))
        hk = np.zeros((max(t, 1) ** 2, 2), np.float64)
        nk = np.zeros((max(t, 1) ** 2, 2), np.float64)
        tab = qmf_factor_table(omega)  # kept alive across the call
        fn = lib.iqcc_gpu_parallel_poly_kernels if partitioned else lib.iqcc_gpu_poly_kernels
        check(fn(self.handle, _addr(tab), int(omega.at_poles()), _addr(words), t, _addr(hk), _addr(nk)))
        return PolyKernels(t, _complex_of(hk[: t * t]).reshape(t, t), _complex_of(nk[: t * t]).reshape(t, t))

def pinned_buffers(n_qubits: int, n_terms: int):
    """Page-locked host arrays (rows uint64[n, 2B], coeffs complex128[n])."""
    import torch
    W = 2 * blocks_for(n_qubits)
    n = max(1, n_terms)
    r = torch.empty((n, W), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
    c = torch.empty((n, 2), dtype=torch.float64, pin_memory=True).numpy().view(np.complex128).reshape(n)
    return r, c


# ----------------------------------------------- reference-shaped functions
def _dressed_copy(h: PauliSum) -> DeviceSum:
    return DeviceSum.upload(h)


def dress_single(h: PauliSum, op: DressOp, opts: MergeOptions = MergeOptions()) -> PauliSum:
    """iqcc/dressing.hpp:197-220."""
    if h.n_qubits != op.generator.n_qubits:
        raise ValueError("dress_single: mismatched qubit counts")
    if op.generator.is_identity():
        raise ValueError("dress_single: identity generator")
    d = DeviceSum.upload(h)
    d.dress(op.generator, op.amplitude, opts.drop_threshold)
    return d.download()


@dataclass
class SortlessStats:
    n_buckets: int = 0
    new_term_streams: int = 0
    new_stream_sorts: int = 0
    merge_comparisons: int = 0


def sortless_dress(h: PauliSum, op: DressOp, opts: MergeOptions = MergeOptions(),
                   stats: SortlessStats | None = None) -> PauliSum:
    """iqcc/dressing.hpp:228-307.  Same sum as dress_single (the device path
    never sorts products); keeps the reference's limit of 64 key bits on the
    entangler support (bucket_by_support, dressing.hpp:163-165)."""
    if h.n_qubits != op.generator.n_qubits:
        raise ValueError("sortless_dress: mismatched qubit counts")
    if op.generator.is_identity():
        raise ValueError("sortless_dress: identity generator")
    B = blocks_for(h.n_qubits)
    support = sum(bin(int(op.generator.row[b]) | int(op.generator.row[B + b])).count("1") for b in range(B))
    if 2 * support > 64:
        raise RuntimeError("entangler support exceeds 64 bits; not supported")
    d = DeviceSum.upload(h)
    if stats is not None:
        # support buckets and new-term streams (dressing.hpp:248-268) counted
        # on the device; no product stream is ever sorted; the heap merge's
        # comparison count has no device counterpart (0)
        g = np.ascontiguousarray(op.generator.row, np.uint64)
        nb, ns = C.c_size_t(), C.c_size_t()
        check(lib.iqcc_gpu_sortless_stats(d.handle, _addr(g), math.sin(op.amplitude), C.byref(nb), C.byref(ns)))
        stats.n_buckets, stats.new_term_streams = nb.value, ns.value
        stats.new_stream_sorts, stats.merge_comparisons = 0, 0
    d.dress(op.generator, op.amplitude, opts.drop_threshold)
    return d.download()


def dress_sequence(h: PauliSum, ansatz: Ansatz, epsilon: float, max_terms: int = U64_MAX,
                   stats: CompressStats | None = None, opts: MergeOptions = MergeOptions(),
                   out: tuple | None = None) -> PauliSum:
    """iqcc/dressing.hpp:311-324 (device resident across the whole ansatz).
    `out` optionally supplies host (rows, coeffs) buffers for the result."""
    return dress_sequence_counted(h, ansatz, epsilon, max_terms, stats, out, opts)[0]


def dress_sequence_counted(h: PauliSum, ansatz: Ansatz, epsilon: float, max_terms: int = U64_MAX,
                           stats: CompressStats | None = None, out: tuple | None = None,
                           opts: MergeOptions = MergeOptions()):
    """dress_sequence that also returns the summed logical input size."""
    if max_terms < 1:
        raise ValueError("dress_sequence: max_terms < 1")
    d = DeviceSum.upload(h)
    tin = d.dress_sequence(ansatz, epsilon, max_terms, stats, opts)
    if out is None:
        n = d.size()
        rows, coeffs = (pinned_buffers(h.n_qubits, n) if _is_pinned(h) else (None, None))
    else:
        rows, coeffs = out
    return d.download(rows, coeffs), tin


def _is_pinned(h: PauliSum) -> bool:
    try:
        import torch
        return torch.from_numpy(h.rows.view(np.int64)).is_pinned()
    except Exception:
        return False


def compress(h: PauliSum, epsilon: float, max_terms: int, stats: CompressStats | None = None) -> PauliSum:
    """iqcc/pauli.hpp:425-474."""
    if epsilon < 0:
        raise ValueError("compress: epsilon < 0")
    if max_terms < 1:
        raise ValueError("compress: max_terms < 1")
    d = DeviceSum.upload(h)
    d.compress(epsilon, max_terms, stats)
    return d.download()


def growth_split(h: PauliSum, p: PauliWord) -> GrowthSplit:
    """iqcc/dressing.hpp:41-50."""
    return DeviceSum.upload(h).growth_split(p)


def expect_sum(omega: QmfState, h: PauliSum) -> float:
    """iqcc/qmf.hpp:83-90."""
    if len(h) and h.n_qubits != omega.n_qubits():
        raise ValueError("expect_sum: mismatched qubit counts")
    return DeviceSum.upload(h).expect(omega)


def qmf_energy_gradient(h: PauliSum, omega: QmfState):
    """iqcc/qmf.hpp:94-148; returns (energy, grad[2n])."""
    return DeviceSum.upload(h).qmf_energy_gradient(omega)


def qcc_energy(h: PauliSum, omega: QmfState, ansatz: Ansatz) -> float:
    """iqcc::qcc_energy (iqcc/optimizer.hpp:19-25)."""
    if len(h) == 0:
        return 0.0
    return DeviceSum.upload(h).qcc_energy(omega, ansatz)


def qcc_gradient(h: PauliSum, omega: QmfState, ansatz: Ansatz) -> np.ndarray:
    """iqcc::qcc_gradient (iqcc/optimizer.hpp:54-77)."""
    if len(h) == 0:
        return np.zeros(ansatz.size())
    return DeviceSum.upload(h).qcc_gradient(omega, ansatz)


def gradient(h: PauliSum, omega: QmfState, p: PauliWord) -> float:
    """iqcc/dis.hpp:39-52."""
    return float(DeviceSum.upload(h).gradients(omega, p.row[None, :])[0])


def dis_candidates(h: PauliSum, omega: QmfState, top_k: int, opts: DisOptions = DisOptions()) -> list:
    """iqcc/dis.hpp:140-191 (seeded tie shuffle included, same generator)."""
    if top_k < 1:
        raise ValueError("dis_candidates: top_k < 1")
    return DeviceSum.upload(h).dis_candidates(omega, top_k, opts)


def _dis_on(d: "DeviceSum", omega: QmfState, top_k: int, opts: DisOptions) -> list:
    t = qmf_factor_table(omega)
    W = 2 * blocks_for(d.n_qubits)
    n = C.c_size_t()
    seed = opts.tie_break_seed
    args = (d.handle, _addr(t), int(omega.at_poles()), top_k, opts.screen_threshold, opts.per_group_cap,
            int(seed is not None), seed or 0)
    check(lib.iqcc_gpu_dis_candidates(*args, None, None, 0, C.byref(n)))
    cap = max(1, min(n.value, top_k))
    rows = np.zeros((cap, W), np.uint64)
    g = np.zeros(cap, np.float64)
    check(lib.iqcc_gpu_dis_candidates(*args, _addr(rows), _addr(g), cap, C.byref(n)))
    k = min(n.value, top_k)
    return [RankedGenerator(PauliWord(d.n_qubits, rows[i]), float(g[i])) for i in range(k)]


DeviceSum.dis_candidates = lambda self, omega, top_k, opts=DisOptions(): _dis_on(self, omega, top_k, opts)


# ------------------------------------------- Pauli text files, FCIDUMP ingest
def _device_of(out: C.c_void_p, n_qubits_hint: int = 0) -> DeviceSum:
    n = C.c_size_t()
    check(lib.iqcc_gpu_sum_qubits(out, C.byref(n)))
    return DeviceSum(out.value, n.value)


def read_pauli_file_device(path: str) -> DeviceSum:
    """parse_pauli_file (iqcc/io.hpp:31-87) into a device sum."""
    native.init()
    out = C.c_void_p()
    check(lib.iqcc_gpu_read_pauli_file(str(path).encode(), C.byref(out)))
    return _device_of(out)


def parse_pauli_file(path: str) -> PauliSum:
    """iqcc/io.hpp:31-87: same grammar and "path:line: ..." errors (RuntimeError)."""
    return read_pauli_file_device(path).download()


def write_pauli_file(h, path: str) -> None:
    """iqcc/io.hpp:90-101 ("# qubits: N", then "%.17g <letters>" per term)."""
    d = h if isinstance(h, DeviceSum) else DeviceSum.upload(h)
    check(lib.iqcc_gpu_write_pauli_file(d.handle, str(path).encode()))


def jordan_wigner_fcidump(path: str, device: bool = False):
    """jordan_wigner(read_fcidump(path)) (iqcc/io.hpp:154-276) built on the
    device; returns (sum, n_electrons) (a DeviceSum when device=True)."""
    native.init()
    out, ne = C.c_void_p(), C.c_size_t()
    check(lib.iqcc_gpu_jordan_wigner_fcidump(str(path).encode(), C.byref(ne), C.byref(out)))
    d = _device_of(out)
    return (d if device else d.download()), ne.value


def choose_partition_bits(h, m: int):
    """iqcc/partition.hpp:52-108 on the device; returns (bits, imbalance)."""
    d = h if isinstance(h, DeviceSum) else DeviceSum.upload(h)
    bits = np.zeros(max(1, m), np.uintp)
    imb = C.c_double()
    check(lib.iqcc_gpu_choose_partition_bits(d.handle, m, _addr(bits), C.byref(imb)))
    return [int(b) for b in bits[:m]], imb.value


# ------------------------------------------------ bit-wise partitioning
class Partition:
    """One shard per rank under the paper's bit-wise partitioning
    (iqcc/partition.hpp:20-123), one process per GPU.

    ``setup`` picks m = log2(world) partition bits with the greedy
    choose_partition_bits on the full Hamiltonian (deterministic, so every
    rank agrees), assigns partition p to rank p (make_partition_map's
    round robin with 2^m == world), keeps only the local shard, and joins
    the engine's NCCL communicator (unique id broadcast with
    torch.distributed).  ``dress`` is one parallel_dress step; products whose
    partition key flips are exchanged pairwise with the rank owning p ^ mask.
    """

    def __init__(self, n_qubits, bits, owner, rank, world):
        self.n_qubits, self.bits, self.owner = n_qubits, list(bits), list(owner)
        self.rank, self.world, self.m = rank, world, len(bits)
        b0 = self.bits[0] if self.bits else None
        # the qubit/plane of the first partition bit (entanglers that put a
        # z (x) letter there flip it)
        self.flip_qubit = None if b0 is None else (b0 if b0 < n_qubits else b0 - n_qubits)
        self.flip_plane = None if b0 is None else ("x" if b0 < n_qubits else "z")

    @staticmethod
    def init_comm(rank: int, world: int) -> None:
        import torch.distributed as dist
        uid = (C.c_char * 128)()
        if rank == 0:
            check(lib.iqcc_gpu_nccl_unique_id(uid))
        obj = [bytes(uid) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        buf = (C.c_char * 128).from_buffer_copy(obj[0])
        check(lib.iqcc_gpu_comm_init(buf, rank, world))

    @staticmethod
    def setup(d: DeviceSum, world: int, rank: int) -> "Partition":
        m = world.bit_length() - 1
        if 1 << m != world:
            raise ValueError("Partition: world size must be a power of two (one shard per rank)")
        bits, _ = choose_partition_bits(d, m)
        owner = list(range(1 << m))
        p = Partition(d.n_qubits, bits, owner, rank, world)
        p.restrict(d)
        Partition.init_comm(rank, world)
        return p

    def restrict(self, d: DeviceSum) -> None:
        b = np.array(self.bits or [0], np.uintp)
        o = np.array(self.owner, np.uintp)
        check(lib.iqcc_gpu_sum_restrict(d.handle, self.m, _addr(b), _addr(o), self.rank))

    def dress(self, d: DeviceSum, gen: PauliWord, tau: float, eps: float, max_terms: int = U64_MAX,
              stats: CompressStats | None = None):
        b = np.array(self.bits or [0], np.uintp)
        o = np.array(self.owner, np.uintp)
        g = np.ascontiguousarray(gen.row, np.uint64)
        xs = native.ExchangeStats()
        cs = native.CompressStatsC()
        check(lib.iqcc_gpu_parallel_dress(d.handle, self.m, _addr(b), _addr(o), _addr(g), math.cos(tau),
                                          math.sin(tau), eps, max_terms, C.byref(xs), C.byref(cs)))
        if stats is not None:
            stats.dropped_terms += cs.dropped_terms
            stats.dropped_weight += cs.dropped_weight
        return xs

    def dress_sequence(self, d: DeviceSum, ansatz: Ansatz, eps: float, max_terms: int = U64_MAX,
                       stats: CompressStats | None = None, exchange: list | None = None) -> int:
        """dress_sequence over parallel_dress steps; returns the logical input
        size summed over the steps and all ranks.  `exchange` (optional list)
        receives one ExchangeStats per entangler."""
        K = ansatz.size()
        b = np.array(self.bits or [0], np.uintp)
        o = np.array(self.owner, np.uintp)
        W = 2 * blocks_for(self.n_qubits)
        gens = np.zeros((max(K, 1), W), np.uint64)
        for k, p in enumerate(ansatz.entanglers):
            gens[k] = p.row
        cs_ = np.array([math.cos(t) for t in ansatz.tau] or [1.0])
        sn_ = np.array([math.sin(t) for t in ansatz.tau] or [0.0])
        xs = (native.ExchangeStats * max(K, 1))()
        cst = native.CompressStatsC()
        tin = C.c_size_t(0)
        check(lib.iqcc_gpu_parallel_dress_sequence(d.handle, self.m, _addr(b), _addr(o), K, _addr(gens),
                                                   _addr(cs_), _addr(sn_), eps, max_terms, xs,
                                                   C.byref(cst) if stats is not None else None,
                                                   C.byref(tin)))
        if stats is not None:
            stats.dropped_terms += cst.dropped_terms
            stats.dropped_weight += cst.dropped_weight
        if exchange is not None:
            exchange.extend(xs[k] for k in range(K))
        return tin.value

    def reserve(self, d: DeviceSum, terms: int) -> None:
        """Size the NVLink receive buffers for shards of up to `terms` terms
        (collective), before a run that grows the store uncapped."""
        check(lib.iqcc_gpu_parallel_reserve(d.handle, int(terms)))

    def compress(self, d: DeviceSum, eps: float, max_terms: int = U64_MAX,
                 stats: CompressStats | None = None) -> None:
        """compress_partitioned (iqcc/partition.hpp:325-396) on this rank's
        shard: collective over the communicator."""
        cs = native.CompressStatsC()
        check(lib.iqcc_gpu_parallel_compress(d.handle, eps, max_terms, C.byref(cs)))
        if stats is not None:
            stats.dropped_terms += cs.dropped_terms
            stats.dropped_weight += cs.dropped_weight

    def total_size(self, d: DeviceSum) -> int:
        n = C.c_size_t()
        check(lib.iqcc_gpu_parallel_size(d.handle, C.byref(n)))
        return n.value

    def expect(self, d: DeviceSum, omega: QmfState) -> float:
        t = qmf_factor_table(omega)
        e = C.c_double()
        check(lib.iqcc_gpu_parallel_expect(d.handle, _addr(t), C.byref(e)))
        return e.value

    def poly_kernels(self, d: DeviceSum, omega: QmfState, ex: "PolyExpansion") -> "PolyKernels":
        """Partitioned build_poly_kernels (iqcc/optimizer.hpp:371-422): local
        sandwiches, allgathered over NCCL, summed in worker order.  Collective."""
        return d.poly_kernels(omega, ex, partitioned=True)

    def qmf_energy_gradient(self, d: DeviceSum, omega: QmfState):
        """qmf_energy_gradient (iqcc/qmf.hpp:94-148) of the global sum: each
        rank's energy and 2n gradients, allgathered and summed in rank order
        (reduce_scalar, iqcc/partition.hpp:233-237).  Collective."""
        t, dt = qmf_factor_table(omega), qmf_deriv_table(omega)
        g = np.zeros(2 * self.n_qubits, np.float64)
        e = C.c_double()
        check(lib.iqcc_gpu_parallel_qmf_energy_gradient(d.handle, _addr(t), _addr(dt), C.byref(e), _addr(g)))
        return e.value, g

    def gradients(self, d: DeviceSum, omega: QmfState, cands: np.ndarray, flip_group_only: bool = False):
        """DIS gradients (iqcc/dis.hpp:39-52) of K candidates over the global
        sum: local vectors allgathered and summed in rank order.  Collective."""
        t = qmf_factor_table(omega)
        c = np.ascontiguousarray(cands, np.uint64).reshape(-1, 2 * blocks_for(self.n_qubits))
        g = np.zeros(max(1, c.shape[0]), np.float64)
        check(lib.iqcc_gpu_parallel_gradients(d.handle, _addr(t), _addr(c), c.shape[0], int(flip_group_only),
                                              _addr(g)))
        return g[: c.shape[0]]


# ------------------------------- PartitionedSum on the device (one caller)
@dataclass
class PartitionMap:
    """iqcc/partition.hpp:20-38."""
    n_qubits: int
    partition_bits: List[int]
    owner: List[int]
    n_workers: int = 1

    def n_partitions(self) -> int:
        return len(self.owner)

    def validate(self) -> None:
        if len(self.owner) != 1 << len(self.partition_bits):
            raise ValueError("PartitionMap: owner table size")
        if any(p >= 2 * self.n_qubits for p in self.partition_bits):
            raise ValueError("PartitionMap: bit position out of range")
        if any(w >= self.n_workers for w in self.owner):
            raise ValueError("PartitionMap: owner out of range")


def make_partition_map(h, m: int, n_workers: int) -> PartitionMap:
    """iqcc/partition.hpp:111-123: greedy bits (on the device), round-robin owners."""
    if n_workers < 1:
        raise ValueError("make_partition_map: no workers")
    bits, _ = choose_partition_bits(h, m)
    return PartitionMap(h.n_qubits, bits, [p % n_workers for p in range(1 << m)], n_workers)


@dataclass
class MessageRecord:
    """iqcc/partition.hpp:135-140."""
    source: int
    destination: int
    terms: int
    bytes: int


@dataclass
class MessageLog:
    """iqcc/partition.hpp:143-165."""
    records: List[MessageRecord] = field(default_factory=list)

    def total_terms(self) -> int:
        return sum(r.terms for r in self.records)

    def total_bytes(self) -> int:
        return sum(r.bytes for r in self.records)

    def to_csv(self) -> str:
        return "source,destination,terms,bytes\n" + "".join(
            f"{r.source},{r.destination},{r.terms},{r.bytes}\n" for r in self.records)


@dataclass
class ParallelDressStats:
    """iqcc/partition.hpp:303-306."""
    compress: CompressStats = field(default_factory=lambda: CompressStats())
    mask: int = 0


class PartitionedSum:
    """The reference's PartitionedSum (iqcc/partition.hpp:145-173) resident on
    the GPUs: 2^m shards, shard p owned by worker map.owner[p], worker w on
    CUDA device devices[w] (default w % device count).  One call drives all
    shards (a worker thread and engine context per shard inside the handle);
    any m, so several partitions may share a worker or a GPU."""

    def __init__(self, handle: int, pmap: PartitionMap):
        self.handle, self.map = handle, pmap
        self.n_qubits = pmap.n_qubits

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            lib.iqcc_gpu_psum_destroy(h)
            self.handle = None

    def _map_arrays(self):
        b = np.array(self.map.partition_bits or [0], np.uintp)
        o = np.array(self.map.owner, np.uintp)
        return b, o

    @staticmethod
    def distribute(h: PauliSum, pmap: PartitionMap, devices: Optional[Sequence[int]] = None) -> "PartitionedSum":
        """distribute (iqcc/partition.hpp:208-220)."""
        native.init()
        pmap.validate()
        if pmap.n_qubits != h.n_qubits:
            raise ValueError("distribute: mismatched qubit counts")
        rows = np.ascontiguousarray(h.rows, np.uint64)
        cf = np.ascontiguousarray(h.coeffs, np.complex128)
        b = np.array(pmap.partition_bits or [0], np.uintp)
        o = np.array(pmap.owner, np.uintp)
        dv = None if devices is None else np.array(devices, np.int32)
        out = C.c_void_p()
        check(lib.iqcc_gpu_psum_distribute(h.n_qubits, _addr(rows), _addr(cf), len(h), len(pmap.partition_bits),
                                           _addr(b), _addr(o), pmap.n_workers,
                                           None if dv is None else _addr(dv), C.byref(out)))
        return PartitionedSum(out.value, pmap)

    @staticmethod
    def from_shards(shards: Sequence[PauliSum], pmap: PartitionMap,
                    devices: Optional[Sequence[int]] = None) -> "PartitionedSum":
        """A reference PartitionedSum's shards uploaded as they are (each term
        must carry its shard's key, PartitionedSum::validate)."""
        native.init()
        pmap.validate()
        if len(shards) != pmap.n_partitions():
            raise ValueError("PartitionedSum: shard count != 2^m")
        rows = [np.ascontiguousarray(s.rows, np.uint64) for s in shards]
        cfs = [np.ascontiguousarray(s.coeffs, np.complex128) for s in shards]
        rp = (C.c_void_p * len(shards))(*[_addr(r) for r in rows])
        cp = (C.c_void_p * len(shards))(*[_addr(c) for c in cfs])
        sz = np.array([len(s) for s in shards], np.uintp)
        b, o = (np.array(pmap.partition_bits or [0], np.uintp), np.array(pmap.owner, np.uintp))
        dv = None if devices is None else np.array(devices, np.int32)
        out = C.c_void_p()
        check(lib.iqcc_gpu_psum_create_shards(pmap.n_qubits, len(pmap.partition_bits), _addr(b), _addr(o),
                                              pmap.n_workers, None if dv is None else _addr(dv), rp, cp,
                                              _addr(sz), C.byref(out)))
        return PartitionedSum(out.value, pmap)

    def shard_sizes(self) -> List[int]:
        sz = np.zeros(self.map.n_partitions(), np.uintp)
        check(lib.iqcc_gpu_psum_shard_sizes(self.handle, _addr(sz)))
        return [int(v) for v in sz]

    def total_terms(self) -> int:
        return sum(self.shard_sizes())

    def worker_loads(self) -> List[int]:
        loads = [0] * self.map.n_workers
        for p, n in enumerate(self.shard_sizes()):
            loads[self.map.owner[p]] += n
        return loads

    def shard(self, p: int) -> PauliSum:
        n = self.shard_sizes()[p]
        B = blocks_for(self.n_qubits)
        rows = np.zeros((max(n, 1), 2 * B), np.uint64)
        cf = np.zeros(max(n, 1), np.complex128)
        got = C.c_size_t()
        check(lib.iqcc_gpu_psum_download_shard(self.handle, p, _addr(rows), _addr(cf), n, C.byref(got)))
        return PauliSum(self.n_qubits, rows[: got.value], cf[: got.value])

    def gather(self) -> PauliSum:
        """gather (iqcc/partition.hpp:222-230), merged on the device."""
        n = self.total_terms()
        B = blocks_for(self.n_qubits)
        rows = np.zeros((max(n, 1), 2 * B), np.uint64)
        cf = np.zeros(max(n, 1), np.complex128)
        got = C.c_size_t()
        check(lib.iqcc_gpu_psum_gather(self.handle, _addr(rows), _addr(cf), n, C.byref(got)))
        return PauliSum(self.n_qubits, rows[: got.value], cf[: got.value])

    def dress(self, op: DressOp, epsilon: float, max_terms: int = U64_MAX, log: Optional[MessageLog] = None,
              stats: Optional[ParallelDressStats] = None) -> None:
        """In place parallel_dress (iqcc/partition.hpp:398-452)."""
        if op.generator.n_qubits != self.n_qubits:
            raise ValueError("parallel_dress: mismatched qubit counts")
        g = np.ascontiguousarray(op.generator.row, np.uint64)
        cap = self.map.n_partitions()
        recs = (native.MessageRecord * cap)()
        nl, mask = C.c_size_t(), C.c_size_t()
        cs = native.CompressStatsC()
        check(lib.iqcc_gpu_psum_dress(self.handle, _addr(g), math.cos(op.amplitude), math.sin(op.amplitude),
                                      epsilon, max_terms, recs, cap, C.byref(nl),
                                      C.byref(cs) if stats is not None else None, C.byref(mask)))
        if log is not None:
            log.records.extend(MessageRecord(recs[i].source, recs[i].destination, recs[i].terms, recs[i].bytes)
                               for i in range(min(nl.value, cap)))
        if stats is not None:
            stats.compress.dropped_terms += cs.dropped_terms
            stats.compress.dropped_weight += cs.dropped_weight
            stats.mask = mask.value

    def expect(self, omega: QmfState) -> float:
        t = qmf_factor_table(omega)
        e = C.c_double()
        check(lib.iqcc_gpu_psum_expect(self.handle, _addr(t), C.byref(e)))
        return e.value

    def qmf_energy_gradient(self, omega: QmfState):
        t, dt = qmf_factor_table(omega), qmf_deriv_table(omega)
        g = np.zeros(2 * self.n_qubits, np.float64)
        e = C.c_double()
        check(lib.iqcc_gpu_psum_qmf_energy_gradient(self.handle, _addr(t), _addr(dt), C.byref(e), _addr(g)))
        return e.value, g

    def gradients(self, omega: QmfState, cands: np.ndarray, flip_group_only: bool = False) -> np.ndarray:
        t = qmf_factor_table(omega)
        c = np.ascontiguousarray(cands, np.uint64).reshape(-1, 2 * blocks_for(self.n_qubits))
        g = np.zeros(max(1, c.shape[0]), np.float64)
        check(lib.iqcc_gpu_psum_gradients(self.handle, _addr(t), _addr(c), c.shape[0], int(flip_group_only),
                                          _addr(g)))
        return g[: c.shape[0]]

    def rebalance(self, threshold: float) -> PartitionMap:
        """rebalance (iqcc/partition.hpp:457-494) + device migration of moved shards."""
        o = np.zeros(self.map.n_partitions(), np.uintp)
        check(lib.iqcc_gpu_psum_rebalance(self.handle, threshold, _addr(o)))
        self.map = PartitionMap(self.map.n_qubits, list(self.map.partition_bits), [int(v) for v in o],
                                self.map.n_workers)
        return self.map


def distribute(h: PauliSum, pmap: PartitionMap, devices: Optional[Sequence[int]] = None) -> PartitionedSum:
    """iqcc/partition.hpp:208-220."""
    return PartitionedSum.distribute(h, pmap, devices)


def gather(ph: PartitionedSum) -> PauliSum:
    """iqcc/partition.hpp:222-230."""
    return ph.gather()


def parallel_dress(ph: PartitionedSum, op: DressOp, epsilon: float, max_terms: int = U64_MAX,
                   log: Optional[MessageLog] = None, mode=None,
                   stats: Optional[ParallelDressStats] = None) -> PartitionedSum:
    """iqcc/partition.hpp:398-452, in place on the device handle (returned).
    `mode` (ExecutionMode) is accepted for signature parity: shards always
    run concurrently and the result is the same either way."""
    ph.dress(op, epsilon, max_terms, log, stats)
    return ph


def parallel_expect(ph: PartitionedSum, omega: QmfState, mode=None) -> float:
    """iqcc/partition.hpp:241-254."""
    return ph.expect(omega)


def rebalance(ph: PartitionedSum, threshold: float) -> PartitionMap:
    """iqcc/partition.hpp:457-494."""
    return ph.rebalance(threshold)


def merge_sums(a: PauliSum, b: PauliSum, opts: MergeOptions = MergeOptions()) -> PauliSum:
    """iqcc/pauli.hpp:383-415 on the device (check_hermitian is moot: real sums)."""
    if a.n_qubits != b.n_qubits:
        raise ValueError("merge_sums: mismatched qubit counts")
    da, db = DeviceSum.upload(a), DeviceSum.upload(b)
    out = C.c_void_p()
    check(lib.iqcc_gpu_merge_sums(da.handle, db.handle, opts.drop_threshold, C.byref(out)))
    return DeviceSum(out.value, a.n_qubits).download()


def partition_key(row, n_qubits: int, bits) -> int:
    """partition_key (iqcc/partition.hpp:40-42) of a reference row."""
    B = blocks_for(n_qubits)
    key = 0
    for i, p in enumerate(bits):
        q = p if p < n_qubits else p - n_qubits
        w = int(row[(0 if p < n_qubits else B) + q // 64])
        key |= ((w >> (q % 64)) & 1) << i
    return key


# ------------------------------------------- polynomial expansion kernels
@dataclass
class PolySubset:
    """iqcc/optimizer.hpp:150-157: entangler indices (ascending), the ordered
    product word and its phase exponent (W_S = i^phase * word)."""
    indices: List[int]
    word: PauliWord
    phase_exponent: int


@dataclass
class PolyExpansion:
    """iqcc/optimizer.hpp:159-217 (subsets of size <= order_k)."""
    order_k: int
    n_entanglers: int
    n_qubits: int
    subsets: List[PolySubset]


@dataclass
class PolyKernels:
    """iqcc/optimizer.hpp:271-281: t x t complex kernels."""
    t: int
    h_kernel: np.ndarray
    n_kernel: np.ndarray


def build_poly(entanglers: Sequence[PauliWord], omega: QmfState, k: int,
               subset_budget: int = 200000) -> PolyExpansion:
    """build_poly (iqcc/optimizer.hpp:219-268): every subset of size <= k in
    lexicographic index order, words extended on the right by multiply."""
    n = len(entanglers)
    if k > n:
        raise ValueError("build_poly: order exceeds N")
    nq = omega.n_qubits()
    for p in entanglers:
        if p.n_qubits != nq:
            raise ValueError("build_poly: mismatched qubit counts")
        if not p.row.any():
            raise ValueError("build_poly: identity entangler")
    count, binom = 0.0, 1.0
    for j in range(k + 1):
        count += binom
        binom = binom * float(n - j) / float(j + 1)
        if count > float(subset_budget):
            raise RuntimeError("build_poly: subset budget exceeded")
    subs = [PolySubset([], PauliWord(nq), 0)]
    beg, end = 0, 1
    for _ in range(1, k + 1):
        nxt = len(subs)
        for s in range(beg, end):
            lo = subs[s].indices[-1] + 1 if subs[s].indices else 0
            for e in range(lo, n):
                w, t = multiply(subs[s].word, entanglers[e])
                subs.append(PolySubset(subs[s].indices + [e], w, (subs[s].phase_exponent + t) & 3))
        beg, end = nxt, len(subs)
    return PolyExpansion(k, n, nq, subs)


def build_poly_kernels(h: PauliSum, omega: QmfState, ex: PolyExpansion) -> PolyKernels:
    """iqcc::build_poly_kernels (iqcc/optimizer.hpp:340-368) on the B200: the
    t(t+1)/2 sandwiches <omega|W_a H W_b|omega> in one pass over the sum."""
    if len(h) == 0:  # zero Hamiltonian: h_kernel is 0, n_kernel still needed
        z = PauliSum(h.n_qubits)
        z.append(PauliWord(h.n_qubits), 0.0)
        return DeviceSum.upload(z).poly_kernels(omega, ex)
    return DeviceSum.upload(h).poly_kernels(omega, ex)


def poly_weights(ex: PolyExpansion, tau: Sequence[float]) -> np.ndarray:
    """PolyExpansion::weights (iqcc/optimizer.hpp:166-190):
    q_S = i^(phase_S + 3|S|) prod_{k in S} sin(tau_k/2) prod_{k not in S} cos(tau_k/2)."""
    ch = [math.cos(t / 2.0) for t in tau]
    sh = [math.sin(t / 2.0) for t in tau]
    q = np.zeros(len(ex.subsets), np.complex128)
    for s, sub in enumerate(ex.subsets):
        mag = 1.0
        idx = set(sub.indices)
        for k in range(ex.n_entanglers):
            mag *= sh[k] if k in idx else ch[k]
        q[s] = mag * (1, 1j, -1, -1j)[(sub.phase_exponent + 3 * len(sub.indices)) & 3]
    return q


def poly_energy_from_kernels(ex: PolyExpansion, ker: PolyKernels, tau: Sequence[float]):
    """poly_energy_from_kernels (iqcc/optimizer.hpp:452-466): the Rayleigh
    quotient q^H H q / q^H N q; returns (energy, norm)."""
    q = poly_weights(ex, tau)
    num = float(np.vdot(q, ker.h_kernel @ q).real)
    nrm = float(np.vdot(q, ker.n_kernel @ q).real)
    if nrm < 1e-14:
        raise RuntimeError("poly_energy: vanishing norm (over-truncation)")
    return num / nrm, nrm
