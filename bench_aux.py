#!/usr/bin/env python3
"""bench_aux.py — the SURVEY.md §8(d) configs other than the headline C3 line.

bench.py carries the driver's one-line contract (C3 dressing throughput);
this script measures the remaining §8(d) rows on one B200 and prints one
JSON object per row (profiles/r1_aux_*.json keeps the committed copy):

  C1      the recorded 5-iteration iQCC trace of h2_ccpvdz (20 qubits) replayed:
          DIS screening + dressing + energy per iteration ("s per iQCC
          iter"); the reference's full iteration timed beside it
  C2      G_uniform(64, 1e6, seed 1): one 4-qubit entangler (tau 0.37, drop
          1e-12) + compress(1e-3), and the max_terms = 1.2e6 variant
          (latency-dominated; roofline (M_in + M_out) * 24 B)
  energy  expect_sum / qmf_energy_gradient on G_mol(124, 1e8, seed 2) at a
          generic Omega (HBM: M * 40 B per call)
  C4      DIS gradient sweep on G_mol(100, 1e7, seed 3): odd-Y candidates
          (seed 4) at a generic Omega (compute-bound, pairs/s) and at HF
          poles with the flip-group restriction (group_gradient)
  C5      200-qubit slice: G_mol(200, 5e7, seed 5) dressed without a cap
          until > 1.25e8 terms (the per-GPU share of 1e9 over 8 B200), then
          compress(max_terms = 1.25e8) (truncation time)
  qcc     qcc_energy / qcc_gradient (iqcc/optimizer.hpp:19-77) on
          G_mol(124, 1e7) with 4 entanglers (uncompressed chains)
  poly    build_poly_kernels (iqcc/optimizer.hpp:340-368) on G_mol(124, 1e7),
          6 entanglers to order 2 (22 subsets, 253 sandwiches), generic omega;
          its CPU arm times oracle/_ref (the reference) on a 2e4-term sample

Times are device-synchronous wall clock around the public API calls (each
call ends with a stream synchronize), after a warm-up call.  Synthetic data
only; nothing here reads /root/reference; oracle/ is used only as the poly
row's CPU arm (the checker timed, never the measured GPU path).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
HBM_GBS = 6551.0


def peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return HBM_GBS


def brev64(a: np.ndarray) -> np.ndarray:
    a = a.astype(np.uint64)
    out = np.zeros_like(a)
    for b in range(64):
        out |= ((a >> np.uint64(b)) & np.uint64(1)) << np.uint64(63 - b)
    return out


def g_uniform(n: int, m: int, seed: int):
    """iid letters over {I,X,Y,Z}, U(-1,1) coefficients, canonical order
    (iqcc/pauli.hpp:146-161: lowest bit most significant, x plane first),
    duplicates dropped (tests/helpers.hpp:74-99 semantics)."""
    from paper_2603_08883_b200 import iqcc
    assert n == 64
    rs = np.random.default_rng(seed)
    x = rs.integers(0, 2**63, m, dtype=np.uint64) | (rs.integers(0, 2, m, dtype=np.uint64) << np.uint64(63))
    z = rs.integers(0, 2**63, m, dtype=np.uint64) | (rs.integers(0, 2, m, dtype=np.uint64) << np.uint64(63))
    kx, kz = brev64(x), brev64(z)
    order = np.lexsort((kz, kx))
    x, z, kx, kz = x[order], z[order], kx[order], kz[order]
    keep = np.ones(m, bool)
    keep[1:] = (kx[1:] != kx[:-1]) | (kz[1:] != kz[:-1])
    rows = np.stack([x[keep], z[keep]], axis=1)
    c = rs.uniform(-1.0, 1.0, int(keep.sum())).astype(np.complex128)
    return iqcc.PauliSum(n, rows, c)


def word(n, qs, ys):
    from paper_2603_08883_b200 import iqcc
    p = iqcc.PauliWord(n)
    B = iqcc.blocks_for(n)
    for q, y in zip(qs, ys):
        p.row[q // 64] |= np.uint64(1 << (q % 64))
        if y:
            p.row[B + q // 64] |= np.uint64(1 << (q % 64))
    return p


def odd_y_candidates(n, k, seed):
    """DIS candidates as dis_candidates makes them (iqcc/dis.hpp:89-116):
    random flip sets of 4 qubits, each with its 2^3 odd-#Y assignments (one
    support per group of 8 candidates)."""
    from paper_2603_08883_b200 import iqcc
    rs = np.random.default_rng(seed)
    B = iqcc.blocks_for(n)
    out = np.zeros((k, 2 * B), np.uint64)
    i = 0
    while i < k:
        qs = sorted(int(q) for q in rs.choice(n, 4, replace=False))
        for m in range(16):
            if bin(m).count("1") % 2 == 1 and i < k:
                out[i] = word(n, qs, [(m >> b) & 1 for b in range(4)]).row
                i += 1
    return out


def timed(fn, reps=3):
    import torch
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best, r


def row(name, **kv):
    d = {"config": name, **kv}
    print(json.dumps(d), flush=True)
    return d


def run_c2(args):
    from paper_2603_08883_b200 import iqcc
    h = g_uniform(64, 1_000_000, 1)
    base = iqcc.DeviceSum.upload(h)
    p = word(64, [3, 17, 40, 59], [1, 0, 0, 0])
    out = []
    for cap in (None, 1_200_000):
        def once():
            d = base.clone()
            t0 = time.perf_counter()
            st = d.dress(p, 0.37, 1e-12)
            d.compress(1e-3, cap if cap else iqcc.U64_MAX)
            import torch
            torch.cuda.synchronize()
            return time.perf_counter() - t0, st.n_in, st.n_out, len(d)
        once()
        best = min(once() for _ in range(5))
        secs, nin, nout, kept = best
        S = 24
        out.append(row("C2", variant="max_terms=1.2e6" if cap else "eps=1e-3", n_in=nin, n_out=nout,
                       kept=kept, ms=1e3 * secs, terms_per_s=nin / secs,
                       hbm_frac=(nin + nout) * S / secs / 1e9 / peak(),
                       note="dress + compress, host-synchronous; latency-dominated at 1e6 terms"))
    return out


def run_energy(args):
    from paper_2603_08883_b200 import iqcc
    n, m = 124, int(args.energy_terms)
    d = iqcc.DeviceSum.generate_mol(n, m, 2)
    rs = np.random.default_rng(7)
    om = iqcc.QmfState(rs.uniform(-3, 3, n), rs.uniform(-3, 3, n))
    S = 40
    t, e = timed(lambda: d.expect(om))
    r1 = row("energy", op="expect_sum", n_qubits=n, terms=m, ms=1e3 * t, terms_per_s=m / t,
             gbs=m * S / t / 1e9, hbm_frac=m * S / t / 1e9 / peak(), energy=e)
    t2, _ = timed(lambda: d.qmf_energy_gradient(om))
    r2 = row("energy", op="qmf_energy_gradient", n_qubits=n, terms=m, ms=1e3 * t2, terms_per_s=m / t2,
             gbs=m * S / t2 / 1e9, hbm_frac=m * S / t2 / 1e9 / peak())
    return [r1, r2]


def run_c4(args):
    from paper_2603_08883_b200 import iqcc
    n, m = 100, int(args.dis_terms)
    d = iqcc.DeviceSum.generate_mol(n, m, 3)
    rs = np.random.default_rng(9)
    generic = iqcc.QmfState(rs.uniform(-3, 3, n), rs.uniform(-3, 3, n))
    hf = iqcc.hf_reference([q < n // 4 for q in range(n)])
    out = []
    kg = int(args.dis_generic)
    cands = odd_y_candidates(n, max(kg, int(args.dis_poles)), 4)
    mg = int(args.dis_generic_terms)
    dg = iqcc.DeviceSum.generate_mol(n, mg, 3) if mg != m else d
    t, g = timed(lambda: dg.gradients(generic, cands[:kg]), reps=1)  # factor ratios (default)
    # useful multiplies per pair: expect_word over supp(T ^ P) = supp(T) | supp(P)
    # for the anticommuting pairs (others are skipped), from a 2e4 x 256 sample
    hs = dg.download()
    rows = hs.rows[np.random.default_rng(1).choice(len(hs), min(len(hs), 20000), replace=False)]
    B = (n + 63) // 64
    sup_t = rows[:, :B] | rows[:, B:]
    cs = cands[: min(kg, 256)]
    sup_p = cs[:, :B] | cs[:, B:]
    anti = np.zeros((len(rows), len(cs)), bool)
    union = np.zeros((len(rows), len(cs)), np.int64)
    for b in range(B):
        tx, tz = rows[:, b][:, None], rows[:, B + b][:, None]
        px, pz = cs[:, b][None, :], cs[:, B + b][None, :]
        anti ^= (np.bitwise_count((tx & pz) ^ (tz & px)) & 1).astype(bool)
        union += np.bitwise_count(sup_t[:, b][:, None] | sup_p[:, b][None, :]).astype(np.int64)
    mul_per_pair = float((union * anti).sum() / anti.size)
    fp64 = None
    try:
        import subprocess
        exe = os.path.join(ROOT, "tools", "_bin", "fp64_peak")
        fp64 = json.loads(subprocess.run([exe], capture_output=True, text=True, timeout=120).stdout)
    except Exception:
        pass
    # the factor-ratio kernel multiplies 2 values per nibble group the
    # candidate touches per anticommuting pair (+2: coefficient and sum)
    anti_frac = float(anti.mean())
    groups = float(np.mean([len({q // 4 for q in range(n) if (int(c[q // 64]) >> (q % 64)) & 1
                                 or (int(c[B + q // 64]) >> (q % 64)) & 1}) for c in cands[:kg]]))
    nib_per_pair = anti_frac * (2 * groups + 2)
    achieved = kg * mg / t * nib_per_pair
    out.append(row("C4", omega="generic", kernel="factor ratios", n_qubits=n, terms=mg, candidates=kg, s=t,
                   pairs_per_s=kg * mg / t, anticommuting_frac=anti_frac, dmul_per_pair=nib_per_pair,
                   dmul_per_s=achieved, fp64_dmul_peak_per_s=fp64["dmul_per_s"] if fp64 else None,
                   fp64_frac=achieved / fp64["dmul_per_s"] if fp64 else None,
                   groups_per_candidate=groups,
                   note="within 1e-13 of the reference per candidate (canonical-order sum); "
                        "<T^P> = E_T * prod over the candidate's nibble groups of f_g((T^P)_g) / f_g(T_g), "
                        "E_T and 1/f_g(T_g) once per staged term (IQCC_DIS_NIB=1: the full nibble product, "
                        "ceil(n/4) multiplies per pair); peak from tools/fp64_peak.cu (measured on this box)"))
    # the bit-exact ascending-qubit kernel (IQCC_DIS_EXACT=1) on a slice of the terms
    me = min(mg, int(args.dis_exact_terms))
    de = iqcc.DeviceSum.generate_mol(n, me, 3)
    os.environ["IQCC_DIS_EXACT"] = "1"
    try:
        te, _ = timed(lambda: de.gradients(generic, cands[:kg]), reps=1)
    finally:
        del os.environ["IQCC_DIS_EXACT"]
    del de
    out.append(row("C4", omega="generic", kernel="exact (IQCC_DIS_EXACT=1)", n_qubits=n, terms=me, candidates=kg,
                   s=te, pairs_per_s=kg * me / te, useful_dmul_per_pair=mul_per_pair,
                   dmul_per_s=kg * me / te * mul_per_pair,
                   fp64_frac=kg * me / te * mul_per_pair / fp64["dmul_per_s"] if fp64 else None,
                   note="bit-exact per candidate: one multiply per qubit of supp(T) | supp(P) per "
                        "anticommuting pair, ascending qubit order"))
    del dg
    kp = int(args.dis_poles)
    t, g = timed(lambda: d.gradients(hf, cands[:kp], True), reps=1)
    out.append(row("C4", omega="HF poles, flip-group restricted", n_qubits=n, terms=m, candidates=kp, s=t,
                   candidates_per_s=kp / t, nonzero=int(np.count_nonzero(g))))
    return out


def run_c5(args):
    from paper_2603_08883_b200 import iqcc
    import torch
    n = 200
    d = iqcc.DeviceSum.generate_mol(n, int(args.c5_terms), 5)
    target = int(args.c5_target)
    steps, tin, secs = 0, 0, 0.0
    k = 0
    while len(d) <= target and steps < 12:
        rs = np.random.default_rng([5, k])
        w = int(rs.integers(2, 5))
        qs = [int(q) for q in rs.choice(n, w, replace=False)]
        ys = [int(y) for y in rs.integers(0, 2, w)]
        if sum(ys) % 2 == 0:
            ys[-1] ^= 1
        p = word(n, qs, ys)
        tau = float(rs.uniform(-0.2, 0.2))
        k += 1
        nin = len(d)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = d.dress(p, tau, 1e-12)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if st.n_anticommuting == 0:
            continue
        steps += 1
        tin += nin
        secs += dt
    grown = len(d)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d.compress(1e-10, target)
    torch.cuda.synchronize()
    tc = time.perf_counter() - t0
    return [row("C5", n_qubits=n, start_terms=int(args.c5_terms), steps=steps, grown_to=grown,
                dress_terms_per_s=tin / secs if secs else None, compress_to=len(d), compress_ms=1e3 * tc,
                compress_gbs=grown * 72 / tc / 1e9,
                note="1-GPU slice of C5: per-GPU share of 1e9 terms over 8 B200 (no exchange)")]


def run_qcc(args):
    """qcc_energy / qcc_gradient (iqcc/optimizer.hpp:19-77, SURVEY.md §8(f)
    rank 1): uncompressed device-resident dressing chains."""
    from paper_2603_08883_b200 import iqcc
    n, m, K = 124, int(args.qcc_terms), 4
    d = iqcc.DeviceSum.generate_mol(n, m, 2)
    rs = np.random.default_rng(11)
    om = iqcc.QmfState(rs.uniform(-3, 3, n), rs.uniform(-3, 3, n))
    ents = []
    for k in range(K):
        r = np.random.default_rng([6, k])
        qs = [int(q) for q in r.choice(n, 4, replace=False)]
        ents.append(word(n, qs, [1, 0, 0, 0]))
    ans = iqcc.Ansatz(ents, [0.1, -0.2, 0.15, 0.05][:K])
    t, e = timed(lambda: d.qcc_energy(om, ans), reps=2)
    r1 = row("qcc", op="qcc_energy", n_qubits=n, terms=m, entanglers=K, ms=1e3 * t, energy=e,
             note="clone + K uncompressed dressings + expect_sum")
    t2, _ = timed(lambda: d.qcc_gradient(om, ans), reps=1)
    r2 = row("qcc", op="qcc_gradient", n_qubits=n, terms=m, entanglers=K, ms=1e3 * t2,
             note="K derivative chains (K(K+1)/2 dressings + K-1 forward) + K expect_sum")
    return [r1, r2]


def run_c1(args):
    """C1: the recorded iQCC trace of h2_ccpvdz (20 qubits,
    tests/golden/c1_h2_ccpvdz.npz, made from the reference) replayed on the
    device, one iteration at a time: DIS screening at the HF state
    (dis_candidates, top 1), dressing with that iteration's generator and
    its recorded amplitude, the energy.  The amplitude optimizer is not on
    the device path (out of scope), so the device figure is an
    iteration without it; the reference's full iteration (DIS, optimize,
    dress, energy; oracle/_ref) is timed beside it for context."""
    from paper_2603_08883_b200 import iqcc
    from oracle.oracle import Oracle
    import torch
    g = np.load(os.path.join(ROOT, "tests", "golden", "c1_h2_ccpvdz.npz"))
    n, ne = int(g["n_qubits"]), int(g["n_electrons"])
    hf = iqcc.hf_reference([j < ne for j in range(n)])
    gens, taus, it = g["gens"], g["taus"], g["gen_iter"]
    iters = int(it.max()) + 1

    def replay():
        d = iqcc.DeviceSum.upload(iqcc.PauliSum(n, g["rows0"], g["coeffs0"]))
        secs, picks_ok, energies = [], True, []
        for i in range(iters):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            picks = d.dis_candidates(hf, 1)
            sel = np.flatnonzero(it == i)
            ans = iqcc.Ansatz([iqcc.PauliWord(n, gens[k]) for k in sel], [float(taus[k]) for k in sel])
            d.dress_sequence(ans, 0.0)
            e = d.expect(hf)
            torch.cuda.synchronize()
            secs.append(time.perf_counter() - t0)
            picks_ok = picks_ok and len(picks) >= 1 and np.array_equal(picks[0].word.row, gens[sel[0]])
            energies.append(e)
        return secs, picks_ok, energies, len(d)

    replay()
    secs, picks_ok, energies, terms = replay()
    e_err = float(np.max(np.abs(np.array(energies) - g["energies"][:iters])))
    kind = "reference" if Oracle.available("reference") else "port"
    orc = Oracle(kind)
    h0 = orc.sum(n, np.ascontiguousarray(g["rows0"], np.uint64), np.ascontiguousarray(g["coeffs0"], np.complex128))
    th = np.where(np.arange(n) < ne, np.pi, 0.0)
    t0 = time.perf_counter()
    orc.iqcc_iteration(h0, th, np.zeros(n), 1)
    tc = time.perf_counter() - t0
    return [row("C1", system="h2_ccpvdz", n_qubits=n, iterations=iters, terms_final=terms,
                s_per_iter=float(np.mean(secs)), s_per_iter_each=[round(x, 6) for x in secs],
                dis_pick_matches_reference=bool(picks_ok), max_energy_err=e_err,
                cpu={"kind": kind, "cores": 1, "s_per_iter_incl_amplitude_optimization": tc},
                note="device: DIS screening + dressing + energy per iteration with the recorded amplitudes "
                     "(the optimizer is out of scope); cpu: the reference's full iqcc_iteration")]


def run_poly(args):
    """build_poly_kernels (iqcc/optimizer.hpp:340-368, SURVEY.md §8(f) rank
    2): t(t+1)/2 sandwiches <omega|W_a H W_b|omega> over a G_mol sum at a
    generic omega; the CPU arm is oracle/_ref (the reference) on a sample."""
    from paper_2603_08883_b200 import iqcc
    from oracle.oracle import Oracle
    n, m, K, order = 124, int(args.poly_terms), 6, 2
    d = iqcc.DeviceSum.generate_mol(n, m, 2)
    rs = np.random.default_rng(13)
    om = iqcc.QmfState(rs.uniform(-3, 3, n), rs.uniform(-3, 3, n))
    ents = []
    for k in range(K):
        r = np.random.default_rng([8, k])
        qs = [int(q) for q in r.choice(n, 4, replace=False)]
        ents.append(word(n, qs, [1, 0, 0, 0]))
    ex = iqcc.build_poly(ents, om, order)
    t_sub = len(ex.subsets)
    pairs = t_sub * (t_sub + 1) // 2
    t, _ = timed(lambda: d.poly_kernels(om, ex), reps=2)
    kind = "reference" if Oracle.available("reference") else "port"
    orc = Oracle(kind)
    ms_ = int(args.poly_cpu_terms)
    hs = orc.gen_mol(n, ms_, 2)
    t0 = time.perf_counter()
    orc.poly_kernels(hs, om.theta, om.phi, np.stack([e.row for e in ents]), order)
    tc = time.perf_counter() - t0
    return [row("poly", op="build_poly_kernels", n_qubits=n, terms=m, entanglers=K, order=order, subsets=t_sub,
                pairs=pairs, ms=1e3 * t, pair_terms_per_s=pairs * m / t,
                cpu={"kind": kind, "cores": 1, "sample_terms": ms_, "s": tc, "pair_terms_per_s": pairs * ms_ / tc})]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,c2,energy,c4,c5,qcc,poly")
    ap.add_argument("--qcc-terms", type=float, default=1e7)
    ap.add_argument("--energy-terms", type=float, default=1e8)
    ap.add_argument("--dis-terms", type=float, default=1e7)
    ap.add_argument("--dis-generic", type=float, default=1e5)
    ap.add_argument("--dis-generic-terms", type=float, default=1e7)
    ap.add_argument("--dis-poles", type=float, default=1e5)
    ap.add_argument("--dis-exact-terms", type=float, default=1e6)
    ap.add_argument("--c5-terms", type=float, default=5e7)
    ap.add_argument("--c5-target", type=float, default=1.25e8)
    ap.add_argument("--poly-terms", type=float, default=1e7)
    ap.add_argument("--poly-cpu-terms", type=float, default=2e4)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    from paper_2603_08883_b200 import native
    native.init(0)
    rows = []
    for part in args.only.split(","):
        rows += {"c1": run_c1, "c2": run_c2, "energy": run_energy, "c4": run_c4, "c5": run_c5, "qcc": run_qcc,
                 "poly": run_poly}[part](args)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
