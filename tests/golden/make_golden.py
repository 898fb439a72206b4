"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run here (needs /root/reference and oracle/_ref/libiqcc_ref.so):
    python tests/golden/make_golden.py
The GPU box has no /root/reference; the committed fixtures carry what the
parity tests need there.

Fixtures
--------
c1_<name>.npz   SURVEY.md §8(d) config C1: the Jordan-Wigner Hamiltonian of
                proj/data/<name>.fcidump (io.hpp:154-310), its HF energy, the
                full DIS at HF (dis.hpp:140), the FCI energy (oracle.hpp:365)
                and an iQCC trace composed as in SURVEY.md §3.6: per
                iteration the picked entanglers, the optimized amplitudes
                (optimizer.hpp:96), the dressed term count, the energy and a
                SHA-256 of the dressed sum's canonical bytes; the final
                dressed sum is stored in full.
small.npz       random cases from the reference test seeds (dress_single,
                compress, dress_sequence outputs with checksums).
io.npz + io_*.txt / fcidump_*.txt   iqcc/io.hpp fixtures: a Pauli text file
                written by the reference's write_pauli_file, a hand-made one with
                comments, blank lines and duplicate words, two synthetic FCIDUMPs
                (random integrals with the 8-fold symmetry, made here), and the
                reference's parse_pauli_file / jordan_wigner(read_fcidump) results.
c2.npz          SURVEY.md §8(d) config C2 at full size: G_uniform(64, 1e6,
                seed 1) dressed by one weight-4 entangler at tau = 0.37 (drop
                1e-12), then compress(1e-3) and compress(0, max_terms=1.2e6);
                sizes + SHA-256 of each result, plus dress_sequence with
                MergeOptions{0.0} and {1e-6} on a G_mol(124, 2e4) sum.
"""
import hashlib
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle  # noqa: E402

DATA = "/root/reference/proj/data"


def digest(rows, coeffs):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(rows, np.uint64).tobytes())
    # values, not bit patterns: -0.0 and +0.0 (e.g. imaginary parts produced
    # by the reference's complex arithmetic) compare equal, as in PauliSum ==
    h.update((np.ascontiguousarray(coeffs, np.complex128).view(np.float64) + 0.0).tobytes())
    return h.hexdigest()


def c1(ref, name, iters, k_per_iter):
    h, ne = ref.jordan_wigner_fcidump(os.path.join(DATA, f"{name}.fcidump"))
    n = h.n_qubits
    theta = np.array([math.pi if j < ne else 0.0 for j in range(n)])
    phi = np.zeros(n)
    rows0, c0 = h.export()
    e_hf = ref.expect_sum(theta, phi, h)
    dis_rows, dis_g = ref.dis_candidates(h, theta, phi, 1 << 20)
    e_fci = ref.ground_energy(h) if n <= 12 else float("nan")
    trace = {"gens": [], "taus": [], "iter": [], "energy": [], "terms": [], "sha": []}
    cur = h
    for it in range(iters):
        nxt, gens, taus, e = ref.iqcc_iteration(cur, theta, phi, k_per_iter)
        if len(taus) == 0:
            break
        r, c = nxt.export()
        for g, t in zip(gens, taus):
            trace["gens"].append(g)
            trace["taus"].append(t)
            trace["iter"].append(it)
        trace["energy"].append(e)
        trace["terms"].append(len(nxt))
        trace["sha"].append(digest(r, c))
        cur = nxt
    rf, cf = cur.export()
    W = rows0.shape[1]
    out = dict(
        n_qubits=n, n_electrons=ne, rows0=rows0, coeffs0=c0, e_hf=e_hf, e_fci=e_fci,
        dis_rows=dis_rows, dis_g=dis_g,
        gens=np.array(trace["gens"], np.uint64).reshape(-1, W), taus=np.array(trace["taus"]),
        gen_iter=np.array(trace["iter"], np.int64), energies=np.array(trace["energy"]),
        terms=np.array(trace["terms"], np.int64), shas=np.array(trace["sha"]),
        rows_final=rf, coeffs_final=cf,
    )
    np.savez_compressed(os.path.join(HERE, f"c1_{name}.npz"), **out)
    print(name, "terms", len(h), "->", trace["terms"], "E", trace["energy"], "DIS", len(dis_g))


def small(ref):
    """Reference outputs for the seeds of tests/test_dressing.cpp:177-196
    (seed 557) and tests/test_partition.cpp:180-208 (seed 631)."""
    cases = {}
    rng = ref.rng(557)
    shas = []
    for t in range(120):
        n = 2 + t % 7
        h = rng.sum(n, 12 * n)
        g = rng.word(n, False)
        tau = rng.uniform(-3.0, 3.0)
        r, c = ref.dress_single(h, g, tau).export()
        shas.append(digest(r, c))
    cases["dress557_sha"] = np.array(shas)
    rng = ref.rng(631)
    shas = []
    for t in range(40):
        n = 3 + t % 4
        h = rng.sum(n, 25 * n)
        g = rng.word(n, False)
        tau = rng.uniform(-3.0, 3.0)
        eps = 1e-3 if t % 3 == 0 else 0.0
        mt = 40 if t % 4 == 0 else 100000
        d = ref.dress_single(h, g, tau)
        if eps > 0 or len(d) > mt:
            d, _ = ref.compress(d, eps, mt)
        r, c = d.export()
        shas.append(digest(r, c))
    cases["pipeline631_sha"] = np.array(shas)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **cases)
    print("small fixtures", {k: len(v) for k, v in cases.items()})


C2_QUBITS, C2_TERMS, C2_SEED, C2_TAU = 64, 1_000_000, 1, 0.37


def c2_entangler():
    """X5 Y21 Z38 X60 (weight 4, reference row layout)."""
    row = np.zeros(2, np.uint64)
    for q, (x, z) in {5: (1, 0), 21: (1, 1), 38: (0, 1), 60: (1, 0)}.items():
        if x:
            row[0] |= np.uint64(1 << q)
        if z:
            row[1] |= np.uint64(1 << q)
    return row


def drop_cases():
    """(n, terms, seed, gens, taus) of the MergeOptions cases."""
    rs = np.random.default_rng(99)
    n, B = 124, 2
    gens, taus = [], []
    for _ in range(4):
        row = np.zeros(2 * B, np.uint64)
        qs = rs.choice(n, 3, replace=False)
        for q, (x, z) in zip(qs, [(1, 0), (1, 1), (1, 0)]):
            if x:
                row[q // 64] |= np.uint64(1 << int(q % 64))
            if z:
                row[B + q // 64] |= np.uint64(1 << int(q % 64))
        gens.append(row)
        taus.append(float(rs.uniform(-0.3, 0.3)))
    return n, 20000, 5, np.stack(gens), np.array(taus)


def c2(ref):
    h = ref.rng(C2_SEED).sum(C2_QUBITS, C2_TERMS)
    d = ref.dress_single(h, c2_entangler(), C2_TAU)
    a, sa = ref.compress(d, 1e-3, 2**64 - 1)
    b, sb = ref.compress(d, 0.0, 1_200_000)
    out = {"n_in": len(h), "sha_in": digest(*h.export())}
    for k, s in (("dressed", d), ("eps", a), ("cap", b)):
        out[f"n_{k}"] = len(s)
        out[f"sha_{k}"] = digest(*s.export())
    out["dropped_eps"], out["dropped_cap"] = sa["dropped_terms"], sb["dropped_terms"]
    n, terms, seed, gens, taus = drop_cases()
    hm = ref.gen_mol(n, terms, seed)
    for tag, drop in (("drop0", 0.0), ("drop6", 1e-6), ("drop12", 1e-12)):
        s, _ = ref.dress_sequence(hm, gens, taus, 0.0, 2**64 - 1, drop=drop)
        out[f"n_{tag}"] = len(s)
        out[f"sha_{tag}"] = digest(*s.export())
    np.savez_compressed(os.path.join(HERE, "c2.npz"), **out)
    print("c2", {k: v for k, v in out.items() if k.startswith("n_")})


def synthetic_fcidump(path, norb, nelec, seed):
    """Random real integrals with h symmetric and (pq|rs) 8-fold symmetric,
    each unique element written once (FCIDUMP convention)."""
    rs = np.random.default_rng(seed)
    lines = [f" &FCI NORB={norb},NELEC={nelec},MS2=0,", "  ORBSYM=" + "1," * norb, "  ISYM=1,", " &END"]
    for i in range(1, norb + 1):
        for j in range(1, i + 1):
            for k in range(1, norb + 1):
                for l in range(1, k + 1):
                    if (i * (i - 1) // 2 + j) < (k * (k - 1) // 2 + l):
                        continue
                    if rs.random() < 0.3:
                        continue  # sparse, like real integral files
                    lines.append(f"{rs.normal(0, 0.3):.16e} {i} {j} {k} {l}")
    for i in range(1, norb + 1):
        for j in range(1, i + 1):
            lines.append(f"{rs.normal(0, 1.0):.16e} {i} {j} 0 0")
    lines.append(f"{rs.normal(0, 1.0):.16e} 0 0 0 0")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


def io_fixtures(ref):
    out = {}
    h = ref.rng(71).sum(10, 300)
    p1 = os.path.join(HERE, "io_sum10.txt")
    ref.write_pauli_file(h, p1)
    out["sha_sum10"] = digest(*h.export())
    out["n_sum10"] = len(h)
    p2 = os.path.join(HERE, "io_dups.txt")
    with open(p2, "w") as f:
        f.write("# a hand-made Pauli file\n# qubits: 6\n\n"
                "0.5 XXIIZZ\n-0.25 IIIIII\n  1e-13 ZZZZZZ\n0.125 XXIIZZ\n"
                "# duplicates merge (0.5 + 0.125), 1e-13 < 1e-12 is dropped\n"
                "3 YIYIYI\n-3 YIYIYI\n0.75 IIIIIX\n")
    d = ref.parse_pauli_file(p2)
    out["rows_dups"], out["coeffs_dups"] = d.export()
    r = ref.parse_pauli_file(p1)
    out["sha_sum10_parsed"] = digest(*r.export())
    for name, norb, ne, seed in (("fcidump_4", 4, 2, 81), ("fcidump_6", 6, 4, 83)):
        path = os.path.join(HERE, f"{name}.txt")
        synthetic_fcidump(path, norb, ne, seed)
        jw, nel = ref.jordan_wigner_fcidump(path)
        out[f"rows_{name}"], out[f"coeffs_{name}"] = jw.export()
        out[f"nelec_{name}"] = nel
    np.savez_compressed(os.path.join(HERE, "io.npz"), **out)
    print("io", {k: (v.shape if hasattr(v, "shape") else v) for k, v in out.items()})


def main():
    ref = Oracle("reference")
    if "--c2" in sys.argv:
        c2(ref)
        return
    if "--io" in sys.argv:
        io_fixtures(ref)
        return
    c1(ref, "h2_sto3g", 5, 1)
    c1(ref, "h2_ccpvdz", 5, 1)
    small(ref)
    c2(ref)
    io_fixtures(ref)


if __name__ == "__main__":
    main()
