"""torchrun worker for the multi-GPU parity test (tests/test_gpu_multi.py).

Every rank builds the same G_mol, keeps its bit-wise partition shard, and
runs parallel_dress steps (some entanglers flip the first partition bit, so
products are exchanged over NCCL).  Rank 0 gathers the shards and compares
their union with the CPU checker's serial pipeline, bit for bit, plus the
partitioned energy."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    n, N, steps = int(sys.argv[1]), int(float(sys.argv[2])), int(sys.argv[3])
    eps, cap = float(sys.argv[4]), int(float(sys.argv[5]))
    seq = len(sys.argv) > 6 and sys.argv[6] == "seq"  # one parallel dress_sequence call
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    from paper_2603_08883_b200 import iqcc, native
    native.init(local)
    d = iqcc.DeviceSum.generate_mol(n, N, 2)
    part = iqcc.Partition.setup(d, world, rank)
    part.reserve(d, 2 * len(d))  # receive buffers mapped once, before the steps
    B = iqcc.blocks_for(n)
    rs = np.random.default_rng(11)
    gens, taus, exch = [], [], 0
    for k in range(steps):
        w = int(rs.integers(2, 5))
        qs = [int(q) for q in rs.choice(n, w, replace=False)]
        ys = [int(y) for y in rs.integers(0, 2, w)]
        if k % 2 == 0:  # flip the first partition bit
            if part.flip_qubit not in qs:
                qs[0] = part.flip_qubit
            i = qs.index(part.flip_qubit)
            if part.flip_plane == "z":
                ys[i] = 1
            if sum(ys) % 2 == 0:
                ys[(i + 1) % w] ^= 1
        elif sum(ys) % 2 == 0:
            ys[-1] ^= 1
        p = iqcc.PauliWord(n)
        for q, y in zip(qs, ys):
            p.row[q // 64] |= np.uint64(1 << (q % 64))
            if y:
                p.row[B + q // 64] |= np.uint64(1 << (q % 64))
        tau = float(rs.uniform(-0.2, 0.2))
        if not seq:
            xs = part.dress(d, p, tau, eps, cap)
            exch += xs.sent_terms
        gens.append(p.row.copy())
        taus.append(tau)
    if seq:
        xl = []
        ans = iqcc.Ansatz([iqcc.PauliWord(n, g) for g in gens], taus)
        tin = part.dress_sequence(d, ans, eps, cap, exchange=xl)
        exch = sum(x.sent_terms for x in xl)
        assert tin > 0
    shard = d.download()
    th = np.where(np.arange(n) < n // 3, np.pi, 0.0)
    ph = np.zeros(n)
    e_par = part.expect(d, iqcc.QmfState(th, ph))
    # partitioned build_poly_kernels (optimizer.hpp:371-422) at the poles
    # (x-run path) and at a generic omega, 3 of the entanglers to order 2
    ents = [iqcc.PauliWord(n, g) for g in gens[:3]]
    th2 = np.random.default_rng(5).uniform(-3, 3, n)
    kers = []
    for tt, pp in ((th, ph), (th2, ph)):
        om = iqcc.QmfState(tt, pp)
        kers.append(part.poly_kernels(d, om, iqcc.build_poly(ents, om, 2)))
    # partitioned QMF energy/gradient and DIS gradients (allgather, rank order)
    th3 = np.random.default_rng(9).uniform(-3, 3, n)
    ph3 = np.random.default_rng(10).uniform(-3, 3, n)
    om3 = iqcc.QmfState(th3, ph3)
    e_qmf, g_qmf = part.qmf_energy_gradient(d, om3)
    cands = np.stack(gens[:4])
    g_dis = part.gradients(d, om3, cands)
    g_dis_poles = part.gradients(d, iqcc.QmfState(th, ph), cands, flip_group_only=True)
    # compress_partitioned alone (partition.hpp:325-396): a cut between
    # the eps floor and a global cap, canonical tie-break across ranks
    cap2 = max(1, (part.total_size(d) * 3) // 5)
    part.compress(d, 1e-6, cap2)
    shard_c = d.download()
    objs = [None] * world
    dist.all_gather_object(objs, (shard.rows, shard.coeffs, exch, shard_c.rows, shard_c.coeffs))
    if rank == 0:
        from oracle.oracle import Oracle
        # the unmodified reference (oracle/_ref, built here and shipped with
        # the snapshot) when present, else its pinned restatement
        port = Oracle("reference") if Oracle.available("reference") else Oracle("port")
        h = port.gen_mol(n, N, 2)
        h, _ = port.dress_sequence(h, np.stack(gens), taus, eps, cap)
        r, c = h.export()
        rows = np.concatenate([o[0] for o in objs])
        coeffs = np.concatenate([o[1] for o in objs])
        # gather (partition.hpp:224-230): canonical merge of disjoint shards
        rows, coeffs = port.from_terms(n, rows, coeffs, drop=0.0, check=False).export()
        ok = rows.shape == r.shape and np.array_equal(rows, r) and np.array_equal(coeffs, c)
        rc, cc = port.compress(h, 1e-6, max(1, (len(r) * 3) // 5))[0].export()
        rows2 = np.concatenate([o[3] for o in objs])
        coeffs2 = np.concatenate([o[4] for o in objs])
        rows2, coeffs2 = port.from_terms(n, rows2, coeffs2, drop=0.0, check=False).export()
        ok = ok and rows2.shape == rc.shape and np.array_equal(rows2, rc) and np.array_equal(coeffs2, cc)
        e_ref = port.expect_sum(th, ph, h)
        e_ok = abs(e_par - e_ref) <= 1e-10 * max(1.0, abs(e_ref))
        for ker, tt in zip(kers, (th, th2)):
            _, _, hc, nc, _ = port.poly_kernels(h, tt, ph, np.stack(gens[:3]), 2)
            scale = max(1e-300, np.abs(hc).max())
            e_ok = e_ok and np.abs(ker.h_kernel - hc).max() <= 1e-12 * scale and np.array_equal(ker.n_kernel, nc)
        e1, g1 = port.qmf_energy_gradient(h, th3, ph3)
        e_ok = e_ok and abs(e_qmf - e1) <= 1e-10 * max(1.0, abs(e1))
        e_ok = e_ok and np.abs(g_qmf - g1).max() <= 1e-10 * max(1.0, np.abs(g1).max())
        gd = np.array([port.gradient(h, th3, ph3, c) for c in cands])
        e_ok = e_ok and np.abs(g_dis - gd).max() <= 1e-10 * max(1.0, np.abs(gd).max())
        gp = np.array([port.gradient(h, th, ph, c) for c in cands])  # exact at the poles
        e_ok = e_ok and np.abs(g_dis_poles - gp).max() <= 1e-10 * max(1.0, np.abs(gp).max())
        print(f"MULTI world={world} checker={port.flavor} terms={len(r)} exchanged={sum(o[2] for o in objs)} "
              f"bitexact={ok} energy_ok={e_ok}", flush=True)
        if not (ok and e_ok):
            sys.exit(1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
