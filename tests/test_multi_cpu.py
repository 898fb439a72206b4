"""The N>1 protocol on CPU (world_size 2, gloo): each rank owns one bit-wise
partition, dresses its shard, ships products whose partition key flips to
the rank owning p ^ mask, merges what it receives, and compresses against a
global budget with a canonical cross-rank tie-break -- the host-level
schedule of paper_2603_08883_b200/csrc/multi.cu, run with the CPU checker
and gloo instead of the engine and NCCL.  The union of the shards must
equal the serial reference pipeline (tests/test_partition.cpp:180-208)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_08883_b200.iqcc import partition_key


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _split(port, osum, n, bits, want):
    r, c = osum.export()
    keep = np.array([partition_key(row, n, bits) == want for row in r], bool)
    return r[keep], c[keep], r[~keep], c[~keep]


def _send_arrays(rows, coeffs, peer):
    dist.send(torch.tensor([rows.shape[0]], dtype=torch.int64), peer)
    if rows.shape[0]:
        dist.send(torch.from_numpy(rows.view(np.int64).copy()), peer)
        dist.send(torch.from_numpy(coeffs.view(np.float64).copy()), peer)


def _recv_arrays(W, peer):
    n = torch.zeros(1, dtype=torch.int64)
    dist.recv(n, peer)
    n = int(n.item())
    r = torch.zeros((n, W), dtype=torch.int64)
    c = torch.zeros(2 * n, dtype=torch.float64)
    if n:
        dist.recv(r, peer)
        dist.recv(c, peer)
    return r.numpy().view(np.uint64), c.numpy().view(np.complex128)


def _global_compress(port, n, rows, coeffs, eps, max_terms):
    """compress_partitioned (iqcc/partition.hpp:325-396) with gloo collectives."""
    mag = np.abs(coeffs)
    ident = ~rows.any(axis=1)
    kept = ident | (mag >= eps)
    rows, coeffs, mag, ident = rows[kept], coeffs[kept], mag[kept], ident[kept]
    tot = torch.tensor([len(rows)], dtype=torch.int64)
    dist.all_reduce(tot)
    if int(tot.item()) <= max_terms:
        return rows, coeffs
    objs = [None, None]
    dist.all_gather_object(objs, (rows, mag, ident))
    allr = np.concatenate([o[0] for o in objs])
    allm = np.concatenate([o[1] for o in objs])
    alli = np.concatenate([o[2] for o in objs])
    budget = max_terms - int(alli.sum())
    cand = [i for i in range(len(allr)) if not alli[i]]
    # larger |c| first, canonical (bit-reversed lexicographic) order on ties
    rev = lambda w: int(f"{int(w):064b}"[::-1], 2)  # noqa: E731
    cand.sort(key=lambda i: (-allm[i], tuple(rev(w) for w in allr[i])))
    chosen = set(cand[:budget]) | {i for i in range(len(allr)) if alli[i]}
    off = 0 if dist.get_rank() == 0 else len(objs[0][0])
    mine = np.array([(off + i) in chosen for i in range(len(rows))], bool)
    return rows[mine], coeffs[mine]


def _worker(rank, world, master_port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(master_port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle
    port = Oracle("port")
    n, eps, cap = 64, 1e-9, 4500
    H = port.gen_mol(n, 3000, 2)
    bits, _ = port.choose_partition_bits(H, 1)
    bits = [int(b) for b in bits]
    mine, peer = rank, 1 - rank  # owner[p] = p
    r, c, _, _ = _split(port, H, n, bits, mine)
    shard = port.sum(n, r, c)
    rs = np.random.default_rng(3)
    B = 1
    gens, taus, shipped = [], [], 0
    b0 = bits[0]
    fq, plane = (b0, "x") if b0 < n else (b0 - n, "z")
    for k in range(6):
        w = int(rs.integers(2, 5))
        qs = [int(q) for q in rs.choice(n, w, replace=False)]
        ys = [int(y) for y in rs.integers(0, 2, w)]
        if k % 2 == 0:
            if fq not in qs:
                qs[0] = fq
            i = qs.index(fq)
            if plane == "z":
                ys[i] = 1
            if sum(ys) % 2 == 0:
                ys[(i + 1) % w] ^= 1
        elif sum(ys) % 2 == 0:
            ys[-1] ^= 1
        gen = np.zeros(2 * B, np.uint64)
        for q, y in zip(qs, ys):
            gen[0] |= np.uint64(1 << q)
            if y:
                gen[1] |= np.uint64(1 << q)
        tau = float(rs.uniform(-0.2, 0.2))
        gens.append(gen)
        taus.append(tau)
        mask = partition_key(gen, n, bits)
        d = port.dress_single(shard, gen, tau, drop=1e-12, check=False)
        if mask == 0:
            lr, lc = d.export()
        else:
            # survivors keep key p; every product carries key p ^ mask
            lr, lc, orow, ocoef = _split(port, d, n, bits, mine)
            assert all(partition_key(x, n, bits) == (mine ^ mask) for x in orow)
            shipped += len(orow)
            if rank == 0:
                _send_arrays(orow, ocoef, peer)
                rr, rc = _recv_arrays(2 * B, peer)
            else:
                rr, rc = _recv_arrays(2 * B, peer)
                _send_arrays(orow, ocoef, peer)
            merged = port.merge_sums(port.sum(n, lr, lc), port.sum(n, rr, rc), drop=1e-12, check=False)
            lr, lc = merged.export()
        lr, lc = _global_compress(port, n, lr, lc, eps, cap)
        shard = port.sum(n, lr, lc)
    objs = [None, None]
    dist.all_gather_object(objs, shard.export())
    if rank == 0:
        ref, _ = port.dress_sequence(H, np.stack(gens), taus, eps, cap)
        rr_, rc_ = ref.export()
        allr = np.concatenate([o[0] for o in objs])
        allc = np.concatenate([o[1] for o in objs])
        gr, gc = port.from_terms(n, allr, allc, drop=0.0, check=False).export()
        out_q.put((gr.shape == rr_.shape and np.array_equal(gr, rr_) and np.array_equal(gc, rc_), shipped))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_partitioned_protocol_matches_serial():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_no, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, shipped = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok
    assert shipped > 0  # the flipping entanglers really exchanged products
