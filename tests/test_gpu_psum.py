"""GPU parity of the device PartitionedSum (iqcc/partition.hpp) driven from one
host thread: distribute / gather / parallel_dress / parallel_expect /
rebalance with any m (several partitions per worker and per GPU), the
MessageLog, and the partitioned QMF / DIS gradients.  Restates the
reference's tests/test_partition.cpp cases (seeds 613-659) against the CPU
checker, which test_oracle.py pins to the unmodified reference.  Runs on one
GPU (all shards on device 0); with two or more visible GPUs the same cases
also run with the workers spread over the devices (NVLink exchange and
shard migration)."""
import math

import numpy as np
import pytest

from helpers import digest

pytestmark = pytest.mark.gpu

U64_MAX = 2**64 - 1


def host(eng, osum):
    r, c = osum.export()
    return eng.PauliSum(osum.n_qubits, r, c)


def same_sum(got, want_osum):
    r, c = want_osum.export()
    return got.rows.shape == r.shape and np.array_equal(got.rows, r) and np.array_equal(got.coeffs, c)


def n_devices():
    import torch
    return torch.cuda.device_count()


def device_layouts(n_workers):
    """One layout with every worker on GPU 0, and (with >= 2 GPUs) one with
    the workers round-robin over the visible GPUs."""
    out = [[0] * n_workers]
    if n_devices() >= 2:
        out.append([w % n_devices() for w in range(n_workers)])
    return out


def pmap_of(eng, port, h, m, workers):
    bits, _ = port.choose_partition_bits(h, m)
    return eng.PartitionMap(h.n_qubits, [int(b) for b in bits], [p % workers for p in range(1 << m)], workers)


def fixed_map(eng, n, bits, workers):
    return eng.PartitionMap(n, list(bits), [p % workers for p in range(1 << len(bits))], workers)


def test_distribute_gather_identity(eng, port):  # test_partition.cpp:114-134 (seed 613)
    rng = port.rng(613)
    for trial in range(20):
        n = 3 + trial % 5
        h = rng.sum(n, 20 * n)
        for devs in device_layouts(4):
            ph = eng.distribute(host(eng, h), pmap_of(eng, port, h, 3, 4), devs)
            assert same_sum(ph.gather(), h)
            assert sum(ph.shard_sizes()) == len(h)
            for p in range(8):  # every term sits in its own shard
                s = ph.shard(p)
                assert all(eng.partition_key(r, n, ph.map.partition_bits) == p for r in s.rows)
    empty = eng.PauliSum(4)
    pe = eng.distribute(empty, fixed_map(eng, 4, [0, 1], 2))
    assert pe.shard_sizes() == [0, 0, 0, 0] and len(pe.gather()) == 0
    single = eng.PauliSum(4)
    single.append(eng.PauliWord.from_string("XYZI"), 0.5)
    ps = eng.distribute(single, fixed_map(eng, 4, [0, 1], 2))
    assert sum(1 for v in ps.shard_sizes() if v) == 1


def test_wrong_shard_rejected(eng, port):  # PartitionedSum::validate (partition.hpp:162-172)
    rng = port.rng(614)
    h = host(eng, rng.sum(5, 60))
    pm = fixed_map(eng, 5, [0, 2], 2)
    with pytest.raises(RuntimeError):
        eng.PartitionedSum.from_shards([h, eng.PauliSum(5), eng.PauliSum(5), eng.PauliSum(5)], pm)
    with pytest.raises(ValueError):  # owner out of range
        eng.distribute(h, eng.PartitionMap(5, [0, 2], [0, 1, 2, 3], 2))
    # a non-canonical input fails with the upload's invalid_argument (not the
    # "another shard failed" of the shards it released), on any device layout
    u = eng.PauliSum(5, h.rows[::-1].copy(), h.coeffs[::-1].copy())
    for devs in device_layouts(2):
        with pytest.raises(ValueError):
            eng.distribute(u, fixed_map(eng, 5, [0, 2], 2), devs)


def test_local_entangler_moves_nothing(eng, port):  # test_partition.cpp:136-155 (seed 617)
    rng = port.rng(617)
    h = rng.sum(5, 60)
    ph = eng.distribute(host(eng, h), fixed_map(eng, 5, [0, 1], 2))
    op = eng.DressOp(eng.PauliWord.from_string("ZZIII"), 0.8)
    log, st = eng.MessageLog(), eng.ParallelDressStats()
    eng.parallel_dress(ph, op, 0.0, U64_MAX, log, None, st)
    assert st.mask == 0 and log.records == []
    want, _ = port.dress_sequence(h, op.generator.row[None, :], [0.8], 0.0, len(h) * 3)
    assert same_sum(ph.gather(), want)


def test_flip_entanglers_match_reference_log(eng, port):  # test_partition.cpp:157-178 (seed 619)
    rng = port.rng(619)
    bits = [0, 2, 6]
    for trial in range(20):
        h = rng.sum(5, 80)
        g = rng.word(5, False)
        want, sizes, log, mask = port.parallel_dress(h, bits, [p % 4 for p in range(8)], 4, g, 1.1, 0.0)
        for devs in device_layouts(4):
            ph = eng.distribute(host(eng, h), fixed_map(eng, 5, bits, 4), devs)
            glog, st = eng.MessageLog(), eng.ParallelDressStats()
            ph.dress(eng.DressOp(eng.PauliWord(5, g), 1.1), 0.0, U64_MAX, glog, st)
            assert st.mask == mask
            assert [(r.source, r.destination, r.terms, r.bytes) for r in glog.records] == [tuple(r) for r in log]
            assert ph.shard_sizes() == list(sizes)
            assert same_sum(ph.gather(), want)
            for r in glog.records:
                assert r.destination == r.source ^ mask and r.terms > 0


@pytest.mark.parametrize("workers", [1, 2, 4, 8])
def test_parallel_equals_reference_all_worker_counts(eng, port, workers):  # :180-208 (seed 631)
    rng = port.rng(631)
    for trial in range(20):
        n = 3 + trial % 4
        h = rng.sum(n, 25 * n)
        g = rng.word(n, False)
        tau = rng.uniform(-3.0, 3.0)
        eps = 1e-3 if trial % 3 == 0 else 0.0
        mt = 40 if trial % 4 == 0 else 100000
        m = 2 if workers == 1 else 3
        bits, _ = port.choose_partition_bits(h, m)
        owner = [p % workers for p in range(1 << m)]
        want, sizes, log, mask = port.parallel_dress(h, bits, owner, workers, g, tau, eps, mt)
        serial, _ = port.dress_sequence(h, g[None, :], [tau], eps, mt)
        assert digest(*want.export()) == digest(*serial.export())
        for devs in device_layouts(workers):
            ph = eng.distribute(host(eng, h), eng.PartitionMap(n, [int(b) for b in bits], owner, workers), devs)
            cs = eng.ParallelDressStats()
            ph.dress(eng.DressOp(eng.PauliWord(n, g), tau), eps, mt, None, cs)
            assert ph.shard_sizes() == list(sizes)
            assert same_sum(ph.gather(), want)


def test_determinism_and_stats(eng, port):  # test_partition.cpp:210-248 (seeds 641, 643)
    rng = port.rng(641)
    h = rng.sum(6, 150)
    g = rng.word(6, False)
    outs = []
    for _ in range(2):
        ph = eng.distribute(host(eng, h), pmap_of(eng, port, h, 3, 4))
        ph.dress(eng.DressOp(eng.PauliWord(6, g), 0.9), 1e-10, 500)
        outs.append([ph.shard(p) for p in range(8)])
    for a, b in zip(*outs):
        assert np.array_equal(a.rows, b.rows) and np.array_equal(a.coeffs, b.coeffs)
    # compress statistics of the partitioned compress match the serial compress
    rng = port.rng(643)
    h = rng.sum(5, 90)
    g = rng.word(5, False)
    ph = eng.distribute(host(eng, h), pmap_of(eng, port, h, 3, 4))
    st = eng.ParallelDressStats()
    ph.dress(eng.DressOp(eng.PauliWord(5, g), -0.7), 1e-9, 30, None, st)
    want, sw = port.dress_sequence(h, g[None, :], [-0.7], 1e-9, 30)
    assert same_sum(ph.gather(), want)
    assert st.compress.dropped_terms == sw["dropped_terms"]
    assert st.compress.dropped_weight == pytest.approx(sw["dropped_weight"], rel=1e-12)


def test_partitioned_energy_and_gradients(eng, port):  # test_partition.cpp:257-272 (seed 647)
    rng = port.rng(647)
    for trial in range(8):
        h = rng.sum(6, 100)
        th, phi = rng.qmf(6)
        om = eng.QmfState(np.array(th), np.array(phi))
        serial = port.expect_sum(th, phi, h)
        e1, g1 = port.qmf_energy_gradient(h, th, phi)
        cands = np.stack([rng.word(6, False) for _ in range(5)])
        gd = np.array([port.gradient(h, th, phi, c) for c in cands])
        for workers in (1, 2, 4):
            bits, _ = port.choose_partition_bits(h, 3)
            owner = [p % workers for p in range(8)]
            want = port.parallel_expect(h, bits, owner, workers, th, phi)
            for devs in device_layouts(workers):
                ph = eng.distribute(host(eng, h), eng.PartitionMap(6, [int(b) for b in bits], owner, workers),
                                    devs)
                par = ph.expect(om)
                tol = 1e-10 * max(1.0, abs(serial))
                assert abs(par - want) <= tol and abs(par - serial) <= tol
                e, g = ph.qmf_energy_gradient(om)
                assert abs(e - e1) <= tol
                assert np.abs(g - g1).max() <= 1e-10 * max(1.0, np.abs(g1).max())
                gg = ph.gradients(om, cands)
                assert np.abs(gg - gd).max() <= 1e-10 * max(1.0, np.abs(gd).max())


def test_rebalance_matches_reference(eng, port):  # test_partition.cpp:274-309 (seeds 653, 659)
    rng = port.rng(653)
    h = rng.sum(6, 160)
    bits = [0, 1, 2]
    want = port.rebalance(h, bits, [0] * 8, 4, 1.5)
    for devs in device_layouts(4):
        ph = eng.distribute(host(eng, h), eng.PartitionMap(6, bits, [0] * 8, 4), devs)
        before_sum = ph.gather()
        om = eng.QmfState.zeros(6)
        before = ph.expect(om)
        new_map = ph.rebalance(1.5)
        assert new_map.owner == [int(o) for o in want]
        loads = ph.worker_loads()
        assert max(loads) / max(1, min(loads)) <= 1.5
        assert ph.expect(om) == pytest.approx(before, abs=1e-12)
        after = ph.gather()  # migrated shards keep their contents
        assert np.array_equal(after.rows, before_sum.rows) and np.array_equal(after.coeffs, before_sum.coeffs)
        # a dressing step after the migration still equals the reference
        g = np.zeros(2, np.uint64)
        g[0] = np.uint64(0b000011)
        g[1] = np.uint64(0b000001)
        wd, sizes, log, mask = port.parallel_dress(h, bits, want, 4, g, 0.4, 0.0)
        ph.dress(eng.DressOp(eng.PauliWord(6, g), 0.4), 0.0)
        assert same_sum(ph.gather(), wd)
    rng = port.rng(659)
    h = rng.sum(6, 120)
    pm = pmap_of(eng, port, h, 3, 4)
    ph = eng.distribute(host(eng, h), pm)
    loads = ph.worker_loads()
    ratio = max(loads) / max(1, min(loads))
    assert ph.rebalance(max(2.0, ratio + 0.5)).owner == pm.owner
    with pytest.raises(ValueError):
        ph.rebalance(1.0)


@pytest.mark.parametrize("n,terms,m,workers", [(124, 60_000, 3, 4), (200, 20_000, 2, 2), (64, 40_000, 4, 2)])
def test_gmol_partitioned_sequence(eng, port, n, terms, m, workers):
    """Overpartitioned dressing sequence on molecular-like sums: 2^m shards
    on `workers` workers, compress after every step, against the serial
    reference pipeline."""
    rs = np.random.default_rng(11 + n)
    h = port.gen_mol(n, terms, 2)
    bits, _ = port.choose_partition_bits(h, m)
    owner = [p % workers for p in range(1 << m)]
    B = (n + 63) // 64
    gens, taus = [], []
    for k in range(5):
        row = np.zeros(2 * B, np.uint64)
        b0 = int(bits[k % m])  # every step flips a partition bit
        q = b0 if b0 < n else b0 - n
        qs = [q] + [int(x) for x in rs.choice([i for i in range(n) if i != q], 2, replace=False)]
        for j, qq in enumerate(qs):
            row[qq // 64] |= np.uint64(1 << (qq % 64))
            if j == 1 or (b0 >= n and j == 0):
                row[B + qq // 64] |= np.uint64(1 << (qq % 64))
        gens.append(row)
        taus.append(float(rs.uniform(-0.3, 0.3)))
    eps, cap = 1e-9, int(terms * 1.1)
    want, _ = port.dress_sequence(h, np.stack(gens), taus, eps, cap)
    for devs in device_layouts(workers):
        ph = eng.distribute(host(eng, h), eng.PartitionMap(n, [int(b) for b in bits], owner, workers), devs)
        masks = []
        for g, t in zip(gens, taus):
            st = eng.ParallelDressStats()
            ph.dress(eng.DressOp(eng.PauliWord(n, g), t), eps, cap, None, st)
            masks.append(st.mask)
        assert all(mk != 0 for mk in masks)
        assert same_sum(ph.gather(), want)


def test_merge_sums_matches_reference(eng, port):  # pauli.hpp:383-415 (test_pauli.cpp seed 37)
    rng = port.rng(37)
    for t in range(30):
        n = 2 + t % 6
        a, b = rng.sum(n, 40), rng.sum(n, 40)
        for drop in (1e-12, 0.0, 0.3):
            want = port.merge_sums(a, b, drop)
            got = eng.merge_sums(host(eng, a), host(eng, b), eng.MergeOptions(drop, True))
            assert same_sum(got, want)
    # cancellation to exactly zero and the identity kept under any threshold
    P = eng.PauliWord.from_string
    x = eng.PauliSum(2, np.stack([P("II").row, P("ZI").row]), [1e-20, 0.5])
    y = eng.PauliSum(2, np.stack([P("II").row, P("ZI").row, P("XI").row]), [1e-20, -0.5, 0.25])
    got = eng.merge_sums(x, y, eng.MergeOptions(0.1, True))
    assert len(got) == 2 and got.word(0).is_identity() and got.coeff(0).real == 2e-20
    got = eng.merge_sums(eng.PauliSum(2), y, eng.MergeOptions(0.1, True))
    assert len(got) == 3 and got.word(0).is_identity()  # XI (0.25) and ZI pass 0.1 too
