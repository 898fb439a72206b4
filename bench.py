#!/usr/bin/env python3
"""bench.py — Pauli terms dressed+merged per second for the iQCC dressing hot path.

Workload (BASELINE.json configs[2]): synthetic
G_mol(124 qubits, 1e8 terms, seed 2), DIS-like entanglers (weight 2-4 X/Y
words with odd #Y, tau ~ U(-0.2, 0.2), one seed per entangler), compress
(eps = 1e-10, max_terms = 1e8) after every dressing step.  One bench step is
one dress_sequence of 10 entanglers continuing on the evolving Hamiltonian
(iQCC keeps dressing the same H); W warm-up steps bring it to the capped
steady state.  The metric counts the logical input terms of every dressing
step (the reference's dress_single input size).

  value    device-resident: H stays in HBM, CUDA events on the engine's stream
  e2e      through the public API with HOST buffers: upload of the PauliSum
           from pinned host memory + dress_sequence (10 steps) + download of
           the dressed sum, every step; --e2e-inflight (default 3) calls in
           flight from as many host threads (one engine context each), so
           one call's H2D overlaps others' dressing and D2H; the one-call-
           at-a-time figure is kept under e2e.sequential; at N > 1 every
           rank uploads / dresses (partitioned) / downloads its shard, one
           call at a time, max over ranks
  roofline the merge kernel (dominant) against MEASURED_PEAKS.json hbm_gbs,
           algorithmic bytes (M_in + M_out) * (16 B + 8) per launch
  cpu_baseline  the UNMODIFIED reference (oracle/_ref, parallel_dress kThreaded)
           on a bounded sample of the same workload, rank 0 only

--impl reference times only that CPU reference arm.  N > 1 (torchrun): terms
are partitioned across ranks by the paper's bit-wise partitioning (see
DESIGN.md); each rank dresses its shard, products whose partition key flips
are exchanged over NCCL.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_QUBITS = 124
N_TERMS = 100_000_000
SEED_H = 2
EPS = 1e-10
ENTANGLERS_PER_STEP = 10
SAMPLE_TERMS = 2_000_000  # bounded CPU sample of the same workload


def blocks_for(n):
    return 1 if n == 0 else (n + 63) // 64


def entangler(n_qubits: int, index: int, flip=None):
    """DIS-like generator #index (odd-Y X/Y word of weight 2-4) and tau.
    flip = (qubit, plane) forces the letter on `qubit` to set that plane's
    bit, so the entangler flips that partition bit."""
    rs = np.random.default_rng([4, index])
    w = int(rs.integers(2, 5))
    qs = [int(q) for q in rs.choice(n_qubits, w, replace=False)]
    ys = [int(y) for y in rs.integers(0, 2, w)]
    if flip is not None:
        fq, plane = flip
        if fq not in qs:
            qs[0] = fq
        i = qs.index(fq)
        if plane == "z":
            ys[i] = 1
        if sum(ys) % 2 == 0:  # restore odd #Y on another position
            j = (i + 1) % w
            ys[j] ^= 1
    elif sum(ys) % 2 == 0:
        ys[-1] ^= 1
    B = blocks_for(n_qubits)
    row = np.zeros(2 * B, np.uint64)
    for q, y in zip(qs, ys):
        row[q // 64] |= np.uint64(1 << (q % 64))
        if y:
            row[B + q // 64] |= np.uint64(1 << (q % 64))
    tau = float(rs.uniform(-0.2, 0.2))
    return row, tau


def step_entanglers(n_qubits, step, flip=None):
    """10 entanglers; #0, #3 and #6 flip the first partition bit (SURVEY.md
    §8(d) C3: at least 3 of the 10 exercise the exchange)."""
    out = []
    for k in range(ENTANGLERS_PER_STEP):
        f = flip if (flip is not None and k in (0, 3, 6)) else None
        out.append(entangler(n_qubits, step * ENTANGLERS_PER_STEP + k, f))
    return out


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) >= 7:
                for nm, v in zip(names, r[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def profile_traffic():
    """DRAM bytes (read + write) per merge launch from the committed
    `ncu --set full` capture at this workload (profiles/merge_traffic.json),
    and which capture it came from."""
    path = os.path.join(ROOT, "profiles", "merge_traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        return float(t["dram_bytes_per_launch"]), t.get("capture")
    except Exception:
        return None, None


# ----------------------------------------------------------------- CPU arm
def cpu_reference(n_terms=SAMPLE_TERMS, steps=1, want_digest=False):
    """UNMODIFIED reference on a bounded sample: parallel_dress (kThreaded) over
    2^ceil(log2 nproc) partitions, 10 entanglers per step, compress each.
    want_digest: also return the SHA-256 of the reference's final sum (one
    step), which the GPU arm reproduces on the same sample."""
    from oracle.oracle import Oracle
    kind = "reference" if Oracle.available("reference") else "port"
    orc = Oracle(kind)
    h = orc.gen_mol(N_QUBITS, n_terms, SEED_H)
    nproc = os.cpu_count() or 1
    m = max(0, math.ceil(math.log2(nproc))) if kind == "reference" else 0
    total_terms, total_s = 0, 0.0
    dig = None
    for s in range(steps):
        ents = step_entanglers(N_QUBITS, s)
        gens = np.stack([e[0] for e in ents])
        taus = np.array([e[1] for e in ents])
        r = orc.time_dress_sequence(h, gens, taus, EPS, n_terms, m_bits=m, threads=nproc,
                                    want_out=want_digest and s == 0)
        secs, tin = r[0], r[1]
        if want_digest and s == 0:
            dig = sum_digest(*r[3].export())
        total_terms += tin
        total_s += secs
    out = {"value": total_terms / total_s, "unit": "terms/s", "cores": min(nproc, 1 << m) if m else 1,
            "kind": kind,
            "sample": f"G_mol({N_QUBITS}q, {n_terms:.0e} terms, seed {SEED_H}), {steps}x10 DIS-like "
                      f"entanglers, eps={EPS}, max_terms={n_terms}, parallel_dress kThreaded m={m}",
            "seconds": total_s}
    if want_digest:
        out["_digest"] = dig
    return out


def sum_digest(rows, coeffs):
    """SHA-256 of a sum's canonical bytes (reference row layout, complex
    coefficients by value: -0.0 == +0.0, as PauliSum == compares)."""
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(rows, np.uint64).tobytes())
    h.update((np.ascontiguousarray(coeffs, np.complex128).view(np.float64) + 0.0).tobytes())
    return h.hexdigest()


def gpu_sample_digest(iqcc):
    """The reference arm's exact sample dressed by the engine (one bench step
    of 10 entanglers with compress), for the in-bench parity check."""
    d = iqcc.DeviceSum.generate_mol(N_QUBITS, SAMPLE_TERMS, SEED_H)
    ents = step_entanglers(N_QUBITS, 0)
    ans = iqcc.Ansatz([iqcc.PauliWord(N_QUBITS, r) for r, _ in ents], [t for _, t in ents])
    d.dress_sequence(ans, EPS, SAMPLE_TERMS)
    out = d.download()
    return sum_digest(out.rows, out.coeffs)


def run_reference_arm(args, rank):
    if rank != 0:
        return
    base = cpu_reference(SAMPLE_TERMS, 1)  # warm the checker + first timing
    vals = []
    for _ in range(max(1, args.steps)):
        vals.append(cpu_reference(SAMPLE_TERMS, 1)["value"])
    v = float(np.mean(vals))
    line = {"impl": "reference", "metric": "pauli_terms_dressed_merged_per_s", "value": v,
            "unit": "terms/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * ENTANGLERS_PER_STEP * SAMPLE_TERMS / v, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C3 bounded CPU sample", "n_qubits": N_QUBITS, "terms": SAMPLE_TERMS,
                       "entanglers_per_step": ENTANGLERS_PER_STEP, "eps": EPS},
            "cpu_baseline": dict(base, value=v),
            "e2e": {"value": v, "unit": "terms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm
def run_gpu_arm(args, rank, world, local_rank):
    import torch
    from paper_2603_08883_b200 import iqcc, native

    torch.cuda.set_device(local_rank)
    native.init(local_rank)
    stream = torch.cuda.current_stream()
    native.set_stream(stream.cuda_stream)
    dist = None
    if world > 1:
        import torch.distributed as dist
    n_terms = int(args.terms)

    # ---- input (setup, not timed)
    d = iqcc.DeviceSum.generate_mol(N_QUBITS, n_terms, SEED_H)
    # the 8-GPU partition bits (greedy, prefix-consistent for m = 1, 2, 3)
    # fix which entanglers flip a partition bit, identically at every N
    bits8, _ = iqcc.choose_partition_bits(d, 3)
    b0 = bits8[0]
    flip = (b0, "x") if b0 < N_QUBITS else (b0 - N_QUBITS, "z")
    part = None
    if world > 1:
        part = iqcc.Partition.setup(d, world, rank)  # restrict to own shard, join NCCL
        assert (part.flip_qubit, part.flip_plane) == flip
    torch.cuda.synchronize()

    def dress_step(store, s):
        ents = step_entanglers(N_QUBITS, s, flip)
        ans = iqcc.Ansatz([iqcc.PauliWord(N_QUBITS, r) for r, _ in ents], [t for _, t in ents])
        if part:
            xl = []
            tin = part.dress_sequence(store, ans, EPS, n_terms, exchange=xl)
            sent[0] += sum(x.sent_terms for x in xl)
            return tin
        return store.dress_sequence(ans, EPS, n_terms)

    sent = [0]
    for w in range(args.warmup):
        dress_step(d, w)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()

    # ---- device-resident timed region
    # timed region with the engine's per-kernel event profiling OFF (its event
    # records sit on the host path between launches); a second, profiled pass
    # of the same length below gives the per-kernel breakdown and the merge
    # roofline
    native.profile(False)
    native.profile_reset()
    launches0 = native.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tin_total = 0
    sent[0] = 0
    with ClockSampler(local_rank) as clk:
        time.sleep(0.6)  # let nvidia-smi start sampling before the timed region
        torch.cuda.synchronize()
        e0.record(stream)
        w0 = time.perf_counter()
        for s in range(args.steps):
            tin_total += dress_step(d, args.warmup + s)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"[bench] wall {1e3 * (time.perf_counter() - w0):.1f} ms for {args.steps} steps", file=sys.stderr)
    launches = native.launch_count() - launches0
    step_bytes = native.profile_bytes("merge")  # (M_in + M_out) * S of every dressing step, timed pass
    native.profile(True)
    native.profile_reset()
    for s in range(args.steps):
        dress_step(d, args.warmup + args.steps + s)
    torch.cuda.synchronize()
    merge_ms, merge_n = native.profile_get("merge")
    fam = {f: native.profile_get(f)[0] for f in
           ["classify", "present", "tile_agg", "carry", "rank", "partition", "merge",
            "select_gather", "select_digits", "exchange", "host_wait", "host_dress", "host_compress", "span_dress", "span_compress", "host_alloc", "host_compress_inner", "spec_redo"]}
    for f in ["materialize", "exch_count", "exch_signal"]:
        fam[f] = native.profile_get(f)[0]
    # N > 1: time per dressing step by kind (mask != 0: products exchanged)
    steps_by_kind = {k: (lambda t: {"steps": t[1], "ms_per_step": t[0] / t[1] if t[1] else None})(
        native.profile_get(f)) for k, f in (("exchange", "step_exchange"), ("local", "step_local"))}
    native.profile(False)
    if dist:
        print(f"[bench] rank {rank}: shard {d.size()} terms, sent {sent[0]} products, ms {ms:.2f}, "
              f"host syncs {native.profile_get('host_wait')[1]}, tie gathers "
              f"{native.profile_get('host_tie_gather')[1]}, kernel_ms "
              + json.dumps({k: round(v, 2) for k, v in fam.items() if v}), file=sys.stderr)
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        # every rank reports the global input size of each step (the
        # partitioned call sums the shards); check they agree
        tt = torch.tensor([float(tin_total), -float(tin_total)], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        assert float(tt[0]) == -float(tt[1]) == float(tin_total), "ranks disagree on the global term count"
    value = tin_total / (ms / 1e3)

    # ---- roofline of the merge kernel (algorithmic bytes per launch)
    S = 16 * iqcc.blocks_for(N_QUBITS) + 8
    # per dressing step: logical in ~ current size, out ~ in + products (approx by stats)
    peak, peak_kind = measured_peaks()
    alg_bytes = native.profile_bytes("merge")
    achieved = alg_bytes / (merge_ms / 1e3) / 1e9 if merge_ms > 0 else 0.0
    traffic, traffic_src = profile_traffic()
    # whole dressing step (plan + merge + compress) against the same peak:
    # the timed pass's algorithmic bytes over its device time (per rank)
    step_achieved = step_bytes / (ms / 1e3) / 1e9 if ms > 0 else 0.0

    spec_redos = native.profile_get("spec_redo")[1]

    # ---- end-to-end through the public API with host buffers
    e2e = None
    if not args.no_e2e and world > 1:
        e2e = e2e_partitioned(iqcc, part, d, n_terms, args, dist)
    if not args.no_e2e and world == 1:
        h_host = d.download_pinned()
        out_bufs = iqcc.pinned_buffers(N_QUBITS, 2 * n_terms)
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        h2d = h_host.rows.nbytes + h_host.coeffs.nbytes
        tin_e2e, d2h = 0, 0
        split = {"upload": 0.0, "dress": 0.0, "download": 0.0}
        # one untimed end-to-end step first: the API's one-time host staging
        # (page-locked) and device buffer allocations, as the device-resident
        # region's warm-up steps do for the kernels
        ents = step_entanglers(N_QUBITS, args.warmup + 2 * args.steps + e2e_steps)  # not a timed step's
        ans = iqcc.Ansatz([iqcc.PauliWord(N_QUBITS, r) for r, _ in ents], [t for _, t in ents])
        dev = iqcc.DeviceSum.upload(h_host)
        dev.dress_sequence(ans, EPS, n_terms)
        dev.download(*out_bufs)
        del dev
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s in range(e2e_steps):
            ents = step_entanglers(N_QUBITS, args.warmup + 2 * args.steps + s)
            ans = iqcc.Ansatz([iqcc.PauliWord(N_QUBITS, r) for r, _ in ents], [t for _, t in ents])
            # iqcc.dress_sequence_counted in its three phases (each call ends
            # device-synchronous): H2D + upload check, the 10 steps, D2H
            ta = time.perf_counter()
            dev = iqcc.DeviceSum.upload(h_host)
            tb = time.perf_counter()
            tin = dev.dress_sequence(ans, EPS, n_terms)
            torch.cuda.synchronize()
            tc = time.perf_counter()
            out = dev.download(*out_bufs)
            td = time.perf_counter()
            del dev
            split["upload"] += tb - ta
            split["dress"] += tc - tb
            split["download"] += td - tc
            tin_e2e += tin
            d2h += out.rows.nbytes + out.coeffs.nbytes
        torch.cuda.synchronize()
        secs = time.perf_counter() - t0
        seq = {"value": tin_e2e / secs, "unit": "terms/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h // e2e_steps, "steps": e2e_steps,
               "ms_per_step": 1e3 * secs / e2e_steps,
               "split_ms_per_step": {k: round(1e3 * v / e2e_steps, 2) for k, v in split.items()},
               "h2d_wire_bytes_per_step": h2d - h_host.coeffs.nbytes // 2,
               "split_note": "upload = pinned H2D of the rows while host threads keep the real parts of the "
                             "complex coefficients (checking every imaginary part is zero), then H2D of those "
                             "and the device check/convert; download = device compaction to the reference "
                             "layout + D2H of the real parts (host threads widen them to complex while the "
                             "rows are on the wire) and of the rows (PCIe bound)",
               "d2h_wire_bytes_per_step": d2h // e2e_steps - (d2h // e2e_steps) // 6}
        del out_bufs
        e2e = dict(seq)
        if args.e2e_inflight > 1:
            # the calls in flight get the device to themselves: drop the
            # device-resident sum and this thread's context (its caches)
            d = None
            native.finalize_thread()
            native.init_thread(local_rank)
            pipe = e2e_pipelined(iqcc, native, h_host, n_terms, args.e2e_pipe_steps, args.e2e_inflight, local_rank,
                                 args.warmup + 2 * args.steps + e2e_steps + 1)
            e2e = {"value": pipe["value"], "unit": "terms/s", "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": pipe["d2h_bytes_per_step"], "steps": pipe["steps"],
                   "ms_per_step": pipe["ms_per_step"], "in_flight": args.e2e_inflight,
                   "h2d_wire_bytes_per_step": seq["h2d_wire_bytes_per_step"],
                   "d2h_wire_bytes_per_step": seq["d2h_wire_bytes_per_step"],
                   "note": f"{args.e2e_inflight} dress_sequence calls in flight (one host thread and engine "
                           "context each, native.init_thread): every step still uploads its H from pinned "
                           "host memory, dresses it 10x and downloads the result; one call's H2D overlaps "
                           "another's dressing and D2H (PCIe is full duplex). ms_per_step = wall time / "
                           "steps completed. The one-call-at-a-time figure is 'sequential'.",
                   "sequential": seq}

    if rank == 0:
        cpu = None if args.no_cpu else cpu_reference(SAMPLE_TERMS, 1, want_digest=True)
        parity = None
        if cpu is not None:
            # in-bench parity: the engine on the reference arm's exact sample
            # must reproduce the reference's final sum bit for bit
            parity = gpu_sample_digest(iqcc) == cpu.pop("_digest")
            if world > 1:  # the CPU baseline is an N=1 figure; the digest still pins parity here
                cpu = None
        line = {
            "metric": "pauli_terms_dressed_merged_per_s", "value": value, "unit": "terms/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic G_mol (SURVEY.md §8(d)); inputs 4 GB >> 126 MB L2 (no flush needed)",
            "config": {"workload": "C3: G_mol 124q 1e8 terms, 10 DIS-like entanglers per step, "
                                   "compress eps=1e-10 max_terms=1e8 after each",
                       "n_qubits": N_QUBITS, "terms": n_terms, "entanglers_per_step": ENTANGLERS_PER_STEP,
                       "eps": EPS, "max_terms": n_terms, "parallelism": f"bitwise-partition x{world}",
                       "l2": "inputs larger than L2"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "roofline": {"bound": "hbm", "kernel": "k_merge1", "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "traffic_source": traffic_src, "launches": merge_n,
                         "algorithmic_bytes": alg_bytes, "bytes_per_term": S},
            "step_roofline": {"bound": "hbm", "achieved": step_achieved, "peak": peak, "unit": "GB/s",
                              "frac": step_achieved / peak,
                              "note": "sum over dressing steps of (M_in + M_out) * S bytes / whole timed "
                                      "region (plan, merge, compress, host gaps) on rank 0"},
            "spec_redos": spec_redos,
            "kernel_ms": fam,
            "kernel_ms_note": "CUDA events per kernel family over a second, profiled pass of the same K steps (the timed pass runs with profiling off)",
            "dressing_steps_by_kind": steps_by_kind if world > 1 else None,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "parity": parity,
            "parity_note": "SHA-256 of the engine's result on the cpu_baseline sample (G_mol 124q 2e6, "
                           "10 entanglers, compress) == the unmodified reference's (null: --no-cpu)",
        }
        print(json.dumps(line), flush=True)


def e2e_partitioned(iqcc, part, d, n_terms, args, dist):
    """End to end at N > 1: every rank uploads its shard from pinned host
    memory, runs the partitioned dress_sequence (products exchanged over
    NVLink) and downloads its shard, one call at a time; the step time is
    the max over ranks, bytes are summed over ranks (whole job)."""
    import torch
    h_host = d.download_pinned()
    out_bufs = iqcc.pinned_buffers(N_QUBITS, 2 * max(len(h_host), 1))  # shards shift as products move
    steps = max(1, min(args.steps, args.e2e_steps))
    h2d = h_host.rows.nbytes + h_host.coeffs.nbytes

    def call(idx):
        ents = step_entanglers(N_QUBITS, idx, (part.flip_qubit, part.flip_plane))
        ans = iqcc.Ansatz([iqcc.PauliWord(N_QUBITS, r) for r, _ in ents], [t for _, t in ents])
        dev = iqcc.DeviceSum.upload(h_host)
        tin = part.dress_sequence(dev, ans, EPS, n_terms)
        out = dev.download(*out_bufs)
        del dev
        return tin, out.rows.nbytes + out.coeffs.nbytes

    base = args.warmup + 2 * args.steps
    call(base + 100)  # untimed: this shape's allocations and host staging
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    tin, d2h = 0, 0
    for s in range(steps):
        a, b = call(base + s)
        tin += a
        d2h += b
    secs = time.perf_counter() - t0
    t = torch.tensor([secs], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    byt = torch.tensor([float(h2d), float(d2h)], device="cuda", dtype=torch.float64)
    dist.all_reduce(byt)
    secs = float(t.item())
    return {"value": tin / secs, "unit": "terms/s", "h2d_bytes_per_step": int(byt[0].item()),
            "d2h_bytes_per_step": int(byt[1].item()) // steps, "steps": steps, "ms_per_step": 1e3 * secs / steps,
            "in_flight": 1,
            "note": "each rank uploads its shard from pinned host memory, dress_sequence over parallel_dress "
                    "steps (products exchanged over NVLink), downloads its shard; one call at a time; wall "
                    "time max over ranks, bytes summed over ranks"}


def e2e_pipelined(iqcc, native, h_host, n_terms, steps_per_thread, inflight, device, ent_base):
    """End-to-end throughput with `inflight` public-API calls in flight: each
    host thread owns an engine context (native.init_thread) and runs
    upload -> dress_sequence(10) -> download on its own steps; the timed
    region is the wall time from a common start until the last thread's
    last download has landed in host memory."""
    barrier = threading.Barrier(inflight + 1)
    done = threading.Barrier(inflight)
    res, errs = [None] * inflight, []
    bufs = [iqcc.pinned_buffers(N_QUBITS, n_terms) for _ in range(inflight)]

    # thread w starts once thread w-1's first upload has landed, so the calls
    # are staggered (in lock step they would contend for the same engine)
    uploaded = [threading.Event() for _ in range(inflight)]
    trace = []  # (thread, upload start, dress start, download start, end)

    def job(w, idx, first=False):
        ents = step_entanglers(N_QUBITS, idx)
        ans = iqcc.Ansatz([iqcc.PauliWord(N_QUBITS, r) for r, _ in ents], [t for _, t in ents])
        if first and w > 0:
            uploaded[w - 1].wait()
        ta = time.perf_counter()
        dev = iqcc.DeviceSum.upload(h_host)
        if first:
            uploaded[w].set()
        tb = time.perf_counter()
        tin = dev.dress_sequence(ans, EPS, n_terms)
        tc = time.perf_counter()
        out = dev.download(*bufs[w])
        td = time.perf_counter()
        del dev
        trace.append((w, ta, tb, tc, td))
        return tin, out.rows.nbytes + out.coeffs.nbytes

    def worker(w):
        try:
            native.init_thread(device)
            try:
                job(w, ent_base + 1000 + w)  # untimed: this context's allocations and host staging
                barrier.wait()
                tin, d2h = 0, 0
                for s in range(steps_per_thread):
                    a, b = job(w, ent_base + inflight * s + w, first=s == 0)
                    tin += a
                    d2h += b
                res[w] = (tin, d2h, time.perf_counter())
                done.wait()  # context teardown (device syncs, frees) only after every call has ended
            finally:
                native.finalize_thread()
        except BaseException as e:  # noqa: BLE001 - reported below
            errs.append(e)
            barrier.abort()
            done.abort()
            for ev in uploaded:
                ev.set()

    ths = [threading.Thread(target=worker, args=(w,)) for w in range(inflight)]
    for t in ths:
        t.start()
    try:
        barrier.wait()
    except threading.BrokenBarrierError:
        pass
    t0 = time.perf_counter()
    for t in ths:
        t.join()
    if errs:
        raise errs[0]
    secs = max(r[2] for r in res) - t0
    n = steps_per_thread * inflight
    if os.environ.get("IQCC_E2E_TRACE"):
        for w, ta, tb, tc, td in trace:
            print(f"[e2e] thread {w} upload {1e3 * (ta - t0):8.1f} dress {1e3 * (tb - t0):8.1f} "
                  f"download {1e3 * (tc - t0):8.1f} end {1e3 * (td - t0):8.1f} ms", file=sys.stderr)
    return {"value": sum(r[0] for r in res) / secs, "ms_per_step": 1e3 * secs / n, "steps": n,
            "d2h_bytes_per_step": sum(r[1] for r in res) // n}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--terms", type=float, default=N_TERMS)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-inflight", type=int, default=3,
                    help="public-API calls in flight for e2e (1: one call at a time only)")
    ap.add_argument("--e2e-pipe-steps", type=int, default=4, help="e2e steps per in-flight call")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank)
        return
    if world > 1:
        # NCCL's banner / INFO lines go to stderr: stdout carries the JSON line only
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_gpu_arm(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
