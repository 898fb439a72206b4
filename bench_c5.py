#!/usr/bin/env python3
"""bench_c5.py — SURVEY.md §8(d) C5 at its full size on the GPUs of one box.

G_mol(200, 4e8, seed 5) is split over N GPUs (one process per GPU, m =
log2 N partition bits from choose_partition_bits on the full sum), dressed
without a cap by DIS-like entanglers (seeded; every other one flips the
first partition bit, so products move over NVLink) until the global size
exceeds --target (1e9) terms, then compress_partitioned(eps = 1e-10,
max_terms = --target).  Rank 0 prints one JSON line: per dressing step the
global input/output size, the time (CUDA events on the engine stream, max
over ranks), the products exchanged and their wire bytes, and the
truncation time.  Synthetic data; nothing here reads /root/reference.

  python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \\
      --master-addr 127.0.0.1 --master-port 29512 bench_c5.py
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from bench import entangler  # noqa: E402  (same DIS-like entangler generator)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--terms", type=float, default=4e8)
    ap.add_argument("--target", type=float, default=1e9)
    ap.add_argument("--max-steps", type=int, default=12)
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    import torch
    import torch.distributed as dist
    from paper_2603_08883_b200 import iqcc, native

    torch.cuda.set_device(local)
    native.init(local)
    stream = torch.cuda.current_stream()
    native.set_stream(stream.cuda_stream)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = 200
    d = iqcc.DeviceSum.generate_mol(n, int(args.terms), 5)
    part = iqcc.Partition.setup(d, world, rank) if world > 1 else None
    if part is not None:  # the shards grow to ~1.5x target / N: map the peer buffers once
        part.reserve(d, int(1.6 * args.target / world))
    flip = None
    if part is not None and part.flip_qubit is not None:
        flip = (part.flip_qubit, part.flip_plane)

    def global_size():
        return part.total_size(d) if part else len(d)

    def tmax(ms):
        if world == 1:
            return ms
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    fams = ["classify", "present", "tile_agg", "carry", "rank", "partition", "merge", "exchange", "host_alloc",
            "host_wait", "select_gather", "select_digits", "host_p2p_prepare"]
    native.profile(True)  # per-family breakdown (CUDA events + host scopes) of every step
    steps = []
    size = global_size()
    k = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    while size <= args.target and len(steps) < args.max_steps:
        row, tau = entangler(n, 5000 + k, flip if k % 2 == 0 else None)
        k += 1
        gen = iqcc.PauliWord(n, row)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        native.profile_reset()
        e0.record(stream)
        if part:
            xs = part.dress(d, gen, tau, 0.0)  # no compress: grow uncapped
            sent, wire = xs.sent_terms, xs.bytes_wire
        else:
            d.dress(gen, tau, 1e-12)
            sent, wire = 0, 0
        e1.record(stream)
        torch.cuda.synchronize()
        ms = tmax(e0.elapsed_time(e1))
        new = global_size()
        if world > 1:
            t = torch.tensor([sent, wire], device="cuda", dtype=torch.float64)
            dist.all_reduce(t)
            sent, wire = int(t[0].item()), int(t[1].item())
        steps.append({"in": size, "out": new, "ms": round(ms, 3), "in_terms_per_s": size / (ms * 1e-3),
                      "exchanged": sent, "wire_bytes": wire,
                      "flip": bool(flip is not None and (k - 1) % 2 == 0),
                      "rank0_ms": {f: round(native.profile_get(f)[0], 2) for f in fams if native.profile_get(f)[0]}})
        size = new
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    if part:
        part.compress(d, 1e-10, int(args.target))
    else:
        d.compress(1e-10, int(args.target))
    e1.record(stream)
    torch.cuda.synchronize()
    cms = tmax(e0.elapsed_time(e1))
    kept = global_size()
    if rank == 0:
        print(json.dumps({"config": "C5", "n_qubits": n, "start_terms": int(args.terms), "n_gpus": world,
                          "steps": steps, "grown_to": size, "compress_ms": round(cms, 3), "kept": kept,
                          "compress_gbs": size * 72 / (cms * 1e-3) / 1e9 / world,
                          "note": "uncapped dressing to > target terms, then compress_partitioned(1e-10, target); "
                                  "ms = CUDA events on the engine stream, max over ranks"}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
