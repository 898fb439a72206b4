"""Multi-GPU parity: bit-wise partitioned dressing with the
NCCL pairwise product exchange equals the serial reference pipeline bit for
bit (tests/test_partition.cpp:180-208 at the process level).  Needs >= 2
visible GPUs; launched with torchrun."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def n_gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("args", [("124", "2e5", "6", "1e-10", "2e5"), ("64", "1e5", "5", "0", "1e18"),
                                  ("124", "2e5", "7", "1e-10", "1.5e5", "seq"),
                                  ("124", "2e5", "7", "1e-10", "1.5e5", "seq", "badspec"),
                                  ("124", "2e5", "7", "1e-10", "1.5e5", "seq", "nccl"),
                                  ("124", "2e5", "7", "1e-10", "1.5e5", "seq", "pull"),
                                  ("124", "2e5", "7", "1e-10", "1.5e5", "seq", "pull", "badspec"),
                                  ("200", "1e5", "6", "1e-10", "1.2e5", "seq"),
                                  ("124", "1e6", "5", "1e-10", "8e5", "seq"),
                                  ("124", "1e6", "5", "1e-10", "8e5", "seq", "chunks16"),
                                  ("124", "1e6", "5", "1e-10", "8e5", "seq", "chunks16", "badspec"),
                                  ("124", "1e6", "5", "1e-10", "8e5", "seq", "chunks1"),
                                  ("124", "1e6", "5", "1e-10", "8e5", "seq", "smpush")])
def test_partitioned_dressing_matches_serial(world, args):
    """The sequence cases exercise the output-slot speculation on the
    exchange and the local steps; "badspec" forces every guess too high
    (IQCC_SPEC_SCALE), so every step is undone and redone exactly; the
    1e6-term cases are large enough for the chunked exchange to split the
    products (the partner's merge starts on chunk 0 while later chunks are
    on the wire; chunks16: many chunks, some empty; chunks1: one SM push
    then the merge); "nccl"
    moves the products with NCCL send/recv (the fallback of the CUDA-IPC
    NVLink push); "pull" lets the partner's merge read them in place over
    NVLink (IQCC_XCHG=pull)."""
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ)
    if args[-1] == "badspec":
        env["IQCC_SPEC_SCALE"] = "64"
        args = args[:-1]
    if args[-1] == "smpush":  # chunks leave through a 148-CTA SM push kernel beside the merge
        env["IQCC_XCHG_SM"] = "148"
        args = args[:-1]
    if args[-1].startswith("chunks"):  # exchange chunk count (1: one SM push, then the merge)
        env["IQCC_XCHG_CHUNKS"] = args[-1][6:]
        args = args[:-1]
    if args[-1] == "nccl":  # products over NCCL send/recv instead of the NVLink push
        env["IQCC_NO_P2P"] = "1"
        args = args[:-1]
    elif args[-1] == "pull":  # the partner's merge reads the products over NVLink
        env["IQCC_XCHG"] = "pull"
        args = args[:-1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tests", "multi_worker.py"),
           *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "bitexact=True" in r.stdout and "energy_ok=True" in r.stdout
    if os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libiqcc_ref.so")):
        assert "checker=reference" in r.stdout  # the unmodified reference is the checker


@pytest.mark.parametrize("world", [2])
def test_c5_script_small(world):
    """bench_c5.py (SURVEY.md §8(d) C5 across GPUs) at a small size: uncapped
    growth over the chunked exchange, receive buffers reserved up front, then
    compress_partitioned to the target; the kept count is the target."""
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    import json
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29534", os.path.join(ROOT, "bench_c5.py"),
           "--terms", "4e5", "--target", "1e6"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["grown_to"] > 1_000_000 and line["kept"] == 1_000_000
    assert any(s["exchanged"] > 0 for s in line["steps"])
