"""bench.py at a small size on one GPU: the driver's JSON line contract
(device-resident value, roofline, e2e with calls in flight and its
one-at-a-time split, launch count, clocks) holds end to end."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_bench_small_line():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    r = subprocess.run([sys.executable, "bench.py", "--terms", "2e6", "--steps", "2", "--warmup", "3",
                        "--no-cpu", "--e2e-inflight", "3", "--e2e-pipe-steps", "2"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["metric"] == "pauli_terms_dressed_merged_per_s" and line["value"] > 0
    assert line["steps"] == 2 and line["warmup"] == 3 and line["n_gpus"] == 1
    assert line["gpu_launches"] > 0 and line["roofline"]["frac"] > 0
    e2e = line["e2e"]
    assert e2e["in_flight"] == 3 and e2e["steps"] == 6 and e2e["value"] > 0
    assert e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert e2e["sequential"]["value"] > 0 and set(e2e["sequential"]["split_ms_per_step"]) == {
        "upload", "dress", "download"}
