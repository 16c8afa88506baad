"""The bench's N > 1 path (torchrun, one process per rank, barrier + max over
ranks, strong scaling: one batch sharded into contiguous slices, the step ends
with the all-gather of the result slices) on the GPUs present: 2 ranks with the
gloo backend share the visible device(s).  (On an 8-GPU box the driver runs it
with NCCL.)"""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--dist-backend", "gloo", *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_two_ranks():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--steps", "3", "--warmup", "3", "--config", "rsa2048-enc", "--count", "65537", "--no-e2e"])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["packets_total"] == 65537 and d["config"]["packets_per_rank"] == 32769
    assert d["cpu_baseline"] is None and d["gpu_launches"] == 2 * 3 and d["gather_ms"] > 0


def test_bench_two_ranks_roundtrip_e2e():
    """The round trip, reassembled by the all-gather, equals the input batch
    (device path and the end-to-end host path through shard.modexp_sharded_host)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--steps", "3", "--warmup", "3", "--config", "rsa2048-roundtrip", "--count", "20001"])
    assert d["verified_roundtrip"] is True and d["e2e"]["verified"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 20001 * 256 and d["gpu_launches"] == 2 * 3 * 2
