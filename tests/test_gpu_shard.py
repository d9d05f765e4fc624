"""Sharded engine (2-3 ranks, may share one GPU) against the single-GPU engine:
every StepReport counter summed over ranks, and every rank's own lanes
bit-identical (membership, order, road_pos, s, v) every 10 steps."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(name, steps, nproc, port, mode=""):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "dist", "shard_worker.py"), name, str(steps)] + ([mode] if mode else [])
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    line = [x for x in out.stdout.splitlines() if x.startswith("SHARD_RESULT")]
    assert line, out.stdout[-3000:] + out.stderr[-3000:]
    print(line[0])
    assert "mismatches=0" in line[0], out.stdout[-3000:]


@pytest.mark.parametrize("name,steps,nproc,port", [("grid6x2", 300, 2, 29611), ("dense", 200, 2, 29612),
                                                   ("grid8x3", 300, 3, 29613)])
def test_sharded_equals_single(name, steps, nproc, port):
    _run(name, steps, nproc, port)


@pytest.mark.parametrize("name,steps,nproc,port", [("grid6x2", 120, 2, 29621), ("grid8x3", 120, 3, 29623)])
def test_sharded_p2p_equals_single(name, steps, nproc, port):
    """The device-driven exchange (pack into CUDA IPC-mapped peer slots,
    release/acquire flags, no host synchronisation per step), ranks sharing
    one GPU: same result as the single engine."""
    _run(name, steps, nproc, port, "p2p")
