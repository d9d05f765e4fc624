"""Sharded engine (2-3 ranks, may share one GPU) against the single-GPU engine:
every StepReport counter summed over ranks, and every rank's own lanes
bit-identical (membership, order, road_pos, s, v) every 10 steps."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _launch(name, steps, nproc, port, mode="", env=None, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "dist", "shard_worker.py"), name, str(steps)] + ([mode] if mode else [])
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT,
                          env=dict(os.environ, **(env or {})))


def _run(name, steps, nproc, port, mode="", env=None, timeout=600):
    out = _launch(name, steps, nproc, port, mode, env, timeout)
    line = [x for x in out.stdout.splitlines() if x.startswith("SHARD_RESULT")]
    assert line, out.stdout[-3000:] + out.stderr[-3000:]
    print(line[0])
    assert "mismatches=0" in line[0], out.stdout[-3000:]
    return line[0]


@pytest.mark.parametrize("name,steps,nproc,port", [("grid6x2", 300, 2, 29611), ("dense", 200, 2, 29612),
                                                   ("grid8x3", 300, 3, 29613)])
def test_sharded_equals_single(name, steps, nproc, port):
    _run(name, steps, nproc, port)


@pytest.mark.parametrize("name,steps,nproc,port", [("grid6x2", 120, 2, 29621), ("grid8x3", 120, 3, 29623)])
def test_sharded_p2p_equals_single(name, steps, nproc, port):
    """The device-driven exchange (pack into CUDA IPC-mapped peer slots,
    release/acquire flags, no host synchronisation per step), ranks sharing
    one GPU: same result as the single engine."""
    assert "p2p_used=1" in _run(name, steps, nproc, port, "p2p")


@pytest.mark.parametrize("name,steps,nproc,port,mode", [("grid6x2mp", 300, 2, 29651, ""),
                                                        ("grid8x3mp", 200, 3, 29652, "p2p")])
def test_sharded_max_pressure(name, steps, nproc, port, mode):
    """Max-pressure signals sharded (signals.py:64-86): each rank advances the
    junctions its vehicles may read at the start of the next step, from its own
    lanes' post-sweep counts and the owners' counts of the other pressure
    lanes (shard.pressure_lanes), exchanged with the ghosts -- own lanes,
    every counter and the merged queries equal the single engine's."""
    _run(name, steps, nproc, port, mode)


@pytest.mark.parametrize("name,steps,nproc,port", [("grid8x3", 150, 3, 29661), ("dense", 150, 2, 29662)])
def test_sharded_global_lane_numbering(name, steps, nproc, port):
    """The sharded engine on the whole network's lane numbering (no local
    renumbering, tsb_create_sharded): same result as the single engine."""
    _run(name, steps, nproc, port, env={"TSB_SHARD_GLOBAL_LANES": "1"})


def test_sharded_p2p_fallback_when_a_rank_cannot_map():
    """A rank that cannot map its peers makes every rank fall back to the
    collective transport; results unchanged."""
    line = _run("grid6x2", 60, 2, 29631, "p2p", env={"TSB_P2P_FAIL_RANK": "1"})
    assert "p2p_used=0" in line


def test_sharded_m1_two_ranks_p2p():
    """The bench workload (M1: 100x100x3 grid, 1M vehicles) split into 2 lane
    bands, ranks sharing one GPU, device-driven exchange: every StepReport
    counter summed over ranks each step and every rank's own lanes bit for bit
    against the single engine, 10 steps (the bulk injection included)."""
    assert "p2p_used=1" in _run("m1", 10, 2, 29641, "p2p", timeout=1200)


def test_sharded_p2p_peer_stall_fails_loudly():
    """A rank that stops stepping: its peer's bounded device-side wait ends
    the step and the engine raises EngineError (TSB_ECUDA) instead of hanging."""
    out = _launch("stall", 0, 2, 29651, timeout=300)
    line = [x for x in out.stdout.splitlines() if x.startswith("STALL_RESULT")]
    assert line, out.stdout[-3000:] + out.stderr[-3000:]
    assert "ok=1" in line[0], line[0]
