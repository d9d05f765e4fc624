"""Step-by-step comparison of the GPU World with the CPU oracle (test helper)."""

from __future__ import annotations

import numpy as np

from oracle.bind import OracleWorld
from paper_2405_12520_b200 import World

FIELDS = (("vix", "vix"), ("lane", "lane"), ("rp", "road_pos"), ("s", "s"), ("v", "v"))


def compare_state(gpu: World, ref: OracleWorld, step: int, exact: bool = True, tol: float = 1e-4):
    a, b = gpu._state(), ref.state()
    assert np.array_equal(a["lane_start"], b["lane_start"]), f"step {step}: lane membership differs"
    for ka, kb in FIELDS:
        x, y = a[ka], b[kb]
        assert x.shape == y.shape, f"step {step}: {ka} shape {x.shape} vs {y.shape}"
        if exact or ka in ("vix", "lane", "rp"):
            if not np.array_equal(x, y):
                bad = np.nonzero(x != y)[0][:5]
                raise AssertionError(f"step {step}: field {ka} differs at {bad}: {x[bad]} vs {y[bad]}")
        else:
            err = np.max(np.abs(x - y) / np.maximum(1.0, np.abs(y))) if x.size else 0.0
            assert err <= tol, f"step {step}: {ka} max rel err {err}"


def compare_reports(gpu: World, ref: OracleWorld, step: int):
    r = ref.report()
    g = gpu._report
    for k in ("time", "step_no", "driving", "waiting", "finished", "dropped", "injected_now",
              "finished_now", "vehicle_updates"):
        assert getattr(g, k) == getattr(r, k), f"step {step}: report.{k} {getattr(g, k)} vs {getattr(r, k)}"


def run_pair(net, trips, config, seed, steps, exact=True, every=1, check_signals=True, debug=0, pow_mode=1):
    """GPU engine and CPU oracle in the same power arithmetic (1: glibc pow,
    what the reference computes; 0: correctly rounded), compared bit for bit."""
    gpu = World(net, trips, config, seed=seed, pow_mode=pow_mode)
    if debug:
        from paper_2405_12520_b200 import _native
        _native.check(_native.lib().tsb_set_debug(gpu._h, debug))
    ref = OracleWorld(net, trips, config, seed=seed, pow_mode=pow_mode)
    reverts = 0
    try:
        for k in range(1, steps + 1):
            gpu.step()
            ref.step(1)
            reverts += ref.report().reverts_last
            compare_reports(gpu, ref, k)
            if k % every == 0 or k == steps:
                compare_state(gpu, ref, k, exact=exact)
                if check_signals:
                    pg, eg = gpu.signal_state()
                    pr, er = ref.signal_state()
                    assert np.array_equal(pg, pr) and np.array_equal(eg, er), f"step {k}: signal state"
        assert gpu.finished == ref.finished_list(), "finished lists differ"
        st_g = gpu._state()["status"]
        st_r = ref.status()[0]
        assert np.array_equal(st_g, st_r), "vehicle status differs"
        return gpu, ref, reverts
    except Exception:
        gpu.close()
        ref.close()
        raise
