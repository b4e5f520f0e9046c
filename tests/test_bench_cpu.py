"""Host logic of bench.py (no GPU): the per-N layouts, the --gpus self-spawn
(one process per GPU through torch.distributed.run on 127.0.0.1) and the
world-size check, and the reference analytics used by the bench lines."""
import argparse
import importlib.util
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def args(**kw):
    d = dict(grid=None, mtiles=0, ktiles=0, ntiles=0)
    d.update(kw)
    return argparse.Namespace(**d)


@pytest.mark.parametrize("P,grid,tn", [(1, (1, 1), 128), (2, (1, 2), 64), (4, (1, 4), 32),
                                      (8, (1, 8), 16)])
def test_spmm_layout_splits_columns(bench, P, grid, tn):
    (pr, pc), (tm, tk, tn_) = bench.layout(bench.CONFIGS["cfg3"], P, args())
    assert (pr, pc) == grid and pr * pc == P
    assert tm == 1 << 22 and tk == -(-(1 << 22) // P) and tn_ == tn


def test_spgemm_layout_square(bench):
    for P, want in [(1, (1, 1)), (2, (2, 1)), (4, (2, 2)), (8, (4, 2))]:
        (pr, pc), _ = bench.layout(bench.CONFIGS["cfg4"], P, args())
        assert (pr, pc) == want


def test_grid_override(bench):
    (pr, pc), (tm, tk, tn) = bench.layout(bench.CONFIGS["cfg3"], 4, args(grid="2x2"))
    assert (pr, pc) == (2, 2) and tn == 64


def test_self_spawn_builds_a_torchrun_command(bench, monkeypatch):
    seen = {}

    def fake_call(cmd):
        seen["cmd"] = cmd
        return 0

    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "5"])
    assert bench.self_spawn(4) == 0
    cmd = seen["cmd"]
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "5"]


def test_main_spawns_when_not_under_torchrun(bench, monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2"])
    monkeypatch.setattr(bench, "self_spawn", lambda n: 7 if n == 2 else 1)
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert e.value.code == 7


def test_world_size_must_match(bench, monkeypatch):
    pytest.importorskip("torch")
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4"])
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert "WORLD_SIZE=2" in str(e.value.code)


def test_p2p_peak_reads_committed_measurement(bench):
    gbs, src = bench.p2p_peak()
    assert gbs > 100 and ("measured" in src or "nominal" in src)


def test_time_imbalance_matches_flop_definition():
    sys.path.insert(0, ROOT)
    from paper_2311_18141_b200.analytics import imbalance_from_flops, imbalance_from_times

    t = np.array([[1.0, 3.0], [1.0, 1.0]])
    r = imbalance_from_times(t)
    f = imbalance_from_flops(t)
    assert r["per_stage_time_imbalance"] == f["per_stage_flop_imbalance"] == pytest.approx(
        4.0 / 3.0)
    assert r["end_to_end_time_imbalance"] == pytest.approx(4.0 / 3.0)
