"""CPU tests of bench.py's multi-GPU launch logic (no GPU needed): --gpus N
without a launcher re-launches itself under torch.distributed.run with N
ranks on 127.0.0.1; under a launcher, a rank count that differs from --gpus
fails loudly."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_gpus_n_without_launcher_spawns_n_ranks(monkeypatch):
    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    with pytest.raises(SystemExit) as ei:
        bench.main()
    assert ei.value.code == 0
    (cmd,) = calls
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]


def test_launcher_rank_count_must_match(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "3")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2"])
    with pytest.raises(SystemExit) as ei:
        bench.main()
    assert "WORLD_SIZE=3" in str(ei.value.code)


def test_reference_structured_cpu_legs_run():
    """The BASELINE.md §4 legs on a small grid: the row-wise jacobi_reference
    on one pinned core and the run_dtb engine port at 1 and N threads."""
    legs = bench._reference_legs(96, 80)
    assert len(legs) >= 2
    assert legs[0]["cores"] == 1 and "jacobi_reference" in legs[0]["leg"]
    assert all(leg["value"] > 0 for leg in legs)
