"""CPU tests of bench.py's launch contract: `--gpus N` outside torchrun re-executes
itself as N ranks (torch.distributed.run, 127.0.0.1), under torchrun WORLD_SIZE must
equal N, and the default workload is C3 at N = 1 and the point-sharded C5 at N > 1."""
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import bench  # noqa: E402


def _args(argv):
    old = sys.argv
    sys.argv = ["bench.py"] + argv
    try:
        return bench._args()
    finally:
        sys.argv = old


def test_default_workloads():
    assert _args([]).config == 3
    assert _args(["--gpus", "4"]).config == 5
    assert _args(["--schedule", "a1"]).config == 1
    assert _args(["--config", "2"]).config == 2


def test_relaunch_under_torchrun(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    seen = {}

    def fake_execv(path, cmd):
        seen["cmd"] = cmd
        raise SystemExit(0)

    monkeypatch.setattr(os, "execv", fake_execv)
    with pytest.raises(SystemExit):
        bench._relaunch_under_torchrun(_args(["--gpus", "2", "--steps", "3"]))
    cmd = seen["cmd"]
    assert "torch.distributed.run" in cmd and "--nproc-per-node=2" in cmd
    assert "--master-addr=127.0.0.1" in cmd and cmd[-2:] != []


def test_world_size_must_match(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    with pytest.raises(SystemExit):
        bench._relaunch_under_torchrun(_args(["--gpus", "4"]))
    monkeypatch.setenv("WORLD_SIZE", "1")
    bench._relaunch_under_torchrun(_args([]))  # N = 1 under a 1-rank launcher: fine
