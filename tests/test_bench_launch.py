"""bench.py's multi-GPU launch contract (CPU only): `python bench.py --gpus N`
outside torchrun re-executes itself under torch.distributed.run with N ranks
(one process per GPU, 127.0.0.1 rendezvous); inside torchrun, or for N = 1 or
the reference arm, it runs in place."""
import argparse
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _args(gpus, impl="b200"):
    return argparse.Namespace(gpus=gpus, impl=impl, steps=2, warmup=3, no_cpu_baseline=False)


def test_relaunch_for_multi_gpu(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    argv = ["--gpus", "8", "--steps", "2"]
    cmd = bench.relaunch_command(_args(8), argv)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=8" in cmd and "127.0.0.1" in cmd
    assert cmd[-5:] == [os.path.abspath(bench.__file__), *argv]
    assert any(c.startswith("--master-port=") for c in cmd)


@pytest.mark.parametrize("gpus,impl,env", [(1, "b200", None), (4, "b200", "4"), (4, "reference", None)])
def test_no_relaunch(monkeypatch, gpus, impl, env):
    if env is None:
        monkeypatch.delenv("WORLD_SIZE", raising=False)
    else:
        monkeypatch.setenv("WORLD_SIZE", env)
    assert bench.relaunch_command(_args(gpus, impl), []) is None
