"""Multi-GPU parity (needs >= 2 GPUs): runs tools/dist_check.py under torchrun.

Bitwise smoother apply on generated row blocks and bitwise V-cycles of a
row-partitioned native hierarchy against the C oracle; distributed PCG/FCG
iteration counts equal to the oracle's (+-1 bar) -- for each halo transport:
NCCL send/recv and the direct NVLink transport (default).
"""

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu


def ngpus():
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:
        return 0


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_dist_check(nproc, grid, graph, transport):
    if ngpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(REPO, "tools", "dist_check.py"), "--grid", str(grid)]
    if graph:
        cmd.append("--graph")
    env = dict(os.environ)
    env["AMGP_HALO"] = "nccl" if transport == "nccl" else "p2p"
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    lines = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == nproc, p.stdout[-2000:] + p.stderr[-2000:]
    for rec in lines:
        assert rec["ok"], rec
    assert p.returncode == 0


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
@pytest.mark.parametrize("graph", [False, True])
def test_dist_check_two_gpus(graph, transport):
    # 24^3: every distributed matrix has < 2 slices per SM per rank -> the
    # single halo-aware launch after the exchange (rows.cuh launch_rows)
    run_dist_check(2, 24, graph, transport)


@pytest.mark.parametrize("nproc", [2, 4])
@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_dist_check_split_launches(nproc, transport):
    # 48^3: the fine level holds >= 2 slices per SM per rank -> interior
    # launch, exchange, boundary launch
    run_dist_check(nproc, 48, True, transport)


def run_dsetup_check(nproc, args):
    if ngpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(REPO, "tools", "dsetup_dist_check.py")] + args
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    lines = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:] + p.stderr[-3000:]
    assert lines[0]["ok"], lines[0]
    assert p.returncode == 0


@pytest.mark.parametrize("args", [["--grid", "32"], ["--grid", "32", "--kind", "pairwise_matching"],
                                  ["--grid", "48", "--replicate-below", "20000"], ["--grid", "20", "--stencil", "27"]])
def test_distributed_device_setup_two_gpus(args):
    """Decoupled distributed device setup == the reference's formulas on the
    gathered blocks (bitwise), V-cycle bitwise vs the oracle on that
    hierarchy, PCG iterations within +-1 of the oracle and of the one-GPU
    (reference) hierarchy."""
    run_dsetup_check(2, args)


def test_distributed_device_setup_four_gpus():
    run_dsetup_check(4, ["--grid", "48"])
