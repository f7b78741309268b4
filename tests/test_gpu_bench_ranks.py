"""bench.py's own multi-rank flow on a one-GPU box (-m gpu).

The driver launches `torchrun ... bench.py --gpus N` with one rank per GPU
over NCCL; NCCL refuses two ranks on one device, so with one GPU the same
file runs here with ESDG_BENCH_DIST_BACKEND=gloo: both ranks share cuda:0,
torch.distributed moves host tensors, the traces go through the
torch.distributed exchange callback. Everything else is the code the driver
runs: Morton partition per rank, dt by all-reduce, barrier + max-over-ranks
timing, rank 0 alone printing the line. (The solver-level two-process parity
tests are in test_gpu_distributed.py.)"""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, extra):
    env = dict(os.environ, ESDG_BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--gpus", str(world), "--steps", "2", "--warmup", "3", "--refinement", "2",
           "--no-cpu-baseline"] + extra
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]           # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_two_ranks_one_gpu(scaling):
    extra = ["--exchange", "torch"]
    if scaling == "strong":
        extra += ["--scaling", "strong", "--case", "baroclinic", "--refinement", "1"]
    line = _run(2, extra)
    assert line["n_gpus"] == 2 and line["steps"] == 2 and line["scaling"] == scaling
    cfg = line["config"]
    assert cfg["partition"] == "morton x2"
    halo = cfg["halo"]
    # every rank holds its Morton range only, and traces do move
    assert 0 < halo["local_elements"] < cfg["elements"]
    assert abs(halo["local_elements"] - cfg["elements"] / 2) <= 1
    assert halo["halo_bytes_per_rhs"] > 0 and halo["exchanges"] > 0
    assert halo["interior_kernel_started_before_last_recv"] in (True, False)
    # the order of kernel and exchange was chosen by timing both after the warm-up
    assert halo["overlap"]["selected_by"] == "auto" and halo["overlap"]["mode"] in ("on", "off")
    assert set(halo["overlap"]["probe_ms_per_step"]) == {"on", "off"}
    assert line["value"] > 0 and line["ms_per_step"] > 0
    assert line["gpu_launches"] >= 2 * 5
    assert line["e2e"]["value"] > 0 and line["e2e"]["coupled_value"] > 0
    # every rank streams its own Morton range of the ensemble's members
    assert "step_stream" in line["e2e"]["call"]
    assert line["e2e"]["h2d_bytes_per_step"] == halo["local_elements"] * 5 * (cfg["order"] + 1) ** 3 * 8


def test_bench_falls_back_when_nccl_cannot_pair_the_ranks():
    """--exchange nccl (the default) with two ranks on one device: the library's
    communicator cannot be created, every rank takes the torch.distributed
    exchange instead, and the run still partitions the mesh."""
    line = _run(2, [])
    halo = line["config"]["halo"]
    assert 0 < halo["local_elements"] < line["config"]["elements"]
    assert "torch.distributed" in halo["exchange"]


def test_bench_overlap_switch():
    """--overlap off: the kernel waits for the traces and runs as one launch;
    the event timeline of the report is still taken with the overlap on."""
    line = _run(2, ["--exchange", "torch", "--overlap", "off"])
    ov = line["config"]["halo"]["overlap"]
    assert ov["mode"] == "off" and ov["selected_by"] == "off" and set(ov["probe_ms_per_step"]) == {"off"}
    assert line["value"] > 0
