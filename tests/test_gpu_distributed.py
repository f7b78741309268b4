"""One process per partition on a GPU box (-m gpu): the distributed solver
(esdg_b200_solver_create_distributed + the torch.distributed exchange
callback bench.py uses) against the single-process solver, bitwise. Only one
GPU is available, so both ranks share cuda:0 and the traces are staged through
the host over gloo; the device-side path (pack kernel, ghost-face reads,
callback ordering on the solver's stream) is exactly the NCCL one."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pyoracle as po
from paper_2605_16684_b200 import capi, halo

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port_no, path, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        mesh = capi.Mesh(capi.bubble_mesh_config(1, True))
        s = capi.GpuSolver(mesh, 3, "f64", distributed=(world, rank, 0))
        cb, ex = halo.make_exchange_callback(s, 0)
        s.exchange_impl = cb
        s.set_path(path)
        ora = po.Oracle("port")
        q = ora.mesh(po.bubble_mesh_config(1, True)).solver(3, "f64").init_case(po.CASE_ENTROPY_TEST, 31)
        s.set_state(q[s.begin:s.end].copy())
        s.rhs(0.0, 1.0)
        k = s.get_state(capi.REG_K)
        for _ in range(3):
            s.step(1e-3)
        np.save(os.path.join(out_dir, f"k{rank}.npy"), k)
        np.save(os.path.join(out_dir, f"q{rank}.npy"), s.get_state())
        assert ex.exchanges == 1 + 15 and ex.staged
        ex.close()          # before the solver (and its stream) goes away
        s.exchange_impl = None
        del s
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("path", [capi.PATH_SPLIT, capi.PATH_STAGE])
def test_two_processes_equal_one(tmp_path, path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), path, str(tmp_path)), nprocs=world, join=True)
    ora = po.Oracle("port")
    q = ora.mesh(po.bubble_mesh_config(1, True)).solver(3, "f64").init_case(po.CASE_ENTROPY_TEST, 31)
    g = capi.GpuSolver(capi.Mesh(capi.bubble_mesh_config(1, True)), 3, "f64")
    g.set_path(path)
    g.set_state(q.copy())
    g.rhs(0.0, 1.0)
    k = g.get_state(capi.REG_K)
    for _ in range(3):
        g.step(1e-3)
    got_k = np.concatenate([np.load(tmp_path / f"k{r}.npy") for r in range(world)])
    got_q = np.concatenate([np.load(tmp_path / f"q{r}.npy") for r in range(world)])
    assert np.array_equal(got_k, k)
    assert np.array_equal(got_q, g.get_state())
