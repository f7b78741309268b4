"""N > 1 data path on CPU: two processes (gloo), each owning one Morton
partition. They exchange face traces with the SAME halo lists and the SAME
HaloExchange class bench.py uses over NCCL, then assemble their share of the
RHS with the oracle; the union must equal the serial RHS bitwise
(reference: tests/test_partition.cpp:94-114). CPU only."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pyoracle as po
from paper_2605_16684_b200 import capi
from paper_2605_16684_b200.halo import HaloExchange


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port_no, order, steps, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ora = po.Oracle("port")
        omesh = ora.mesh(po.bubble_mesh_config(1, True))
        s = omesh.solver(order, "f64")
        q = s.init_case(po.CASE_ENTROPY_TEST, 31)          # full state; only our range is used
        halo = capi.rank_halo(capi.Mesh(capi.bubble_mesh_config(1, True)), world, rank)
        b, e = halo["begin"], halo["end"]
        n2 = (order + 1) ** 2
        tl = 5 * n2
        ng = len(halo["send_elem"])
        send, recv = torch.zeros(ng * tl, dtype=torch.float64), torch.zeros(ng * tl, dtype=torch.float64)
        ex = HaloExchange(halo["peers"], tl, send, recv)
        face_of = omesh.face_of
        slot_of = -np.ones(omesh.nfaces, np.int32)
        for g in range(ng):
            slot_of[face_of[b + halo["send_elem"][g], halo["send_face"][g]]] = g
        a_coef, b_coef, _ = ora.lsrk()
        k = s.kreg
        dt = 1e-3
        for step in range(max(1, steps)):
            for st in range(5 if steps else 1):
                # K4 on the CPU: the pack kernel's gather, slot by slot
                for g in range(ng):
                    lf = int(halo["send_face"][g])
                    send[g * tl:(g + 1) * tl] = torch.from_numpy(
                        s.extract_trace(q, b + int(halo["send_elem"][g]), lf // 2, lf % 2).ravel())
                ex.begin()
                ex.end()
                ghost = recv.numpy().reshape(ng, 5, n2)
                if steps:
                    s.assemble_rhs_rank(q, k, a_coef[st], dt, b, e, slot_of, ghost)
                    q[b:e] += b_coef[st] * k[b:e]
                else:
                    s.assemble_rhs_rank(q, k, 0.0, 1.0, b, e, slot_of, ghost)
        np.save(os.path.join(out_dir, f"part{rank}.npy"), (q if steps else k)[b:e])
        assert ex.exchanges == (5 * steps if steps else 1)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("steps", [0, 2])
def test_two_ranks_gloo_bitwise_serial(tmp_path, steps):
    order, world = 3, 2
    mp.spawn(_worker, args=(world, _free_port(), order, steps, str(tmp_path)), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"part{r}.npy") for r in range(world)])
    ora = po.Oracle("port")
    s = ora.mesh(po.bubble_mesh_config(1, True)).solver(order, "f64")
    q = s.init_case(po.CASE_ENTROPY_TEST, 31)
    if steps:
        for _ in range(steps):
            s.step(1e-3)
        want = s.state
    else:
        want = s.assemble_rhs(q.copy())
    assert np.array_equal(got, want)
