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


# ---- the exchange in the library itself (NCCL bound in C++) --------------------

def test_native_nccl_single_rank_and_event_timeline():
    """esdg_b200_solver_create_nccl with world_size 1 (all a one-GPU box can
    run): NCCL is bound at run time, the communicator comes up, the solver
    steps, and the RankEvents timeline of a recorded RHS is ordered."""
    uid = capi.nccl_unique_id()
    assert len(uid) == 128 and any(uid)
    mesh = capi.Mesh(capi.bubble_mesh_config(2, False))
    s = capi.GpuSolver(mesh, 4, "f64", nccl=(1, 0, 0, uid))
    assert capi.lib().esdg_b200_solver_nccl_version(s.h) >= 21800
    s.init_case(capi.CASE_BUBBLE_SHARP)
    ref = capi.GpuSolver(mesh, 4, "f64")
    ref.init_case(capi.CASE_BUBBLE_SHARP)
    dt = ref.compute_dt(0.5)
    s.record_events(True)
    for _ in range(3):
        s.step(dt)
        ref.step(dt)
    assert np.array_equal(s.get_state(), ref.get_state())
    ev = s.rank_events()
    assert 0 <= ev["volume_start_ns"] < ev["volume_end_ns"]
    assert s.halo_bytes == 0


@pytest.mark.parametrize("path", [capi.PATH_SPLIT, capi.PATH_FUSED, capi.PATH_STAGE])
def test_delayed_exchange_overlap_and_results(path):
    """The GPU analogue of tests/test_partition.cpp:116-152: with the trace
    transfer held back (esdg_b200_solver_set_exchange_delay, the counterpart
    of Transport::send_hook) the kernel that needs no ghost trace -- the
    volume kernel, or the one-pass kernel over the element groups without a
    ghost face -- starts BEFORE the last trace arrives, the ghost-face work
    waits for it, and the results are bitwise those of the undelayed run.
    Recorded with CUDA events on the partitions' own streams."""
    mesh = capi.Mesh(capi.bubble_mesh_config(3, False))
    s = capi.GpuSolver(mesh, 4, "f64", ranks=4)
    s.set_path(path)
    s.init_case(capi.CASE_BUBBLE_SHARP)
    one = capi.GpuSolver(mesh, 4, "f64")
    one.set_path(path)
    one.init_case(capi.CASE_BUBBLE_SHARP)
    dt = one.compute_dt(0.5)
    s.step(dt)                      # warm
    one.step(dt)
    s.set_exchange_delay(3000)      # 3 ms per RHS, a kernel takes ~50 us here
    s.record_events(True)
    s.step(dt)
    one.step(dt)
    assert np.array_equal(s.get_state(), one.get_state())
    assert s.halo_bytes > 0
    for r in range(4):
        ev = s.rank_events(r)
        assert ev["sends_posted_ns"] > 0, ev
        assert ev["last_arrival_ns"] >= 3_000_000, ev
        assert ev["sends_posted_ns"] <= ev["volume_start_ns"] < ev["last_arrival_ns"], ev
        assert ev["volume_end_ns"] < ev["last_arrival_ns"], ev      # the whole kernel hid behind the transfer
        assert ev["wait_end_ns"] >= ev["last_arrival_ns"], ev
    s.set_exchange_delay(0)
    s.step(dt)
    one.step(dt)
    assert np.array_equal(s.get_state(), one.get_state())


def _n_devices():
    return capi.lib().esdg_b200_device_count()


@pytest.mark.parametrize("path", [capi.PATH_SPLIT, capi.PATH_STAGE])
def test_partitions_on_several_devices_bitwise(path):
    """In-process partitions on DIFFERENT GPUs (traces by cudaMemcpyPeerAsync
    over NVLink): bitwise the one-device result. Needs >= 2 devices."""
    n = _n_devices()
    if n < 2:
        pytest.skip("one GPU visible")
    mesh = capi.Mesh(capi.bubble_mesh_config(3, False))
    one = capi.GpuSolver(mesh, 4, "f64")
    one.set_path(path)
    one.init_case(capi.CASE_BUBBLE_SHARP)
    dt = one.compute_dt(0.5)
    for _ in range(5):
        one.step(dt)
    for parts in sorted({2, min(4, n), min(8, n)}):
        s = capi.GpuSolver(mesh, 4, "f64", ranks=parts, devices=list(range(parts)))
        s.set_path(path)
        s.init_case(capi.CASE_BUBBLE_SHARP)
        for _ in range(5):
            s.step(dt)
        assert np.array_equal(s.get_state(), one.get_state()), parts


@pytest.mark.parametrize("precision", [8, 4])
def test_nccl_exchange_routine_against_itself(precision):
    """The C++ exchange routine of the process-per-GPU path (NcclTransport::
    exchange: one ncclRecv / ncclSend pair per peer block in one group on a
    stream) on a one-rank communicator, both peer blocks addressed to rank 0:
    everything of the NCCL data plane a one-GPU box can execute -- run-time
    binding of libnccl.so.2, communicator, grouped point-to-point on the
    library's own stream, the byte layout of the blocks."""
    import ctypes as C
    bad = C.c_int64(-1)
    rc = capi.lib().esdg_b200_nccl_selftest(0, precision, 5 * 25 * 1000 + 3, C.byref(bad))
    assert rc == 0, capi.lib().esdg_b200_last_message().decode()
    assert bad.value == 0


def _nccl_worker(rank, world, path, out_dir):
    torch.cuda.set_device(rank)
    id_file = os.path.join(out_dir, "nccl_id.bin")
    if rank == 0:
        with open(id_file + ".tmp", "wb") as f:
            f.write(capi.nccl_unique_id())
        os.replace(id_file + ".tmp", id_file)
    else:
        import time
        while not os.path.exists(id_file):
            time.sleep(0.01)
    uid = open(id_file, "rb").read()
    mesh = capi.Mesh(capi.bubble_mesh_config(3, False))
    s = capi.GpuSolver(mesh, 4, "f64", nccl=(world, rank, rank, uid))
    s.set_path(path)
    s.init_case(capi.CASE_BUBBLE_SHARP)
    dt = 0.0621602889129292      # compute_dt(0.5) of the whole mesh
    s.record_events(True)
    for _ in range(5):
        s.step(dt)
    np.save(os.path.join(out_dir, f"q{rank}.npy"), s.get_state())
    np.save(os.path.join(out_dir, f"ev{rank}.npy"), np.array(list(s.rank_events().values())))
    del s


@pytest.mark.parametrize("path", [capi.PATH_SPLIT, capi.PATH_STAGE])
def test_native_nccl_processes_bitwise(tmp_path, path):
    """One process per GPU, traces by ncclSend/ncclRecv issued from C++ (no
    Python inside step): the union of the ranks' states equals the one-process
    state bitwise (tests/test_partition.cpp:94-114). Needs >= 2 devices."""
    n = _n_devices()
    if n < 2:
        pytest.skip("one GPU visible")
    world = min(n, 4)
    mp.spawn(_nccl_worker, args=(world, path, str(tmp_path)), nprocs=world, join=True)
    mesh = capi.Mesh(capi.bubble_mesh_config(3, False))
    one = capi.GpuSolver(mesh, 4, "f64")
    one.set_path(path)
    one.init_case(capi.CASE_BUBBLE_SHARP)
    for _ in range(5):
        one.step(0.0621602889129292)
    got = np.concatenate([np.load(tmp_path / f"q{r}.npy") for r in range(world)])
    assert np.array_equal(got, one.get_state())
