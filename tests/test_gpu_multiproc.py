"""The multi-GPU data path through the CUDA library from SEPARATE PROCESSES.

Two processes (torch.distributed, gloo over 127.0.0.1) each own one z-slab
context of libnsfr_b200.so in external-halo mode and move the face-trace
planes between them with gloo send/recv -- the same routing exchange() does
over NCCL (rank r's send_lo -> rank r-1's recv_hi, send_hi -> rank r+1's
recv_lo) -- plus the lambda MAX allreduce for the global dt. The gathered RHS
and three RK4 steps must equal one whole-box context BITWISE.

This pool has one GPU per box, so both ranks share cuda:0. Their kernels
never wait on each other: every exchange is host-side (gloo), between
complete stages, so the ranks run as on two GPUs, only serialised.
"""
import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

P_DEG, M, STEPS = 3, 6, 3
C1D = 0.5 * 3.80e-3


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _swap(dist, g, rank, world):
    """Exchange the z-halo planes with the two ring neighbours over gloo."""
    import torch
    send_lo, send_hi = (torch.from_numpy(np.ascontiguousarray(x)) for x in g.halo_get())
    recv_lo, recv_hi = torch.empty_like(send_lo), torch.empty_like(send_hi)
    lo, hi = (rank - 1) % world, (rank + 1) % world
    ops = [dist.P2POp(dist.isend, send_lo, lo), dist.P2POp(dist.irecv, recv_hi, hi),
           dist.P2POp(dist.isend, send_hi, hi), dist.P2POp(dist.irecv, recv_lo, lo)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    g.halo_set(recv_lo.numpy(), recv_hi.numpy())


def _worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist

    import paper_2312_07725_b200 as pkg
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = pkg.GpuSolver(pkg.SolverConfig(p=P_DEG, m=M, c1d=C1D, rank=rank, nranks=world, device=0))
    g.init_case()
    g.project()
    _swap(dist, g, rank, world)
    rhs = g.residual()
    lams, dts = [], []
    for _ in range(STEPS):
        lam = torch.tensor([g.max_wavespeed()], dtype=torch.float64)
        dist.all_reduce(lam, op=dist.ReduceOp.MAX)
        dt = 0.1 * (10.0 / (M * (P_DEG + 1))) / float(lam[0])
        lams.append(float(lam[0]))
        dts.append(dt)
        g.project()
        for s in range(1, 5):
            _swap(dist, g, rank, world)
            g.stage(s, dt)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), rhs=rhs, uq=g.get_state_q(), k0=g.k0,
             lams=np.array(lams), dts=np.array(dts), comm=np.array(list(g.comm_info().values())))
    g.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_processes_match_whole_box(world):
    import torch.multiprocessing as mp

    import paper_2312_07725_b200 as pkg
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
        whole = pkg.GpuSolver(pkg.SolverConfig(p=P_DEG, m=M, c1d=C1D))
        whole.init_case()
        np.testing.assert_array_equal(np.concatenate([x["rhs"] for x in parts]), whole.rhs())
        for k in range(STEPS):
            assert all(x["lams"][k] == whole.max_wavespeed() for x in parts)
            whole.rk4_step_dt(parts[0]["dts"][k])
        np.testing.assert_array_equal(np.concatenate([x["uq"] for x in parts]), whole.get_state_q())
        assert [int(x["k0"]) for x in parts] == [pkg.halo_plan(M, P_DEG, r, world)["k0"] for r in range(world)]
        # external-halo contexts carry no NCCL communicator
        assert all(int(x["comm"][0]) == 0 for x in parts)


def _nccl_worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist

    import paper_2312_07725_b200 as pkg
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    obj = [pkg.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    g = pkg.GpuSolver(pkg.SolverConfig(p=P_DEG, m=M, c1d=C1D, rank=rank, nranks=world, device=rank),
                      nccl_id=obj[0])
    comm = g.comm_info()
    g.init_case()
    rhs = g.rhs()
    t = g.advance(STEPS, cfl=0.1)
    np.savez(os.path.join(outdir, f"nccl{rank}.npz"), rhs=rhs, uq=g.get_state_q(), t=t,
             l2=g.l2_error(), comm=np.array([comm["nccl_nranks"], comm["nccl_rank"], comm["cuda_device"]]))
    g.close()
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_slabs_on_two_gpus_match_whole_box():
    """The NCCL path between DISTINCT GPUs (one process per GPU, grouped
    send/recv halos, lambda MAX and L2 SUM allreduces, inside the step graph):
    gathered slabs equal the whole box bitwise. Needs >= 2 GPUs (this pool has
    one per box, so it skips here; it runs on any multi-GPU node)."""
    import torch
    import torch.multiprocessing as mp

    import paper_2312_07725_b200 as pkg
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_nccl_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"nccl{r}.npz")) for r in range(world)]
        whole = pkg.GpuSolver(pkg.SolverConfig(p=P_DEG, m=M, c1d=C1D))
        whole.init_case()
        np.testing.assert_array_equal(np.concatenate([x["rhs"] for x in parts]), whole.rhs())
        t = whole.advance(STEPS, cfl=0.1)
        assert all(float(x["t"]) == t for x in parts)
        np.testing.assert_array_equal(np.concatenate([x["uq"] for x in parts]), whole.get_state_q())
        np.testing.assert_allclose(parts[0]["l2"], whole.l2_error(), rtol=1e-14)
        assert [tuple(x["comm"][:2]) for x in parts] == [(world, r) for r in range(world)]
