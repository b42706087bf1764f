"""Multi-rank z-slab path on CPU (gloo, world size 2 and 3).

Each rank owns the slab the product's halo plan assigns
(nsfr_gpu_halo_plan_for), computes its boundary face traces with the CPU
checker, exchanges them with the SAME send/recv pattern the CUDA path issues
through NCCL (send lo->peer_lo, recv hi<-peer_hi, send hi->peer_hi,
recv lo<-peer_lo), then evaluates the residual with the received halos. The
gathered result must equal the whole-box residual bitwise, and the allreduced
lambda_max / L2 / entropy change must match the whole-box values."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle_lib import Config, CpuSolver


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, m, p, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2312_07725_b200 as P
        plan = P.halo_plan(m, p, rank, world)
        cfg = Config(p=p, m=m, k0=plan["k0"], k1=plan["k1"], workers=2)
        solver = CpuSolver("oracle", cfg)
        full = CpuSolver("oracle", Config(p=p, m=m, workers=2))
        u_all = full.initial_state()
        u = np.ascontiguousarray(u_all[m * m * plan["k0"]:m * m * plan["k1"]])
        send_lo, send_hi = solver.boundary_traces(u)
        halo_lo = torch.empty(send_lo.shape, dtype=torch.float64)
        halo_hi = torch.empty(send_hi.shape, dtype=torch.float64)
        reqs = [dist.isend(torch.from_numpy(send_lo), plan["peer_lo"], tag=1),
                dist.irecv(halo_hi, plan["peer_hi"], tag=1),
                dist.isend(torch.from_numpy(send_hi), plan["peer_hi"], tag=2),
                dist.irecv(halo_lo, plan["peer_lo"], tag=2)]
        for r in reqs:
            r.wait()
        dudt, ds = solver.rhs(u, halo_lo.numpy(), halo_hi.numpy(), entropy=True)
        lam = torch.tensor([solver.max_wavespeed(u)], dtype=torch.float64)
        dist.all_reduce(lam, op=dist.ReduceOp.MAX)
        l2 = torch.from_numpy(solver.l2_sq(u, 0.0))
        dist.all_reduce(l2)
        ds_t = torch.tensor([ds], dtype=torch.float64)
        parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, ds_t)  # fixed rank-order combine (deterministic)
        ds_sum = sum(float(x) for x in parts)
        np.save(os.path.join(out_dir, f"dudt_{rank}.npy"), dudt)
        if rank == 0:
            want, ds_want = full.rhs(u_all, entropy=True)
            np.save(os.path.join(out_dir, "want.npy"), want)
            np.save(os.path.join(out_dir, "scalars.npy"),
                    np.array([float(lam[0]), full.max_wavespeed(u_all), *l2.numpy(),
                              *full.l2_sq(u_all, 0.0), ds_sum, ds_want]))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m", [(2, 4), (3, 6)])
def test_slab_exchange_matches_whole_box(tmp_path, world, m):
    p = 3
    mp.spawn(_worker, args=(world, _free_port(), m, p, str(tmp_path)), nprocs=world, join=True)
    import paper_2312_07725_b200 as P
    want = np.load(tmp_path / "want.npy")
    got = []
    for r in range(world):
        got.append(np.load(tmp_path / f"dudt_{r}.npy"))
        h = P.halo_plan(m, p, r, world)
        assert got[-1].shape[0] == m * m * (h["k1"] - h["k0"])
    np.testing.assert_array_equal(np.concatenate(got), want)
    s = np.load(tmp_path / "scalars.npy")
    assert s[0] == s[1]                                # lambda_max allreduce(MAX)
    np.testing.assert_allclose(s[2:4], s[4:6], rtol=1e-13)  # L2 sums allreduce(SUM)
    assert s[6] == pytest.approx(s[7], rel=1e-12)      # entropy change
