"""bench.py — RHS DOF-updates/s of the B200 NSFR path (BASELINE.json metric).

Workload (BASELINE.json configs[4], the metric's own config): isentropic vortex
on 128^3 curvilinear hexes (beta = 1/20 warp), p = 4, c_+, EC + Roe surface
flux, weight-adjusted inverse, classical RK4 at CFL 0.1. One STEP = one RK4
step = 4 RHS evaluations, each updating every DOF (DOF = elements x (p+1)^3 x 5).
Strong scaling: the 128^3 box is split into z-slabs over N GPUs (one process
per GPU, NCCL face-halo exchange + lambda_max allreduce per step).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

`python bench.py --gpus N` (N > 1) outside torchrun re-launches itself under
`torch.distributed.run` with N ranks; every rank prints the NCCL communicator
it got (size, rank, device) to stderr, and rank 0's JSON carries the list.

Prints ONE JSON line on rank 0. The CPU legs (cpu_baseline and --impl
reference) run the reference's own compiled primitives (oracle/_ref, built
from /root/reference/proj/src) under the residual glue, on a bounded sample:
the periodic 128x128x16 z-slab of the 128^3 box, one RHS
per sample, median of the samples, scaled per element to 128^3 (extrapolation).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from flop_model import bytes_per_element, per_element, survey_per_element  # noqa: E402

METRIC = "RHS DOF-updates/sec (fp64, 3D Euler NSFR)"
UNIT = "DOF-updates/s"
P_DEG, M = 4, 128
C_PLUS4 = 0.5 * 4.67e-5
WORKLOAD = "isentropic-vortex-128^3-p4-c_plus-EC+Roe-RK4"
CPU_SLAB = 16  # bounded CPU sample: planes [0, 16) of the 128^3 box, its own halos (periodic slab)


def read_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no nvidia-smi samples"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class CpuSlab:
    """The reference's CPU path (oracle/_ref) on the periodic 128x128x16 z-slab
    of the bench box: same p / c_+ / EC+Roe / metrics as the GPU workload. The
    slab's halo planes are its own end planes (wrapped), taken once from the
    initial state, so every sample is one full RHS of 262,144 elements."""

    def __init__(self, threads: int):
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from oracle_lib import LIBS, Config, CpuSolver  # CPU baseline legs only
        self.kind = "ref" if os.path.exists(LIBS["ref"][0]) else "oracle"
        self.threads = threads
        t0 = time.perf_counter()
        self.s = CpuSolver(self.kind, Config(p=P_DEG, m=M, c1d=C_PLUS4, case="vortex", roe=True,
                                             k0=0, k1=CPU_SLAB, workers=threads))
        self.u = self.s.initial_state()
        lo, hi = self.s.boundary_traces(self.u)
        self.halo_lo, self.halo_hi = hi, lo
        self.setup_s = time.perf_counter() - t0
        self.dof = M * M * CPU_SLAB * (P_DEG + 1) ** 3 * 5

    def rhs_seconds(self) -> float:
        t0 = time.perf_counter()
        self.s.rhs(self.u, self.halo_lo, self.halo_hi)
        return time.perf_counter() - t0

    def sample(self, n: int, warmup: int = 1):
        for _ in range(warmup):
            self.rhs_seconds()
        secs = [self.rhs_seconds() for _ in range(n)]
        med = statistics.median(secs)
        return self.dof / med, med, secs

    def describe(self, n: int) -> str:
        return (f"periodic {M}x{M}x{CPU_SLAB} z-slab of the {M}^3 box (262,144 elements, p=4, c_+, "
                f"EC+Roe, the reference's metrics of those elements), one RHS per sample, median of "
                f"{n} after 1 warm-up, {self.threads} threads; DOF-updates/s per element is the "
                f"128^3 rate (extrapolation: the full box needs ~75 GB of reference metrics)")

    @property
    def kind_name(self) -> str:
        return "reference" if self.kind == "ref" else "port"


def run_reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    cs = CpuSlab(threads)
    val, med, secs = cs.sample(args.steps, warmup=args.warmup)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": med * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (analytic isentropic vortex IC)",
        "config": {"workload": WORKLOAD, "p": P_DEG, "elements": f"{M}x{M}x{CPU_SLAB} slab of {M}^3",
                   "step": "one RHS of the slab (median over steps)"},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": cs.kind_name,
                         "sample": cs.describe(args.steps), "cpu_model": cpu_model(),
                         "setup_s": cs.setup_s, "rhs_s": secs},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch_command(args, argv) -> list[str] | None:
    """`bench.py --gpus N` (N > 1) outside a torchrun environment: the command
    that re-runs it with N ranks (one process per GPU), else None."""
    if args.impl != "b200" or args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *argv]


def run_gpu_arm(args):
    import torch
    import paper_2312_07725_b200 as pkg

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}: launch N>1 with "
                         f"`python bench.py --gpus N` (it starts N ranks) or under torchrun")
    device = local
    torch.cuda.set_device(device)
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        obj = [pkg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    cfg = pkg.SolverConfig(p=P_DEG, m=M, c1d=C_PLUS4, case="vortex", roe=True, device=device,
                           rank=rank, nranks=world)
    g = pkg.GpuSolver(cfg, nccl_id=nccl_id)
    comm = {"rank": rank, "world": world, **g.comm_info()}
    print(json.dumps({"nccl_comm": comm}), file=sys.stderr, flush=True)
    if world > 1:
        import torch.distributed as dist
        comms = [None] * world
        dist.all_gather_object(comms, comm)
        bad = [c for c in comms if c["nccl_nranks"] != world]
        if bad:
            raise SystemExit(f"bench.py: NCCL communicator size != {world}: {bad}")
    else:
        comms = [comm]
    g.init_case()
    fp64_peak, peak_mhz = pkg.measure_fp64_peak(device, with_clock=True)
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    nominal = sms * 128 * peak_mhz * 1e6 / 1e12  # SMs x 64 DFMA/clk x 2 flop x measured clock

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    # warm-up (also captures the CUDA graph of one step)
    g.advance(args.warmup, cfl=0.1)
    barrier()
    launches0 = g.launch_count()
    with ClockSampler(device) as clk:
        ms_total, kms = g.time_steps(args.steps, cfl=0.1, per_kernel=True)
    launches = g.launch_count() - launches0
    barrier()
    ms_max = ms_total
    # per-launch averages (4 K2 + 4 K3 launches per step; K1 is the prologue, outside)
    k2_ms = kms[1] / (4 * args.steps)
    k3_ms = kms[2] / (4 * args.steps)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms_total], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t[0])
    ne_total = M ** 3
    dof_total = ne_total * (P_DEG + 1) ** 3 * 5
    value = 4 * dof_total * args.steps / (ms_max / 1e3)

    # e2e through the public API with host buffers (pinned): every step uploads
    # the state from host memory, runs one RK4 step and downloads the new state
    # (rk4_step_host: the copies pipelined with the compute over element chunks).
    # Headline: the reference's loop `dt = adaptive_dt(u, 0.1); u = rk4_step(u, dt)`
    # (SPEC.md:466-483), adaptive_dt of each output computed on its way out, so the
    # CFL-0.1 adaptive steps of `value` run without a barrier inside the step.
    # Also reported: dt <= 0 (lambda_max of the uploaded state first: the
    # pipeline drains once per step) and the unpipelined set_state/step/get_state.
    host = torch.empty(g.state_shape, dtype=torch.float64, pin_memory=True).numpy()
    g.get_state(out=host)
    e2e_steps = max(1, min(args.steps, 3))

    def e2e_run(step):
        step()  # warm-up
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            step()
        sec = (time.perf_counter() - t0) / e2e_steps
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([sec], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sec = float(t[0])
        return sec

    dt_box = [g.rk4_step_host(host, host, cfl=0.1)[2]]

    def chained():
        dt_box[0] = g.rk4_step_host(host, host, dt=dt_box[0], cfl=0.1)[2]

    e2e_sec = e2e_run(chained)
    e2e_barrier_sec = e2e_run(lambda: g.rk4_step_host(host, host, dt=0.0, cfl=0.1))
    e2e_plain_sec = e2e_run(lambda: (g.set_state(host), g.rk4_step(0.1), g.get_state(out=host)))
    e2e_val = 4 * dof_total / e2e_sec
    state_bytes = host.nbytes

    fm = per_element(P_DEG)
    sv = survey_per_element(P_DEG)["flops_total"]
    ne_local = g.ne
    k2_tflops = fm["flops_k2"] * ne_local / (k2_ms * 1e-3) / 1e12
    step_rate = ne_local * 4 * args.steps / (ms_total * 1e-3) / 1e12  # element-RHS per s / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "k_residual_p4_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            tr = json.load(f)
        traffic = tr.get("dram_bytes_per_element", 0) * ne_local
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "node_updates_per_s": value / 5,  # the metric per node (5 states per node)
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (analytic isentropic vortex IC on the reference's warped grid)",
        "config": {"workload": WORKLOAD, "elements": f"{M}^3", "p": P_DEG, "c1d": C_PLUS4,
                   "surface_flux": "EC+Roe", "parallelism": f"z-slab x{world}",
                   "l2_flush": "inputs larger than L2 (state 10.5 GB per copy)"},
        "roofline": {"bound": "fp64", "achieved": k2_tflops, "peak": fp64_peak, "unit": "TFLOP/s",
                     "frac": k2_tflops / fp64_peak, "traffic": traffic,
                     "kernel": f"k_residual<{P_DEG + 1}>",
                     "peak_source": "measured live: DFMA loop (nsfr_gpu_measure_fp64_peak_ex); "
                                    "MEASURED_PEAKS.json has no fp64 entry",
                     "peak_sm_mhz": peak_mhz, "peak_nominal": nominal,
                     "frac_nominal": k2_tflops / nominal,
                     "flops_per_element": fm["flops_k2"], "elements_per_launch": ne_local,
                     "launch_ms": k2_ms, "k3_launch_ms": k3_ms,
                     "k3_tflops": fm["flops_k3"] * ne_local / (k3_ms * 1e-3) / 1e12,
                     "step_frac": (fm["flops_total"] * ne_local * 4 * args.steps / (ms_total * 1e-3) / 1e12)
                     / fp64_peak,
                     "step_frac_table": {
                         "model_vs_measured": fm["flops_total"] * step_rate / fp64_peak,
                         "model_vs_nominal": fm["flops_total"] * step_rate / nominal,
                         "survey_vs_measured": sv * step_rate / fp64_peak,
                         "survey_vs_nominal": sv * step_rate / nominal,
                         "flops_model": fm["flops_total"], "flops_survey": sv},
                     "hbm_b_alg_gbs": bytes_per_element(P_DEG)["b_alg"] * ne_local / (
                         (k2_ms + k3_ms) * 1e-3) / 1e9,
                     "hbm_peak_gbs": read_peaks().get("hbm_gbs")},
        "clocks": clk.summary(),
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": state_bytes,
                "d2h_bytes_per_step": state_bytes, "steps": e2e_steps,
                "api": "rk4_step_host (nsfr_gpu_rk4_step_host): dt = adaptive_dt(u, 0.1) of the "
                       "previous output, pinned host state in and out every step",
                "in_step_adaptive_value": 4 * dof_total / e2e_barrier_sec,
                "unpipelined_value": 4 * dof_total / e2e_plain_sec},
        "gpu_launches": int(launches),
        "nccl": comms,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        g.close()  # host RAM for the reference's slab metrics
        threads = os.cpu_count() or 1
        cs = CpuSlab(threads)
        val, med, secs = cs.sample(3)
        out["cpu_baseline"] = {"value": val, "unit": UNIT, "cores": threads, "kind": cs.kind_name,
                               "cpu_model": cpu_model(), "sample": cs.describe(3),
                               "setup_s": cs.setup_s, "rhs_s": secs}
    g.close()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cmd = relaunch_command(args, sys.argv[1:])
    if cmd:
        raise SystemExit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
