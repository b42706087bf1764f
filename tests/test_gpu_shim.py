"""The drop-in boundary from the reference's side, on the GPU: oracle/_ref/shim_demo
(built by oracle/Makefile where the reference headers are) builds operators,
the warped mapping and conservative-curl metrics with the reference's own
setup code, drives libnsfr_b200.so through the C++ shim of INTEGRATION.md
(integration/gpu_solver.hpp: assemble_rhs, adaptive_dt, rk4_step(field, dt)
on host fields) and checks it against the reference build under the residual
glue in the same process: RHS within max(1e-12, 4 x the reference's 1-ulp
floor), three RK4 step increments within 1e-10, adaptive dt within 1e-14."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "oracle", "_ref", "shim_demo")


@pytest.mark.skipif(not os.path.exists(DEMO), reason="oracle/_ref/shim_demo not built (needs the reference headers)")
@pytest.mark.parametrize("p,m,cplus", [(3, 4, 1), (4, 3, 0), (5, 2, 1)])
def test_reference_shim_drives_the_gpu(p, m, cplus):
    r = subprocess.run([DEMO, str(p), str(m), str(cplus)], capture_output=True, text=True, timeout=600)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else "{}"
    res = json.loads(line)
    assert r.returncode == 0 and res.get("ok"), (r.returncode, res, r.stderr[-2000:])
