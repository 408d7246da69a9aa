"""The ctypes snippet of INTEGRATION.md §3, executed as written (so the
documented minimal binding stays correct), against the same run through
paper_2010_04760_b200.hwgpu."""
import os
import re

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_integration_ctypes_snippet(cuda_ok):
    from paper_2010_04760_b200 import synthetic
    from paper_2010_04760_b200.hwgpu import GpuEvolution, SchemeSpec
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"```python\n(.*?)```", text, re.S).group(1)
    n, nt = 256, 16
    prob = synthetic.problem(n, nt)
    env = dict(n=n, nt=nt, drho=prob["drho"], dth=prob["dtheta"], parity=prob["parity"],
               coef=np.ascontiguousarray(prob["coef"]), cot=np.ascontiguousarray(prob["cotth"]),
               u=synthetic.initial_state(prob), dt=synthetic.select_dt(prob))
    u0 = env["u"].copy()
    cwd = os.getcwd()
    os.chdir(ROOT)
    try:
        exec(compile(code, "INTEGRATION.md", "exec"), env)
    finally:
        os.chdir(cwd)
    assert env["rc"] == 0
    g = GpuEvolution(n, nt, prob["drho"], prob["dtheta"], prob["parity"], prob["coef"],
                     prob["cotth"], SchemeSpec("weno5", "mixed"))
    g.set_state(u0)
    g.launch_steps("ssprk33", env["dt"], 0, 1000)
    assert np.array_equal(env["u"][:, 2:-2, 4:-4], g.get_state()[:, 2:-2, 4:-4])


def test_integration_assembly_snippet(cuda_ok):
    """INTEGRATION.md §3's coefficient-assembly snippet (second python block),
    executed as written on the reference's own DD grid: the planes are the
    reference's assemble_coefficients output bit for bit."""
    import ctypes as C
    import oracle as O
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.findall(r"```python\n(.*?)```", text, re.S)[1]
    ref = O.RefSolver(O.Physics(a=0.9, spin=-2, mmode=0), 256, 16, workers=4)
    want, ms = ref.coeffs_all_dd()
    rho, cth = ref.grid_dd()
    env = dict(C=C, np=np, dp=C.POINTER(C.c_double),
               lib=C.CDLL(os.path.join(ROOT, "paper_2010_04760_b200", "libhwgpu.so")),
               nrho=256, ntheta=16, rho_dd=np.ascontiguousarray(rho), costh_dd=np.ascontiguousarray(cth))
    exec(compile(code, "INTEGRATION.md", "exec"), env)
    assert env["rc"] == 0
    for q in range(14):
        assert np.array_equal(env["planes"][q].view(np.int64), want[q].reshape(-1).view(np.int64)), q
    assert np.array_equal(env["ms"].view(np.int64), ms.view(np.int64))
