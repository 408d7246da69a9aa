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
