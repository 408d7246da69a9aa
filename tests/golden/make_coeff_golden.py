"""Generate tests/golden/coef_kat.npz: the reference's 36-digit known-answer
vectors of the generated wave-operator kernels (proj/tests/golden_coeffs.inc,
checked by proj/tests/test_geometry.cpp:119-139 at 1e-26) as double-double
pairs, with the inputs the reference test builds (rat(p, q) = DDReal(p) /
DDReal(q), test_geometry.cpp:14) and the UNMODIFIED reference library's own
wave_op_coeffs<DDReal> outputs on those inputs (the bitwise target of the
GPU evaluator).  Run in the build container:

    python tests/golden/make_coeff_golden.py
"""
from __future__ import annotations

import os
import re
import sys
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402

INC = "/root/reference/proj/tests/golden_coeffs.inc"


def dd_of(text: str) -> tuple[float, float]:
    """Nearest double-double of a decimal string (hi = round(x), lo = round(x - hi))."""
    x = Fraction(text)
    hi = float(x)
    return hi, float(x - Fraction(hi))


def parse(path: str):
    body = open(path).read()
    rows = []
    pat = re.compile(r"\{([-\d,\s]+),\s*\{([^}]*)\}\}", re.S)
    for m in pat.finditer(body.split("golden_coeff_rows[] = {", 1)[1]):
        ints = [int(t) for t in m.group(1).replace("\n", " ").split(",") if t.strip()]
        vals = re.findall(r'"([^"]+)"', m.group(2))
        assert len(ints) == 12 and len(vals) == 11, (ints, vals)
        rows.append((ints, vals))
    return rows


def main():
    rows = parse(INC)
    n = len(rows)
    inp = np.zeros((n, 5, 2))
    sm = np.zeros((n, 2), dtype=np.int32)
    want = np.zeros((n, 11, 2))
    for i, (ints, vals) in enumerate(rows):
        Mp, Mq, ap, aq, Sp, Sq, spin, mmode, rp, rq, cp, cq = ints
        for q, (p_, q_) in enumerate(((rp, rq), (cp, cq), (Mp, Mq), (ap, aq), (Sp, Sq))):
            inp[i, q] = O.ref_rat(p_, q_)
        sm[i] = (spin, mmode)
        for q, v in enumerate(vals):
            want[i, q] = dd_of(v)
    host = O.ref_wave_op_coeffs(inp, sm)
    out = os.path.join(HERE, "coef_kat.npz")
    np.savez_compressed(out, inp=inp, spin_mmode=sm, want=want, host=host,
                        source=np.array("proj/tests/golden_coeffs.inc"))
    print(f"{out}: {n} rows")


if __name__ == "__main__":
    main()
