"""Driver for an ncu capture of the device coefficient assembly (assemble_kernel):
the C3 grid's 9 planes (16384x128, a = 0.9, s = -2, m = 0) in one batch."""
import sys; sys.path.insert(0,'.')
from paper_2010_04760_b200 import planes
p = planes.problem(16384, 128, a=0.9, spin=-2, mmode=0)
print("max_speed", p["max_speed"])
