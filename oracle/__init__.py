"""CPU oracle for the FPCK v2 checkpoint image — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package. See fpck.py's header.
"""
from . import fpck  # noqa: F401
